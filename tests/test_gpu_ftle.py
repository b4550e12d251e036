"""GPU FTLE (lag_ftle) against the oracle's FTLE
(oracle/ftle.py, pinned in test_oracle_pins.py).

Tolerance: the gradient differs by at most 1 ulp per entry (the GPU
multiplies by 1/dx where numpy divides). C = J^T J differs by summation order
(a few ulp of its terms). lambda_max comes from LAPACK on one side and Jacobi
on the other; both are backward stable, so they agree to ~10 eps ||C|| =
10 eps lambda_max. FTLE = ln(lambda_max) / (2|T|) then agrees to ~1e-15 / |T|.
The test allows 1e-12 / |T|, absolute."""
import numpy as np
import pytest

import lag_inputs as L
from helpers import global_slices, gpu_block

pytestmark = pytest.mark.gpu


def _lattice_pts(dims, spacing):
    idx = np.indices(dims[::-1]).reshape(len(dims), -1)[::-1].T
    return idx * np.asarray(spacing, dtype=np.float64)


def _gpu_ftle(F, dims, sp, T):
    import torch
    import paper_2004_02003_b200 as P
    out, nd = P.lag_ftle(torch.from_numpy(np.ascontiguousarray(F)).cuda(), dims, sp, T)
    return out.cpu().numpy(), nd


def _check(F, dims, sp, T):
    from oracle.ftle import ftle
    ref, nref = ftle(F, dims, sp, T)
    got, ngot = _gpu_ftle(F, dims, sp, T)
    assert ngot == nref
    np.testing.assert_array_equal(np.isnan(got), np.isnan(ref))
    ok = ~np.isnan(ref)
    np.testing.assert_allclose(got[ok], ref[ok], rtol=0, atol=1e-12 / abs(T))
    return got


def test_ftle_closed_forms_on_gpu():
    dims, sp = (9, 7, 5), (0.25, 0.5, 0.125)
    X = _lattice_pts(dims, sp)
    got = _check(X * np.array([2.0, 0.5, 1.0]), dims, sp, 1.0)
    np.testing.assert_allclose(got, np.log(2.0), atol=1e-14)
    got = _check(X + 0.3, dims, sp, 2.0)
    np.testing.assert_allclose(got, 0.0, atol=1e-14)
    k = 1.7
    F = X.copy()
    F[:, 0] += k * X[:, 1]
    got = _check(F, dims, sp, 3.0)
    np.testing.assert_allclose(got, 0.5 * np.log(1 + k * k / 2 + k * np.sqrt(1 + k * k / 4)) / 3.0, rtol=1e-13)


@pytest.mark.parametrize("dims", [(33, 29, 17), (130, 3, 2), (1, 5, 6), (61, 47), (2, 2)])
def test_ftle_smooth_random_maps_vs_oracle(dims):
    rng = np.random.default_rng(len(dims) * 100 + dims[0])
    sp = tuple(0.05 + 0.1 * rng.random(len(dims)))
    X = _lattice_pts(dims, sp)
    A = rng.standard_normal((len(dims), len(dims)))
    F = X @ (np.eye(len(dims)) + 0.5 * A).T + 0.2 * np.sin(3.0 * X[:, ::-1]) * rng.random(len(dims))
    _check(F, dims, sp, -1.25)


def test_ftle_degenerate_and_nonfinite():
    dims, sp = (6, 5, 4), (1.0, 1.0, 1.0)
    F = np.zeros((120, 3))
    got, nd = _gpu_ftle(F, dims, sp, 1.0)
    assert nd == 120 and (got == 0).all()
    F = _lattice_pts(dims, sp)
    F[37] = np.nan
    _check(F, dims, sp, 1.0)


def test_ftle_of_a_gpu_flow_map_after_gridfill():
    """The post hoc chain on the GPU — extract (BTO, C2 2x2x2 at 24^3),
    GridFill, FTLE — against the oracle's GridFill + FTLE on the same
    flow map."""
    import torch
    import paper_2004_02003_b200 as P
    from oracle.metrics import grid_fill
    from oracle.ftle import ftle
    cfg = L.make_config("C2", scale=24, interval=8, cycles=8)
    g = cfg["grid"]
    sl = global_slices(cfg, cfg["interval"])
    dims = tuple(int(x) for x in g.nodes[:g.dim])
    n = int(np.prod(dims))
    ends = np.zeros((n, g.dim))
    valid = np.zeros(n, bool)
    for b in L.decompose(g, cfg["layout"]):
        start, end, status, _ = gpu_block(cfg, b, sl, 1)
        node = np.rint((start - np.array(g.origin[:g.dim])) / np.array(g.spacing[:g.dim])).astype(np.int64)
        flat = node[:, 0] + dims[0] * (node[:, 1] + dims[1] * node[:, 2])
        ends[flat] = end
        valid[flat] = status == 0
    T = cfg["interval"] * cfg["dt"]
    sp = tuple(g.spacing[:g.dim])
    filled, _ = P.lag_gridfill(torch.from_numpy(ends).cuda(), torch.from_numpy(valid.astype(np.uint8)).cuda(), dims)
    got, _ = P.lag_ftle(filled, dims, sp, T)
    got = got.cpu().numpy()
    lat = np.indices(dims[::-1]).reshape(3, -1)[::-1].T
    ref_fill, ref_in = grid_fill(lat, ends, valid, ~valid)
    ref_ends = np.where(valid[:, None], ends, ref_fill)
    ref, _ = ftle(ref_ends, dims, sp, T)
    np.testing.assert_array_equal(np.isnan(got), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert ok.sum() > 0.8 * n          # (global-face exits leave unfillable lines)
    np.testing.assert_allclose(got[ok], ref[ok], rtol=0, atol=1e-12 / T)
