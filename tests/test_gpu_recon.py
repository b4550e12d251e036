"""GPU GridFill reconstruction (lag_gridfill, NEXT-2 in SURVEY.md §8(f))
against the oracle's GridFill (oracle/metrics.py:grid_fill, pinned in
test_oracle_pins.py).  Both evaluate Eq. 1 along the shortest-bracket axis in
uncontracted f64 in the same order, so holes must match bitwise."""
import numpy as np
import pytest

import lag_inputs as L
from helpers import global_slices, gpu_block

pytestmark = pytest.mark.gpu


def _lattice(dims):
    idx = np.indices(dims[::-1]).reshape(len(dims), -1)[::-1].T     # x fastest
    return np.ascontiguousarray(idx)


def _gpu_fill(values, valid, dims):
    import torch
    import paper_2004_02003_b200 as P
    v = torch.from_numpy(values).cuda()
    ok = torch.from_numpy(valid.astype(np.uint8)).cuda()
    out, filled = P.lag_gridfill(v, ok, dims)
    return out.cpu().numpy(), filled.cpu().numpy().astype(bool)


def _check(values, valid, dims):
    from oracle.metrics import grid_fill
    lat = _lattice(dims)
    ref, ref_filled = grid_fill(lat, np.where(valid[:, None], values, np.nan), valid, ~valid)
    out, filled = _gpu_fill(np.where(valid[:, None], values, np.nan), valid, dims)
    np.testing.assert_array_equal(filled, ref_filled)
    np.testing.assert_array_equal(out[valid], values[valid])
    np.testing.assert_array_equal(out[filled], ref[filled])                 # bitwise
    assert np.isnan(out[~valid & ~filled]).all()
    return int(filled.sum())


@pytest.mark.parametrize("dims", [(37, 23), (17, 13, 11), (1, 9), (5, 1, 7), (64, 3, 2)])
def test_gridfill_random_masks_bitwise(dims):
    rng = np.random.default_rng(sum(dims))
    n = int(np.prod(dims))
    for k in (1, len(dims)):
        values = rng.standard_normal((n, k))
        valid = rng.random(n) < 0.7
        assert _check(values, valid, dims) >= 0


def test_gridfill_band_holes_and_affine_exactness():
    """Bands of holes 1..6 seeds wide (the BTO pattern next to block faces);
    an affine field is reproduced exactly up to rounding (Eq. 2)."""
    dims = (40, 30, 20)
    lat = _lattice(dims).astype(np.float64)
    values = lat @ np.array([[0.5, -1.0, 2.0], [1.5, 0.25, -0.5], [-0.75, 1.0, 0.125]]) + 3.0
    valid = np.ones(lat.shape[0], bool)
    for w, x0 in zip(range(1, 7), (3, 9, 15, 21, 28, 33)):
        valid &= ~((lat[:, 0] >= x0) & (lat[:, 0] < x0 + w))
    valid &= ~((lat[:, 1] >= 12) & (lat[:, 1] < 15) & (lat[:, 2] < 4))
    assert _check(values, valid, dims) > 0
    out, filled = _gpu_fill(np.where(valid[:, None], values, np.nan), valid, dims)
    np.testing.assert_allclose(out[filled], values[filled], rtol=0, atol=1e-12)


def test_gridfill_bto_holes_from_the_cuda_path():
    """Real hole pattern: C2 (ABC 3D) BTO flow map of the 2x2x2 decomposition
    from the CUDA path, assembled on the global seed lattice; GPU GridFill
    equals the oracle's GridFill on it bitwise."""
    cfg = L.make_config("C2", scale=24, interval=8, cycles=8)
    g = cfg["grid"]
    sl = global_slices(cfg, cfg["interval"])
    stride = 1
    dims = tuple(int(x) for x in g.nodes[:g.dim])
    values = np.full((int(np.prod(dims)), g.dim), np.nan)
    valid = np.zeros(values.shape[0], bool)
    for b in L.decompose(g, cfg["layout"]):
        start, end, status, _ = gpu_block(cfg, b, sl, stride)
        node = np.rint((start - np.array(g.origin[:g.dim])) / np.array(g.spacing[:g.dim])).astype(np.int64)
        flat = node[:, 0] + dims[0] * (node[:, 1] + dims[1] * (node[:, 2] if g.dim == 3 else 0))
        values[flat] = end
        valid[flat] = status == 0
    assert (~valid).sum() > 0
    assert _check(np.nan_to_num(values), valid, dims) > 0


def test_gridfill_rejects_bad_arguments():
    import torch
    import paper_2004_02003_b200 as P
    v = torch.zeros((6, 2), dtype=torch.float64, device="cuda")
    ok = torch.ones(6, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        P.lag_gridfill(v, ok, (4, 2))
    with pytest.raises(P.LagError):
        P.lag_gridfill(v.cpu(), ok.cpu(), (3, 2))                  # host memory


def test_gridfill_crossing_slabs_leave_unfillable_lines():
    """Three crossing hole slabs (the pattern at block-face intersections):
    nodes on the slab-intersection lines have no bracket on any axis and stay
    NaN / unfilled, everything else matches the oracle bitwise."""
    dims = (24, 20, 16)
    lat = _lattice(dims)
    near = [np.abs(lat[:, a] - dims[a] // 2) < 2 for a in range(3)]
    valid = ~(near[0] | near[1] | near[2])
    values = np.random.default_rng(5).standard_normal((lat.shape[0], 3))
    _check(values, valid, dims)
    out, filled = _gpu_fill(np.where(valid[:, None], values, np.nan), valid, dims)
    two = (near[0].astype(int) + near[1] + near[2]) >= 2
    assert not filled[two].any() and np.isnan(out[two]).all()
    assert filled[~valid & ~two].all()
