"""GPU pathline stitching (lag_stitch) against the oracle
(oracle/pathline.py, pinned in test_oracle_pins.py).

Tolerance: each step computes u = (x - o)/h, the Kuhn weights and the sum of
d + 1 weighted ends in f64. The GPU and numpy differ only in the summation
order of that last sum (a few ulp). Over K steps these differences are
amplified by the flow maps' Lipschitz constants (< 2 per step here). We allow
1e-9 lattice spacings. Statuses must be equal, except where the oracle's
trajectory passes within 1e-9 spacings of the hull (an ulp can decide
inside/outside there)."""
import numpy as np
import pytest

import lag_inputs as L
from helpers import global_slices, gpu_block

pytestmark = pytest.mark.gpu

TOL = 1e-9
EXCUSE = 1e-9


def _lat(dims, origin, sp):
    idx = np.indices(dims[::-1]).reshape(len(dims), -1)[::-1].T
    return np.asarray(origin) + idx * np.asarray(sp)


def _gpu(ends, valid, dims, o, sp, starts):
    import torch
    import paper_2004_02003_b200 as P
    e = torch.from_numpy(np.ascontiguousarray(ends)).cuda()
    v = None if valid is None else torch.from_numpy(np.ascontiguousarray(valid).astype(np.uint8)).cuda()
    path, st = P.lag_stitch(e, torch.from_numpy(np.ascontiguousarray(starts)).cuda(), dims, o, sp, valid=v)
    return path.cpu().numpy(), st.cpu().numpy()


def _check(ends, valid, dims, o, sp, starts):
    from oracle.pathline import stitch
    ref, rst, _, min_hull = stitch(ends, valid, dims, o, sp, starts)
    got, gst = _gpu(ends, valid, dims, o, sp, starts)
    excused = min_hull < EXCUSE
    assert not ((gst != rst) & ~excused).any(), np.nonzero((gst != rst) & ~excused)[0][:10]
    same = gst == rst
    both = same[:, None] & ~np.isnan(ref[:, :, 0]) & ~np.isnan(got[:, :, 0])
    np.testing.assert_array_equal(np.isnan(got[same]), np.isnan(ref[same]))
    err = np.abs(got - ref)[both] / np.asarray(sp)
    assert err.size == 0 or err.max() <= TOL, err.max()
    return got, gst, rst


@pytest.mark.parametrize("dim", [2, 3])
def test_stitch_nonlinear_maps_with_holes_and_exits(dim):
    rng = np.random.default_rng(dim)
    dims = (17, 13, 11)[:dim]
    o = (-0.5, 0.25, 1.0)[:dim]
    sp = tuple(0.1 + 0.2 * rng.random(dim))
    X = _lat(dims, o, sp)
    K = 5
    ends = np.stack([X + 0.6 * np.asarray(sp) * np.sin(1.3 * X[:, ::-1] + k) + 0.2 * np.asarray(sp)
                     for k in range(K)])
    valid = rng.random((K, X.shape[0])) > 0.02
    lo, hi = np.asarray(o), np.asarray(o) + (np.asarray(dims) - 1) * np.asarray(sp)
    starts = lo + (hi - lo) * (rng.random((3000, dim)) * 1.1 - 0.05)
    starts[:50] = X[rng.integers(0, X.shape[0], 50)]                       # exactly on nodes
    _, gst, rst = _check(ends, valid, dims, o, sp, starts)
    assert (rst == 0).any() and (rst == 1).any() and (rst == 2).any()
    _check(ends, None, dims, o, sp, starts)


def test_stitch_affine_composition_on_gpu():
    dims, o, sp = (9, 8, 7), (-1.0, 0.5, 2.0), (0.5, 0.25, 0.3)
    X = _lat(dims, o, sp)
    c = np.array(o) + (np.array(dims) - 1) * np.array(sp) / 2
    M = np.array([[1.02, 0.05, 0.0], [-0.03, 0.98, 0.02], [0.01, 0.0, 1.01]])
    b = np.array([0.02, -0.01, 0.03])
    ends = np.stack([(X - c) @ M.T + c + b] * 3)
    q = c + (np.random.default_rng(4).random((500, 3)) - 0.5) * (np.array(dims) - 1) * np.array(sp) * 0.5
    got, gst = _gpu(ends, None, dims, o, sp, q)
    assert (gst == 0).all()
    x = q.copy()
    for k in range(3):
        x = (x - c) @ M.T + c + b
        np.testing.assert_allclose(got[:, k + 1], x, rtol=0, atol=1e-13)


def test_stitched_bto_pathlines_vs_ground_truth():
    """The post hoc chain on the GPU. BTO flow maps of K = 4 intervals of a
    2x2x2 decomposition (C2, ABC, 24^3, stride 2) are filled by lag_gridfill
    and stitched by lag_stitch from the odd nodes, which lie between the
    stride-2 seeds. The path is compared with the oracle stitching the
    oracle-GridFilled maps, and, as an accuracy property, with the ground
    truth: one RK4 run at full resolution over all K*I cycles (SPEC.md:338
    asks for within 2 cells)."""
    import torch
    import paper_2004_02003_b200 as P
    from oracle.metrics import grid_fill
    K, I, stride = 4, 8, 2
    cfg = L.make_config("C2", scale=24, interval=I, cycles=K * I)
    g = cfg["grid"]
    dims = tuple(int(-(-g.nodes[a] // stride)) for a in range(3))
    n = int(np.prod(dims))
    sp = tuple(stride * h for h in g.spacing)
    lat = np.indices(dims[::-1]).reshape(3, -1)[::-1].T
    ends_gpu, ends_ref = [], []
    for k in range(K):
        sl = global_slices(cfg, I, t0_cycle=k * I)
        ends = np.zeros((n, 3))
        valid = np.zeros(n, bool)
        for b in L.decompose(g, cfg["layout"]):
            start, end, status, _ = gpu_block(cfg, b, sl, stride)
            node = np.rint(start / np.array(sp)).astype(np.int64)
            flat = node[:, 0] + dims[0] * (node[:, 1] + dims[1] * node[:, 2])
            ends[flat] = end
            valid[flat] = status == 0
        f, _ = P.lag_gridfill(torch.from_numpy(ends).cuda(), torch.from_numpy(valid.astype(np.uint8)).cuda(), dims)
        ends_gpu.append(f.cpu().numpy())
        rf, rin = grid_fill(lat, ends, valid, ~valid)
        ends_ref.append(np.where(valid[:, None], ends, rf))
    ends_gpu = np.stack(ends_gpu)
    np.testing.assert_array_equal(np.isnan(ends_gpu), np.isnan(np.stack(ends_ref)))
    # ground truth: one block over the whole domain, stride 1, one K*I-cycle interval
    whole = L.Block(0, (0, 0, 0), (0, 0, 0), g.nodes)
    gt_start, gt_end, gt_status, _ = gpu_block(cfg, whole, global_slices(cfg, K * I), 1)
    node = np.rint(gt_start / np.array(g.spacing)).astype(np.int64)
    odd = (node % 2 == 1).all(axis=1) & (gt_status == 0)
    starts = gt_start[odd]
    vmask = ~np.isnan(ends_gpu).any(axis=2)                  # unfillable holes stay invalid
    got, gst, rst = _check(np.stack(ends_ref), vmask, dims, (0.0, 0.0, 0.0), sp, starts)
    gpath, gst2 = _gpu(ends_gpu, vmask, dims, (0.0, 0.0, 0.0), sp, starts)
    np.testing.assert_array_equal(gpath, got)                 # same maps bitwise -> same paths
    ok = gst == 0
    assert ok.mean() > 0.7
    err = np.linalg.norm(got[ok, K] - gt_end[odd][ok], axis=1) / g.spacing[0]
    assert np.median(err) < 2.0, np.median(err)
