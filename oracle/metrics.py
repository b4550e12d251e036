"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's accuracy metric and its post hoc reconstruction, on CPU.

* Eq. 5 (§4.3): total average L2 = (1/p) sum_i ||b_i - m_i||.
  The printed sum runs i = 0..p while dividing by p; reading R9 takes
  i = 1..p (p terms).
* Eq. 6: Accuracy% = (C - L) / C * 100, C = cell side
  (reading R10: C = extent / (N - 1), min over axes; the paper's printed
  accuracy cells are (C - L)/C*100 truncated to 0.1 — pinned in
  tests/golden/paper_tables.json).
* Max-L2 folds: greatest max over intervals; average of
  per-interval maxima.
* Post hoc reconstruction (§3.2): Delaunay triangulation over the
  start locations of valid basis flows of the own and adjacent blocks, then
  barycentric interpolation of the end positions.  Reading R12: Qhull with
  joggle (QJ) over spatial tiles of the hole bands.
* Eq. 2 (§3.3): linear interpolation through a reconstructed hole
  equals interpolation between its valid neighbours — grid_fill_1d (the pin)
  and grid_fill (the lattice GridFill reconstruction), the
  fast alternative to Delaunay for large flow maps.
"""
from __future__ import annotations

import math
from typing import Dict, Iterable, List, Tuple

import numpy as np


def total_avg_l2(b: np.ndarray, m: np.ndarray) -> float:
    """Eq. 5 with i = 1..p (reading R9)."""
    b = np.asarray(b, dtype=np.float64)
    m = np.asarray(m, dtype=np.float64)
    if b.shape != m.shape:
        raise ValueError("length mismatch")
    p = b.shape[0]
    if p == 0:
        raise ValueError("no particles")
    return float(np.sqrt(((b - m) ** 2).sum(axis=1)).sum()) / p


def accuracy_pct(L: float, C: float) -> float:
    """Eq. 6: (C - L) / C * 100."""
    if not C > 0:
        raise ValueError("cell side must be positive")
    return (C - L) / C * 100.0


def paper_printed_accuracy(L: float, C: float) -> float:
    """How the paper prints Eq. 6: truncated (floored) to one decimal
    (reading R10; reproduces 33 of 35 printed cells)."""
    return math.floor(accuracy_pct(L, C) * 10.0 + 1e-9) / 10.0


def cell_side(grid) -> float:
    """C = extent / (N - 1) per axis = h_a; min over axes (reading R10)."""
    return float(min(grid.spacing[a] for a in range(grid.dim)))


def max_l2_stats(per_interval_max: Iterable[float]) -> Tuple[float, float]:
    """(greatest maximum, average maximum) over intervals."""
    vals = [float(v) for v in per_interval_max]
    if not vals:
        raise ValueError("no intervals")
    return max(vals), sum(vals) / len(vals)


def grid_fill_1d(f: np.ndarray, valid: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Eq. 1 / Eq. 2 along a lattice line: fill each invalid sample by linear
    interpolation between its nearest valid neighbours (Eq. 1), then evaluate
    the piecewise-linear interpolant at x.  Eq. 2 says this equals direct
    interpolation between the valid neighbours."""
    f = np.asarray(f, dtype=np.float64).copy()
    valid = np.asarray(valid, dtype=bool)
    idx = np.arange(f.size)
    vi = idx[valid]
    for i in idx[~valid]:
        left = vi[vi < i]
        right = vi[vi > i]
        if left.size == 0 or right.size == 0:
            raise ValueError("unfillable hole")
        x0, x2 = left[-1], right[0]
        f[i] = (i - x0) / (x2 - x0) * f[x2] + (x2 - i) / (x2 - x0) * f[x0]
    return np.interp(x, idx.astype(np.float64), f)


def barycentric_interpolate(points: np.ndarray, values: np.ndarray, queries: np.ndarray,
                            joggle: bool = True):
    """Delaunay over `points`, barycentric interpolation of `values`
    at `queries`.  Returns (interpolated [m, k], inside mask [m])."""
    from scipy.spatial import Delaunay
    points = np.asarray(points, dtype=np.float64)
    queries = np.asarray(queries, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    dim = points.shape[1]
    tri = Delaunay(points, qhull_options="QJ" if joggle else None)
    simp = tri.find_simplex(queries)
    inside = simp >= 0
    out = np.full((queries.shape[0], values.shape[1]), np.nan)
    if inside.any():
        s = simp[inside]
        T = tri.transform[s]                       # [m, dim+1, dim]
        r = queries[inside] - T[:, dim]
        lam = np.einsum("mij,mj->mi", T[:, :dim], r)
        lam = np.concatenate([lam, 1.0 - lam.sum(axis=1, keepdims=True)], axis=1)
        verts = tri.simplices[s]                   # [m, dim+1]
        out[inside] = np.einsum("mv,mvk->mk", lam, values[verts])
    return out, inside


def _recon_tile(args):
    pts_start, pts_end, q = args
    return barycentric_interpolate(pts_start, pts_end, q)


def reconstruct_holes(g_seeds: np.ndarray, start: np.ndarray, end: np.ndarray,
                      valid: np.ndarray, hole: np.ndarray, stride: int,
                      margin: int = 3, tile: int = 16, workers: int = 0):
    """Reconstruct end positions for `hole` seeds from the valid basis flows
    around them (own + adjacent blocks: with the global seed set the union is
    the same).  Holes are grouped in spatial tiles of `tile`
    lattice steps; each tile triangulates the valid seeds inside the bounding
    box of its holes grown by `margin` lattice steps (reading R12).  Tiles are
    independent and run in parallel over `workers` processes (0 = all cores).
    Returns (recon [n, dim] with NaN where not reconstructed, inside mask)."""
    g = np.asarray(g_seeds) // stride
    dim = start.shape[1]
    recon = np.full(end.shape, np.nan)
    inside = np.zeros(g.shape[0], dtype=bool)
    hidx = np.nonzero(hole)[0]
    if hidx.size == 0:
        return recon, inside
    tkey = g[hidx, :dim] // tile
    uniq, inv = np.unique(tkey, axis=0, return_inverse=True)
    inv = inv.ravel()
    # valid seeds indexed on the lattice for fast box queries
    shape = tuple(int(x) + 1 for x in g[:, :dim].max(axis=0))
    lattice = np.full(shape, -1, dtype=np.int64)
    vidx = np.nonzero(valid)[0]
    lattice[tuple(g[vidx, a] for a in range(dim))] = vidx
    jobs, sels = [], []
    for t in range(uniq.shape[0]):
        hsel = hidx[inv == t]
        lo = np.maximum(g[hsel, :dim].min(axis=0) - margin, 0)
        hi = np.minimum(g[hsel, :dim].max(axis=0) + margin + 1, shape)
        box = lattice[tuple(slice(int(lo[a]), int(hi[a])) for a in range(dim))].ravel()
        pts = box[box >= 0]
        if pts.size < dim + 1:
            continue
        jobs.append((start[pts], end[pts], start[hsel]))
        sels.append(hsel)
    if workers == 1 or len(jobs) < 4:
        results = [_recon_tile(j) for j in jobs]
    else:
        import multiprocessing as mp
        import os
        n = workers or os.cpu_count() or 1
        # spawn, not fork: the caller may hold CUDA / thread-pool locks
        with mp.get_context("spawn").Pool(n) as pool:
            results = pool.map(_recon_tile, jobs, chunksize=max(1, len(jobs) // (4 * n)))
    for hsel, (vals, ins) in zip(sels, results):
        recon[hsel] = vals
        inside[hsel] = ins
    return recon, inside


def grid_fill(lat: np.ndarray, values: np.ndarray, valid: np.ndarray, hole: np.ndarray):
    """GridFill reconstruction on the seed lattice (justified
    by Eq. 2): each hole is filled by linear interpolation (Eq. 1)
    between the nearest valid seeds on both sides along a lattice axis, using
    the axis with the shortest such bracket (ties averaged; reading R18).  `lat` are integer
    lattice coordinates [n, dim] (seed node // stride); returns
    (filled values [n, k] with NaN where no axis has both bounds, filled mask)."""
    lat = np.asarray(lat)
    dim = lat.shape[1]
    lo = lat.min(axis=0)
    shape = tuple(int(x) for x in (lat.max(axis=0) - lo + 1))
    idx = tuple((lat[:, a] - lo[a]) for a in range(dim))
    k = values.shape[1]
    V = np.full(shape + (k,), np.nan)
    ok = np.zeros(shape, dtype=bool)
    V[idx] = np.where(valid[:, None], values, np.nan)
    ok[idx] = valid
    fills, spans = [], []
    for a in range(dim):
        n = shape[a]
        pos = np.arange(n).reshape([-1 if b == a else 1 for b in range(dim)])
        pos = np.broadcast_to(pos, shape)
        left = np.where(ok, pos, -1)
        left = np.maximum.accumulate(left, axis=a)             # nearest valid at or before
        right = np.where(ok, pos, n)
        right = np.flip(np.minimum.accumulate(np.flip(right, axis=a), axis=a), axis=a)
        both = (left >= 0) & (right < n) & ~ok
        li = np.clip(left, 0, n - 1)
        ri = np.clip(right, 0, n - 1)
        vl = np.take_along_axis(V, li[..., None], axis=a) if False else np.take_along_axis(
            V, np.expand_dims(li, -1).repeat(k, -1), axis=a)
        vr = np.take_along_axis(V, np.expand_dims(ri, -1).repeat(k, -1), axis=a)
        span = np.where(both, right - left, 1).astype(np.float64)
        wr = np.where(both, (pos - left) / span, 0.0)
        fill = (1.0 - wr)[..., None] * np.nan_to_num(vl) + wr[..., None] * np.nan_to_num(vr)
        fills.append(fill[idx])
        spans.append(np.where(both, right - left, np.iinfo(np.int64).max)[idx])
    # Eq. 1 along the axis with the shortest valid bracket (the most local
    # linear interpolant); ties are averaged
    spans = np.stack(spans, 1)
    best = spans.min(axis=1)
    use = (spans == best[:, None]) & (best[:, None] < np.iinfo(np.int64).max)
    cntv = use.sum(axis=1)
    res = sum(np.where(use[:, a:a + 1], fills[a], 0.0) for a in range(dim)) / np.maximum(cntv, 1)[:, None]
    out = np.full(values.shape, np.nan)
    got = cntv > 0
    out[got] = res[got]
    filled = got & hole
    return out, filled


def agreement(grid, g_seeds, start, bto_end, bto_status, comm_end, comm_status, stride,
              method: str = "delaunay", recon=None):
    """BTO-vs-comm flow-map agreement for one interval (§4.3):
    over seeds valid in the comm flow map, b = BTO end if valid, else its
    reconstruction (Delaunay + barycentric, or GridFill, Eq. 2);
    L = Eq. 5, accuracy = Eq. 6.  Seeds that cannot be reconstructed (outside
    the hull / no bounding pair) are excluded and counted.  `recon`
    = (values [n, dim], filled mask [n]) supplies a reconstruction computed
    elsewhere (e.g. the CUDA GridFill) instead of computing one here."""
    comm_ok = np.asarray(comm_status) == 0
    bto_ok = np.asarray(bto_status) == 0
    hole = comm_ok & ~bto_ok
    if recon is not None:
        recon, inside = recon
        inside = np.asarray(inside, dtype=bool) & hole
    elif method == "gridfill":
        lat = np.asarray(g_seeds)[:, :grid.dim] // stride
        recon, inside = grid_fill(lat, bto_end, bto_ok, hole)
    else:
        recon, inside = reconstruct_holes(g_seeds, start, bto_end, bto_ok, hole, stride)
    b = np.where(bto_ok[:, None], bto_end, recon)
    use = comm_ok & (bto_ok | inside)
    diff = np.linalg.norm(b[use] - comm_end[use], axis=1)
    L = float(diff.mean()) if diff.size else 0.0
    C = cell_side(grid)
    return dict(L=L, max_l2=float(diff.max()) if diff.size else 0.0,
                accuracy=accuracy_pct(L, C), C=C, compared=int(use.sum()),
                holes=int(hole.sum()), excluded=int((hole & ~inside).sum()),
                discarded=int((~bto_ok).sum()), seeded=int(bto_ok.size))
