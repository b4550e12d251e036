"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Pathline stitching from the basis flows of successive intervals (SURVEY.md
§8(f)2).  Paper: "a trajectory can be stitched together by using basis flows
of successive nonoverlapping intervals" (§3.2). To compute a new
particle trajectory, a particle identifies a neighbourhood (convex hull) of
basis flows and uses barycentric coordinate interpolation of their end
positions. SPEC.md:332-340 states the operation.

Reading R16: the seeds of every interval sit on the same uniform
lattice. Every lattice cube has cospherical corners, so its Delaunay
triangulation is not unique. Ties are broken by the fixed Kuhn (Freudenthal)
template, as in SPEC.md:359's fixed simplex template. In the cube at lattice
index i with local coordinates f in [0,1]^d, sorted descending as
f_(1) >= ... >= f_(d) along axes pi_1..pi_d, the simplex has vertices
v_0 = i, v_j = v_{j-1} + e_{pi_j}. The barycentric weights are
w_0 = 1 - f_(1), w_j = f_(j) - f_(j+1), w_d = f_(d). The template is
conforming, so the interpolant is continuous across cubes and simplices.

Per interval k and query x:
  * u = (x - origin) / spacing.
  * Outside the lattice hull (some u_a < 0 or u_a > dims_a - 1, or not a
    number): the pathline is truncated (status OUT_OF_HULL) at its last
    sample. SPEC.md:358: no clamping.
  * Otherwise cube i = min(floor(u), dims - 2) and f = u - i.
  * If a vertex with weight > 0 has an invalid basis flow: status
    INVALID_FLOW, truncated. Fill the holes first (GridFill) to avoid this.
  * x <- sum_j w_j end_k[v_j].  The sample is appended.
"""
from __future__ import annotations

from typing import Optional, Sequence, Tuple

import numpy as np

COMPLETE, OUT_OF_HULL, INVALID_FLOW = 0, 1, 2


def kuhn_weights(f: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """f [m, d] in [0,1]^d -> (vertex offsets [m, d+1, d] (0/1), weights [m, d+1])."""
    m, d = f.shape
    order = np.argsort(-f, axis=1, kind="stable")          # pi_1..pi_d
    fs = np.take_along_axis(f, order, axis=1)             # f_(1) >= ... >= f_(d)
    w = np.empty((m, d + 1))
    w[:, 0] = 1.0 - fs[:, 0]
    for j in range(1, d):
        w[:, j] = fs[:, j - 1] - fs[:, j]
    w[:, d] = fs[:, d - 1]
    off = np.zeros((m, d + 1, d), dtype=np.int64)
    for j in range(1, d + 1):
        off[:, j] = off[:, j - 1]
        off[np.arange(m), j, order[:, j - 1]] = 1
    return off, w


def stitch(ends: np.ndarray, valid: Optional[np.ndarray], dims: Sequence[int], origin: Sequence[float],
           spacing: Sequence[float], starts: np.ndarray):
    """ends [K, n, d] end positions of K successive intervals on the same dense
    lattice (x fastest, n = prod(dims)); valid [K, n] bool or None (all valid);
    starts [m, d].  Returns (path [m, K+1, d] with NaN after truncation,
    status [m] u8, samples [m] = number of valid path points, min_hull [m] =
    the smallest distance, in lattice units, of any visited position to the
    hull faces)."""
    ends = np.asarray(ends, dtype=np.float64)
    K, n, d = ends.shape
    dims = np.asarray(dims, dtype=np.int64)
    origin = np.asarray(origin, dtype=np.float64)[:d]
    spacing = np.asarray(spacing, dtype=np.float64)[:d]
    x = np.asarray(starts, dtype=np.float64).copy()
    m = x.shape[0]
    path = np.full((m, K + 1, d), np.nan)
    path[:, 0] = x
    status = np.zeros(m, dtype=np.uint8)
    alive = np.ones(m, dtype=bool)
    samples = np.ones(m, dtype=np.int64)
    min_hull = np.full(m, np.inf)
    stride = np.concatenate([[1], np.cumprod(dims[:-1])])
    for k in range(K):
        u = (x - origin) / spacing
        dist = np.minimum(u, (dims - 1) - u).min(axis=1)
        min_hull = np.where(alive, np.minimum(min_hull, np.abs(dist)), min_hull)
        out = alive & ~((u >= 0) & (u <= dims - 1)).all(axis=1)      # a NaN position is outside too
        status[out] = OUT_OF_HULL
        alive &= ~out
        idx = np.nonzero(alive)[0]
        if idx.size == 0:
            break
        uu = u[idx]
        i = np.minimum(np.floor(uu).astype(np.int64), dims - 2)
        f = uu - i
        off, w = kuhn_weights(f)
        vert = ((i[:, None, :] + off) * stride).sum(axis=2)        # [m', d+1] flat node ids
        if valid is not None:
            bad = ((w > 0) & ~np.asarray(valid[k], dtype=bool)[vert]).any(axis=1)
            status[idx[bad]] = INVALID_FLOW
            alive[idx[bad]] = False
            keep = ~bad
            idx, vert, w = idx[keep], vert[keep], w[keep]
        xn = np.einsum("mj,mjc->mc", w, ends[k][vert])
        x[idx] = xn
        path[idx, k + 1] = xn
        samples[idx] += 1
    return path, status, samples, min_hull
