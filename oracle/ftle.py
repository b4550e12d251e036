"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

FTLE from an extracted flow map.  The paper names FTLE
fields computed post hoc from the basis flows as its qualitative output
(§4.3, "FTLE scalar fields generated post hoc using basis flows");
SPEC.md:460-468 states the operation:

  * flow-map gradient dF/dX by central differences on the seed lattice,
    one-sided at the lattice faces;
  * right Cauchy-Green tensor C = (dF/dX)^T (dF/dX);
  * FTLE = ln(sqrt(lambda_max(C))) / |T|;
  * lambda_max <= 0 (degenerate tensor) gives 0, and is counted.

Written as that definition with library primitives: numpy.gradient (second
order central differences inside, first order one-sided at the faces, i.e.
edge_order=1) and numpy.linalg.eigvalsh.  No blocking or reordering.
"""
from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np


def ftle(ends: np.ndarray, dims: Sequence[int], spacing: Sequence[float], T: float) -> Tuple[np.ndarray, int]:
    """ends [n, dim] end positions on a dense lattice, x fastest
    (n = prod(dims)); spacing = seed spacing per axis (stride * h);
    T = integration time.  Returns (FTLE [n], number of degenerate tensors)."""
    dim = len(dims)
    if T == 0:
        raise ValueError("T must be nonzero")
    ends = np.asarray(ends, dtype=np.float64)
    shape = tuple(int(d) for d in dims[::-1])                 # numpy order: slowest axis first
    F = [ends[:, c].reshape(shape) for c in range(dim)]
    J = np.zeros(shape + (dim, dim))                          # J[..., c, a] = dF_c / dX_a
    for a in range(dim):
        npax = dim - 1 - a                                    # lattice axis a in numpy order
        if shape[npax] < 2:
            continue                                          # no extent: derivative undefined, left 0
        for c in range(dim):
            J[..., c, a] = np.gradient(F[c], float(spacing[a]), axis=npax, edge_order=1)
    C = np.einsum("...ca,...cb->...ab", J, J).reshape(-1, dim, dim)
    fin = np.isfinite(C).all(axis=(1, 2))                     # non-finite ends propagate as NaN
    lam = np.full(C.shape[0], np.nan)
    lam[fin] = np.linalg.eigvalsh(C[fin])[:, -1]
    bad = fin & ~(lam > 0)
    out = np.full(C.shape[0], np.nan)
    ok = fin & ~bad
    out[ok] = np.log(np.sqrt(lam[ok])) / abs(T)
    out[bad] = 0.0
    return out, int(bad.sum())
