"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 CPU reference for the in situ Lagrangian
flow-map extraction hot path of arXiv 2004.02003.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2004_02003_b200``) never imports it and shares no code with it;
both sides take their synthetic inputs from ``lag_inputs`` only.

Layout:
  lag_oracle.c   per-particle RK4 cycle, multilinear interpolation, boundary
                 classification (C, fp64, -ffp-contract=off, OpenMP over particles)
  __init__.py    build + ctypes wrapper, seeding, interval driver,
                 flow-map assembly
  metrics.py     Eq. 5 / Eq. 6 / max-L2 folds, post hoc
                 reconstruction

Citations: P:nnn = /root/reference/PAPER.md line nnn; S:nnn = SPEC.md line.
Pins: tests/test_oracle_pins.py.  Every function here is pinned; none is
"parity unpinned" except the agreement *values* on our synthetic fields, which
the paper cannot fix.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Iterable, Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lag_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

VALID, TERM_BOUNDARY, EXIT_DOMAIN = 0, 1, 2
BTO, COMM = 0, 1


def build(force: bool = False) -> str:
    """Compile lag_oracle.c -> oracle/liboracle.so (gcc, fp64, no contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-std=c11", "-Wall", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Grid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("N", ctypes.c_int64 * 3), ("o", ctypes.c_double * 3),
                ("h", ctypes.c_double * 3)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        _lib.orc_tri.argtypes = [P(_Grid), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib.orc_cycle.argtypes = [P(_Grid), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                   ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib.orc_rk4_free.argtypes = [P(_Grid), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                      ctypes.c_int64, ctypes.c_void_p]
    return _lib


def _cgrid(grid) -> _Grid:
    g = _Grid()
    g.dim = grid.dim
    for a in range(3):
        g.N[a] = int(grid.nodes[a])
        g.o[a] = float(grid.origin[a])
        g.h[a] = float(grid.spacing[a])
    return g


def _f32(V) -> np.ndarray:
    V = np.ascontiguousarray(np.asarray(V, dtype=np.float32))
    return V


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# primitives
# ---------------------------------------------------------------------------

def tri(grid, V, q) -> np.ndarray:
    """Multilinear interpolation of the global node array V ([Nz,Ny,Nx,dim]
    fp32) at physical points q [m, dim] (fp64).  lag_oracle.c:orc_tri."""
    lib = _load()
    V = _f32(V)
    q = np.ascontiguousarray(np.asarray(q, dtype=np.float64).reshape(-1, grid.dim))
    out = np.zeros_like(q)
    g = _cgrid(grid)
    for m in range(q.shape[0]):
        lib.orc_tri(ctypes.byref(g), _ptr(V), ctypes.c_void_p(q.ctypes.data + m * q.strides[0]),
                    ctypes.c_void_p(out.ctypes.data + m * out.strides[0]))
    return out


def rk4_free(grid, V0, V1, dt, pos) -> np.ndarray:
    """One RK4 step of the time-lerped multilinear field, no boundary logic."""
    lib = _load()
    pos = np.ascontiguousarray(np.array(pos, dtype=np.float64).reshape(-1, grid.dim))
    V0, V1 = _f32(V0), _f32(V1)
    lib.orc_rk4_free(ctypes.byref(_cgrid(grid)), _ptr(V0), _ptr(V1), float(dt),
                     pos.shape[0], _ptr(pos))
    return pos


def seeds(grid, lo, hi, stride: int) -> np.ndarray:
    """Seed lattice of a block (§2.3: "particles are seeded along a
    uniform grid"; 1:X data reduction, X = stride^dim).  Reading R4: nodes of
    the global lattice g_a = 0 mod stride with lo_a <= g_a < hi_a, x fastest.
    Returns integer node coordinates [n, 3] (unused axis = 0)."""
    axes = []
    for a in range(3):
        if a >= grid.dim:
            axes.append(np.zeros(1, dtype=np.int64))
            continue
        first = -(-lo[a] // stride) * stride
        axes.append(np.arange(first, hi[a], stride, dtype=np.int64))
    gz, gy, gx = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
    return np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)


def node_position(grid, g: np.ndarray) -> np.ndarray:
    """x(n) = o + n h (fp64), [n, dim]."""
    g = np.asarray(g)
    return np.stack([grid.origin[a] + g[:, a].astype(np.float64) * grid.spacing[a]
                     for a in range(grid.dim)], axis=1)


class Interval:
    """One extraction interval of one block (seed, advect for
    `interval` cycles, save end positions).  mode=COMM integrates on the whole
    domain (block := Omega), which is what the exchange baseline computes
    (reading R7)."""

    def __init__(self, grid, lo, hi, stride: int, mode: int = BTO, g_seeds=None,
                 faces=None):
        self.grid = grid
        self.mode = mode
        self.lo = np.array(lo, dtype=np.int64)
        self.hi = np.array(hi, dtype=np.int64)
        if mode == COMM:
            self.blo = np.zeros(3, dtype=np.int64)
            self.bhi = np.array(grid.nodes, dtype=np.int64)
        else:
            self.blo, self.bhi = self.lo, self.hi
        self.g = seeds(grid, lo, hi, stride) if g_seeds is None else np.asarray(g_seeds)
        self.start = node_position(grid, self.g)
        self.pos = self.start.copy()
        n = self.g.shape[0]
        self.status = np.zeros(n, dtype=np.uint8)
        self.term_cycle = np.full(n, -1, dtype=np.int32)
        self.cycle_index = 0
        # excuse-band instrumentation: faces = (lo, hi) of the block whose
        # boundary decides the flags (defaults to this block)
        flo, fhi = faces if faces is not None else (lo, hi)
        self.flo = np.array(flo, dtype=np.int64)
        self.fhi = np.array(fhi, dtype=np.int64)
        self.min_face = np.full(n, np.inf)

    @property
    def n(self) -> int:
        return self.g.shape[0]

    def cycle(self, V0, V1, dt: float, touched: Optional[np.ndarray] = None):
        lib = _load()
        V0, V1 = _f32(V0), _f32(V1)
        lib.orc_cycle(ctypes.byref(_cgrid(self.grid)), _ptr(self.blo), _ptr(self.bhi),
                      int(self.mode), _ptr(V0), _ptr(V1), float(dt), self.n,
                      _ptr(self.pos), _ptr(self.status), _ptr(self.term_cycle),
                      int(self.cycle_index),
                      _ptr(touched) if touched is not None else None,
                      _ptr(self.flo), _ptr(self.fhi), _ptr(self.min_face))
        self.cycle_index += 1

    def active(self) -> int:
        return int((self.status == VALID).sum())


def run_interval(grid, lo, hi, stride, slices: Iterable, dt: float, mode: int = BTO,
                 g_seeds=None, faces=None) -> Interval:
    """Drive one interval given an iterable of consecutive global slices
    V_c, V_{c+1}, ... (len = cycles + 1)."""
    it = Interval(grid, lo, hi, stride, mode, g_seeds, faces)
    prev = None
    for V in slices:
        if prev is not None:
            it.cycle(prev, V, dt)
        prev = V
    return it
