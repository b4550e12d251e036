"""Synthetic analytic velocity fields and the five benchmark configurations.

Fields are evaluated at grid nodes in fp64 and rounded ONCE to fp32; the oracle
and the CUDA path consume the identical fp32 arrays.  The
formulas are inputs, not the method: no RK4 / interpolation lives here.

Configurations (BASELINE.json "configs"):
  C1  2D double gyre 64x32, 1 block, stride 1, 100 cycles, interval 20
  C2  ABC 128^3, 8 blocks (2x2x2), stride 1, interval 25
  C3  CloverLeaf3D-shaped vortical field, 256^3 per GPU, stride 2, interval 50
  C4  Nyx-like turbulence, 512^3 over 8 GPUs, stride 4, intervals 10/50/100
  C5  ABC weak scaling, 128^3 per GPU, stride 1, 500 cycles, interval 25
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, Optional, Sequence, Tuple

import numpy as np

from .blocks import Grid, layout_for

TWO_PI = 2.0 * math.pi


@dataclasses.dataclass(frozen=True)
class FieldSpec:
    kind: str                 # "double_gyre" | "abc" | "clover" | "nyx" | "uniform" | "rotation" | "affine"
    params: Tuple = ()        # kind-specific constants
    period: float = 1.0       # T in time modulations


# ----------------------------------------------------------------------------
# analytic formulas (fp64), vectorised over node coordinate arrays
# ----------------------------------------------------------------------------

def _xp(a):
    if isinstance(a, np.ndarray):
        return np
    import torch
    return torch


def _eval(spec: FieldSpec, X, Y, Z, t: float):
    xp = _xp(X)
    if spec.kind == "double_gyre":
        # SPEC.md:62 / SURVEY.md §8(d) C1: psi = A sin(pi f) sin(pi y),
        # f = a x^2 + b x, a = eps sin wt, b = 1 - 2 eps sin wt.
        A, eps, om = 0.1, 0.25, TWO_PI / 10.0
        a = eps * math.sin(om * t)
        b = 1.0 - 2.0 * eps * math.sin(om * t)
        f = a * X * X + b * X
        u = -math.pi * A * xp.sin(math.pi * f) * xp.cos(math.pi * Y)
        v = math.pi * A * xp.cos(math.pi * f) * xp.sin(math.pi * Y) * (2.0 * a * X + b)
        return (u, v)
    if spec.kind == "abc":
        # SURVEY.md §8(c) reading 7: A(t) = sqrt3 (1 + 1/2 sin(2 pi t / T)).
        A = math.sqrt(3.0) * (1.0 + 0.5 * math.sin(TWO_PI * t / spec.period))
        B, C = math.sqrt(2.0), 1.0
        return (A * xp.sin(Z) + C * xp.cos(Y),
                B * xp.sin(X) + A * xp.cos(Z),
                C * xp.sin(Y) + B * xp.cos(X))
    if spec.kind == "clover":
        # U0[(1 + 1/2 sin 2pi t/T) TG(x) + 1/2 rhat exp(-((r-2-0.5t)/0.75)^2)],
        # kappa = 2pi/5, r from the corner (0,0,0).  U0 = 2/3 bounds |v| <= 1 at t = 0.
        kap = TWO_PI / 5.0
        U0 = 2.0 / 3.0
        m = 1.0 + 0.5 * math.sin(TWO_PI * t / spec.period)
        sx, cx = xp.sin(kap * X), xp.cos(kap * X)
        sy, cy = xp.sin(kap * Y), xp.cos(kap * Y)
        cz = xp.cos(kap * Z)
        r = xp.sqrt(X * X + Y * Y + Z * Z)
        rs = xp.where(r > 0, r, xp.ones_like(r)) if xp is np else xp.where(r > 0, r, xp.ones_like(r))
        pulse = 0.5 * xp.exp(-((r - 2.0 - 0.5 * t) / 0.75) ** 2) / rs
        return (U0 * (m * sx * cy * cz + pulse * X),
                U0 * (-m * cx * sy * cz + pulse * Y),
                U0 * (pulse * Z))
    if spec.kind == "nyx":
        # g(t) sum_m A_m p_m cos(k_m.x + phi_m + w_m t), p_m ⟂ k_m,
        # A_m ∝ |k|^(-5/6), normalised so max|v| = 1 on a 48^3 sample at g = 1;
        # g = 0.5 + 0.5 t / T.
        K, P, Am, phi, om = spec.params
        g = 0.5 + 0.5 * t / spec.period
        u = xp.zeros_like(X); v = xp.zeros_like(X); w = xp.zeros_like(X)
        for m in range(len(Am)):
            ph = xp.cos(K[m][0] * X + K[m][1] * Y + K[m][2] * Z + (phi[m] + om[m] * t))
            u = u + (g * Am[m] * P[m][0]) * ph
            v = v + (g * Am[m] * P[m][1]) * ph
            w = w + (g * Am[m] * P[m][2]) * ph
        return (u, v, w)
    if spec.kind == "uniform":
        return tuple(xp.full_like(X, c) for c in spec.params)
    if spec.kind == "rotation":
        # solid-body rotation about the axis through (cx, cy) parallel to z, rate w
        w, cx, cy = spec.params
        out = (-w * (Y - cy), w * (X - cx))
        return out + ((xp.zeros_like(X),) if Z is not None else ())
    if spec.kind == "affine":
        # v = (A0 + t A1) x + b  (A0, A1: dim x dim, b: dim); time-linear affine
        A0, A1, b = spec.params
        coords = (X, Y, Z)[:len(b)]
        out = []
        for i in range(len(b)):
            acc = xp.full_like(X, float(b[i]))
            for j in range(len(b)):
                acc = acc + (A0[i][j] + t * A1[i][j]) * coords[j]
            out.append(acc)
        return tuple(out)
    raise ValueError(f"unknown field kind {spec.kind}")


def field_at_nodes(spec: FieldSpec, grid: Grid, t: float, lo=None, hi=None,
                   device=None, backend: str = "numpy"):
    """Velocity at nodes n in [lo, hi) (default: all) at time t.

    Returns an array shaped [nz, ny, nx, dim], fp32, AoS per node, x fastest.
    Node coordinates are x_a(n) = o_a + n_a * h_a evaluated in fp64.  Nodes
    outside [0, N) evaluate the formula anyway (callers only use them as
    never-read ghost padding)."""
    lo = tuple(lo) if lo is not None else (0, 0, 0)
    hi = tuple(hi) if hi is not None else tuple(grid.nodes)
    if backend == "numpy":
        xp = np
        ax = [grid.origin[a] + np.arange(lo[a], hi[a], dtype=np.float64) * grid.spacing[a]
              for a in range(3)]
        Z, Y, X = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    else:
        import torch
        ax = [grid.origin[a] + torch.arange(lo[a], hi[a], dtype=torch.float64, device=device)
              * grid.spacing[a] for a in range(3)]
        Z, Y, X = torch.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    comps = _eval(spec, X, Y, Z if grid.dim == 3 else None, float(t))
    if backend == "numpy":
        out = np.stack([np.asarray(c, dtype=np.float64) for c in comps], axis=-1)
        return out.astype(np.float32)
    import torch
    return torch.stack([c.to(torch.float64) for c in comps], dim=-1).to(torch.float32)


# ----------------------------------------------------------------------------
# configurations
# ----------------------------------------------------------------------------

def _nyx_modes(seed: int = 2004_02003, n: int = 64):
    rng = np.random.default_rng(seed)
    K, P, A, phi = [], [], [], []
    for _ in range(n):
        kmag = TWO_PI * rng.uniform(1.0, 16.0)
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        k = kmag * d
        r = rng.normal(size=3); r -= r.dot(d) * d; r /= np.linalg.norm(r)   # p ⟂ k
        K.append(tuple(float(c) for c in k)); P.append(tuple(float(c) for c in r))
        A.append(kmag ** (-5.0 / 6.0)); phi.append(float(rng.uniform(0.0, TWO_PI)))
    A = np.asarray(A); A = A / A.sum()
    # normalise so that max |v| = 1 on a 48^3 lattice of the unit box at g = 1, t = 0
    ax = np.linspace(0.0, 1.0, 48)
    Z, Y, X = np.meshgrid(ax, ax, ax, indexing="ij")
    U = np.zeros(X.shape + (3,))
    for m in range(n):
        ph = np.cos(K[m][0] * X + K[m][1] * Y + K[m][2] * Z + phi[m])
        U += A[m] * np.asarray(P[m]) * ph[..., None]
    A = A / float(np.linalg.norm(U, axis=-1).max())
    urms = math.sqrt(float((A * A).sum()) / 2.0)
    om = [float(np.linalg.norm(k)) * urms for k in K]
    return (tuple(K), tuple(P), tuple(float(a) for a in A), tuple(phi), tuple(om))


def make_config(name: str, nranks: int = 1, scale: Optional[int] = None,
                interval: Optional[int] = None, cycles: Optional[int] = None) -> Dict:
    """Configuration dict for C1..C5.  ``scale`` shrinks the per-block node
    count (parity-test sizes); ``nranks`` picks the weak-scaling layout for
    C3/C5 (one block per GPU)."""
    name = name.upper()
    if name == "C1":
        n = (64, 32, 1)
        grid = Grid(2, n, (0.0, 0.0, 0.0), (2.0 / 63, 1.0 / 31, 1.0))
        spec = FieldSpec("double_gyre")
        cfg = dict(grid=grid, layout=(1, 1, 1), field=spec, dt=0.1, cycles=100,
                   interval=20, stride=1, cfl=None)
    elif name == "C2":
        nn = scale or 128
        h = TWO_PI / (nn - 1)
        grid = Grid(3, (nn, nn, nn), (0.0, 0.0, 0.0), (h, h, h))
        dt = 1.25e-3 * (128 - 1) / (nn - 1)
        spec = FieldSpec("abc", period=1000 * dt)
        cfg = dict(grid=grid, layout=(2, 2, 2), field=spec, dt=dt, cycles=250,
                   interval=25, stride=1)
    elif name == "C3":
        per = scale or 256
        lay = layout_for(nranks)
        h = 10.0 / 255
        nodes = tuple(per * lay[a] for a in range(3))
        grid = Grid(3, nodes, (0.0, 0.0, 0.0), (h, h, h))
        dt = 0.25 * h
        spec = FieldSpec("clover", period=500 * dt)
        cfg = dict(grid=grid, layout=lay, field=spec, dt=dt, cycles=500, interval=50, stride=2)
    elif name == "C4":
        nn = scale or 512
        h = 1.0 / (nn - 1)
        grid = Grid(3, (nn, nn, nn), (0.0, 0.0, 0.0), (h, h, h))
        dt = 0.25 * h
        spec = FieldSpec("nyx", params=_nyx_modes(), period=500 * dt)
        cfg = dict(grid=grid, layout=(2, 2, 2), field=spec, dt=dt, cycles=500, interval=10,
                   stride=4 if scale is None else max(1, min(4, nn // 32)))
    elif name == "C5":
        per = scale or 128
        lay = layout_for(nranks)
        h = TWO_PI / 128
        nodes = tuple(per * lay[a] for a in range(3))
        grid = Grid(3, nodes, (0.0, 0.0, 0.0), (h, h, h))
        dt = 1.25e-3
        spec = FieldSpec("abc", period=1000 * dt)
        cfg = dict(grid=grid, layout=lay, field=spec, dt=dt, cycles=500, interval=25, stride=1)
    else:
        raise ValueError(f"unknown config {name}")
    if interval is not None:
        cfg["interval"] = interval
    if cycles is not None:
        cfg["cycles"] = cycles
    cfg["name"] = name
    return cfg


CONFIGS = ("C1", "C2", "C3", "C4", "C5")


def config_names():
    return CONFIGS
