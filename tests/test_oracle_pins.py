"""Pins of the fp64 oracle against what the paper and mathematics fix
(closed forms, brute force, invariants, the paper's printed values).

Nothing here compares the oracle with itself: each expected value is derived
independently of oracle/lag_oracle.c (tent-function sums, matrix power series,
scipy ODE integration, closed-form crossing schedules, the paper's tables).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import metrics
import lag_inputs as L

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def grid3(n, o=(0.0, 0.0, 0.0), h=(1.0, 1.0, 1.0)):
    return L.Grid(3, tuple(n), tuple(o), tuple(h))


def nodes_xyz(grid):
    ax = [grid.origin[a] + np.arange(grid.nodes[a]) * grid.spacing[a] for a in range(3)]
    Z, Y, X = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return X, Y, Z


# ---------------------------------------------------------------- Tri (pins 1, 2)

def tent_sum(grid, V, q):
    """Brute force: sum over ALL nodes n of prod_a max(0, 1 - |u_a - n_a|) V[n].
    Independent of floor / clamp logic (a closed upper face gets weight 1 on
    the last node)."""
    d = grid.dim
    u = [(q[a] - grid.origin[a]) / grid.spacing[a] for a in range(d)]
    out = np.zeros(d)
    for idx in np.ndindex(*[grid.nodes[a] for a in reversed(range(3))]):
        n = idx[::-1]
        w = 1.0
        for a in range(d):
            w *= max(0.0, 1.0 - abs(u[a] - n[a]))
        if w:
            out += w * V[idx].astype(np.float64)
    return out


@pytest.mark.parametrize("dims", [(3, 3, 3), (4, 3, 2), (2, 2, 2)])
def test_tri_brute_force_3d(dims):
    rng = np.random.default_rng(7)
    g = grid3(dims, o=(-0.5, 1.0, 2.0), h=(0.7, 1.3, 0.4))
    V = rng.normal(size=(dims[2], dims[1], dims[0], 3)).astype(np.float32)
    ext = [(dims[a] - 1) * g.spacing[a] for a in range(3)]
    pts = [g.origin[a] + rng.uniform(0, 1, 40) * ext[a] for a in range(3)]
    q = np.stack(pts, axis=1)
    # closed upper faces and corners exactly
    q = np.vstack([q, [g.origin[a] + ext[a] for a in range(3)],
                   [g.origin[0], g.origin[1] + ext[1], g.origin[2] + 0.3 * ext[2]]])
    got = oracle.tri(g, V, q)
    for m in range(q.shape[0]):
        np.testing.assert_allclose(got[m], tent_sum(g, V, q[m]), rtol=0, atol=1e-12)


def test_tri_brute_force_2d():
    rng = np.random.default_rng(8)
    g = L.Grid(2, (3, 2, 1), (0.25, -1.0, 0.0), (0.5, 2.0, 1.0))
    V = rng.normal(size=(1, 2, 3, 2)).astype(np.float32)
    q = np.stack([0.25 + rng.uniform(0, 1, 30) * 1.0, -1.0 + rng.uniform(0, 1, 30) * 2.0], 1)
    q = np.vstack([q, [1.25, 1.0]])
    got = oracle.tri(g, V, q)
    for m in range(q.shape[0]):
        np.testing.assert_allclose(got[m], tent_sum(g, V, q[m]), atol=1e-12)


def test_tri_returns_node_values_and_is_exact_on_affine():
    g = grid3((5, 4, 6), o=(-1.0, 0.0, 0.5), h=(0.5, 0.25, 1.0))
    X, Y, Z = nodes_xyz(g)
    # integer-valued affine field: exact in fp32
    A = np.array([[2, -1, 3], [0, 4, -2], [1, 1, 1]], dtype=np.float64)
    b = np.array([1.0, -3.0, 0.5])
    V = np.stack([A[i, 0] * X + A[i, 1] * Y + A[i, 2] * Z + b[i] for i in range(3)], -1)
    assert np.array_equal(V.astype(np.float32).astype(np.float64), V)
    V32 = V.astype(np.float32)
    # nodes
    idx = [(0, 0, 0), (4, 3, 5), (2, 1, 3)]
    q = np.array([[g.origin[a] + i[a] * g.spacing[a] for a in range(3)] for i in idx])
    got = oracle.tri(g, V32, q)
    for m, i in enumerate(idx):
        np.testing.assert_array_equal(got[m], V[i[2], i[1], i[0]])
    # arbitrary points: exact affine reproduction
    rng = np.random.default_rng(3)
    q = np.stack([g.origin[a] + rng.uniform(0, (g.nodes[a] - 1) * g.spacing[a], 50)
                  for a in range(3)], 1)
    np.testing.assert_allclose(oracle.tri(g, V32, q), q @ A.T + b, atol=1e-12)


# ---------------------------------------------------------------- RK4 closed forms

def test_rk4_uniform_field_exact():
    """x_n = x0 + n dt v exactly."""
    g = grid3((9, 9, 9), h=(1.0, 1.0, 1.0))
    v = (0.25, -0.5, 0.125)
    V = L.field_at_nodes(L.FieldSpec("uniform", v), g, 0.0)
    x = np.array([[3.0, 5.0, 2.0], [4.5, 4.25, 6.0]])
    for n in range(1, 6):
        x = oracle.rk4_free(g, V, V, 0.5, x)
        np.testing.assert_array_equal(x, np.array([[3.0, 5.0, 2.0], [4.5, 4.25, 6.0]])
                                      + n * 0.5 * np.array(v))


def test_rk4_zero_field_no_motion():
    g = grid3((4, 4, 4))
    V = np.zeros((4, 4, 4, 3), np.float32)
    x0 = np.array([[0.3, 0.3, 0.3]])
    np.testing.assert_array_equal(oracle.rk4_free(g, V, V, 0.1, x0), x0)


def test_rk4_solid_body_rotation_circle():
    """v = w (-(y-cy), x-cx) is linear in space (Tri exact) and steady.
    One RK4 step multiplies z = (x-cx) + i(y-cy) by R(i theta), R(z) = sum_{k<=4} z^k/k!,
    theta = w dt; |R(i theta)|^2 = 1 - theta^6/72 + theta^8/576 (the "circle")."""
    g = L.Grid(3, (17, 17, 3), (-4.0, -4.0, 0.0), (0.5, 0.5, 0.5))
    V = L.field_at_nodes(L.FieldSpec("rotation", (1.0, 0.0, 0.0)), g, 0.0)
    X, Y, _ = nodes_xyz(g)
    assert np.array_equal(V[..., 0], (-Y).astype(np.float32))
    dt = 0.1
    th = 1.0 * dt
    R = sum((1j * th) ** k / math.factorial(k) for k in range(5))
    z0 = 1.5 + 0.5j
    x = np.array([[z0.real, z0.imag, 0.5]])
    for n in range(1, 21):
        x = oracle.rk4_free(g, V, V, dt, x)
        zn = z0 * R ** n
        assert abs(x[0, 0] - zn.real) < 1e-13 and abs(x[0, 1] - zn.imag) < 1e-13
        assert x[0, 2] == 0.5
        r2 = x[0, 0] ** 2 + x[0, 1] ** 2
        assert abs(r2 - abs(z0) ** 2 * (1 - th ** 6 / 72 + th ** 8 / 576) ** n) < 1e-13


def test_rk4_affine_one_step_power_series():
    """v = A x + b (steady): one RK4 step = P(M) x + dt (I + M/2 + M^2/6 + M^3/24) b,
    M = dt A, P(M) = I + M + M^2/2 + M^3/6 + M^4/24."""
    g = grid3((9, 9, 9), o=(-2.0, -2.0, -2.0), h=(0.5, 0.5, 0.5))
    A = np.array([[0, -1, 0.5], [1, 0, -0.25], [0.25, 0.5, -1]])
    b = np.array([0.5, -0.25, 1.0])
    spec = L.FieldSpec("affine", (A.tolist(), np.zeros((3, 3)).tolist(), b.tolist()))
    V = L.field_at_nodes(spec, g, 0.0)
    X, Y, Z = nodes_xyz(g)
    assert np.array_equal(V[..., 0].astype(np.float64), A[0, 0] * X + A[0, 1] * Y + A[0, 2] * Z + b[0])
    dt = 0.125
    M = dt * A
    I = np.eye(3)
    P = I + M + M @ M / 2 + M @ M @ M / 6 + M @ M @ M @ M / 24
    Qb = I + M / 2 + M @ M / 6 + M @ M @ M / 24
    rng = np.random.default_rng(1)
    x0 = rng.uniform(-1, 1, (10, 3))
    got = oracle.rk4_free(g, V, V, dt, x0)
    np.testing.assert_allclose(got, x0 @ P.T + dt * (Qb @ b), atol=1e-14)


def test_rk4_time_lerp_fourth_order():
    """v = (A0 + t A1) x is reproduced exactly by the alpha-lerp of slices at t_c
    and t_c + dt; the global error at T against a tight scipy integration
    shrinks by 2^4 per dt halving (observed order in [3.5, 4.5]).
    A wrong stage time (alpha) would drop the order below 3."""
    from scipy.integrate import solve_ivp
    g = grid3((9, 9, 9), o=(-2.0, -2.0, -2.0), h=(0.5, 0.5, 0.5))
    A0 = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, -0.5]])
    A1 = np.array([[0.5, 0.0, 1.0], [0.0, -1.0, 0.0], [1.0, 0.0, 0.0]])
    spec = L.FieldSpec("affine", (A0.tolist(), A1.tolist(), [0.0, 0.0, 0.0]))
    x0 = np.array([0.5, -0.25, 0.75])
    T = 1.0
    ref = solve_ivp(lambda t, x: (A0 + t * A1) @ x, (0, T), x0, method="DOP853",
                    rtol=1e-13, atol=1e-15).y[:, -1]
    errs = []
    for n in (8, 16, 32):
        dt = T / n
        x = x0[None, :].copy()
        for c in range(n):
            V0 = L.field_at_nodes(spec, g, c * dt)
            V1 = L.field_at_nodes(spec, g, (c + 1) * dt)
            x = oracle.rk4_free(g, V0, V1, dt, x)
        errs.append(np.linalg.norm(x[0] - ref))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(3.5 <= o <= 4.5 for o in orders), (errs, orders)


def test_rk4_abc_one_step_vs_fine_euler():
    """one RK4 step on the (gridded) ABC field agrees with 1000 Euler
    sub-steps of the same interpolated field within the RK4/Euler error."""
    c = L.make_config("C2", scale=33)
    g = c["grid"]
    V = L.field_at_nodes(c["field"], g, 0.0)
    x0 = np.array([[1.0, 1.0, 1.0]])
    dt = 0.01
    rk = oracle.rk4_free(g, V, V, dt, x0)
    x = x0.copy()
    for _ in range(1000):
        x = x + (dt / 1000) * oracle.tri(g, V, x)
    assert np.abs(rk - x).max() < 1e-6


# ---------------------------------------------------------------- flags (pin 7)

def test_bto_flags_closed_form_two_blocks():
    """Two blocks split at node 8 of 17, constant v = (U,0,0), U dt / h = 1/4.
    Block 0: TERM_BOUNDARY iff x0 + I U dt >= x_f (landing exactly on the shared
    face counts, half-open rule S:231), at cycle c* = min{c : x0 + (c+1) U dt >= x_f},
    end = x0 + c* U dt.  Block 1: EXIT_DOMAIN iff x0 + I U dt > x_max (closed face)."""
    g = grid3((17, 5, 5), h=(1.0, 1.0, 1.0))
    U, dt, I = 0.5, 0.5, 7         # displacement 1/4 cell per cycle, exact in binary
    V = L.field_at_nodes(L.FieldSpec("uniform", (U, 0.0, 0.0)), g, 0.0)
    blocks = L.decompose(g, (2, 1, 1))
    xf = float(blocks[0].hi[0])
    xmax = 16.0
    for b in blocks:
        it = oracle.Interval(g, b.lo, b.hi, 1, oracle.BTO)
        for _ in range(I):
            it.cycle(V, V, dt)
        x0 = it.start[:, 0]
        for p in range(it.n):
            disp = I * U * dt
            if b.rank == 0 and x0[p] + disp >= xf:
                cstar = math.ceil((xf - x0[p]) / (U * dt)) - 1
                assert it.status[p] == oracle.TERM_BOUNDARY
                assert it.term_cycle[p] == cstar
                assert it.pos[p, 0] == x0[p] + cstar * U * dt
            elif b.rank == 1 and x0[p] + disp > xmax:
                assert it.status[p] == oracle.EXIT_DOMAIN
            else:
                assert it.status[p] == oracle.VALID
                assert it.pos[p, 0] == x0[p] + disp
    # exact tie: a particle starting 1.75 cells before the face lands on it at cycle 6
    assert (xf - 1.75) + I * U * dt == xf


def _abc_slices(c, ncyc):
    g = c["grid"]
    return [L.field_at_nodes(c["field"], g, k * c["dt"]) for k in range(ncyc + 1)]


@pytest.fixture(scope="module")
def abc_small():
    c = L.make_config("C2", scale=25)
    c["dt"] = 0.02          # CFL ~ 0.45 so a few % terminate within 12 cycles
    sl = _abc_slices(c, 12)
    return c, sl


def test_bto_vs_global_replay_and_agreement(abc_small):
    """Brute-force replay and AGREEMENT: the COMM oracle
    (decomposition-free) gives each particle's full trajectory; a BTO particle
    that stays VALID has bitwise the same end; every particle whose committed
    COMM positions leave its block at cycle c is BTO-terminated at or before c;
    accounting seeded = valid + term + exit."""
    c, sl = abc_small
    g = c["grid"]
    blocks = L.decompose(g, c["layout"])
    for b in blocks:
        bto = oracle.Interval(g, b.lo, b.hi, 1, oracle.BTO)
        com = oracle.Interval(g, b.lo, b.hi, 1, oracle.COMM)
        first_exit = np.full(bto.n, 10 ** 9)
        blo = np.array([g.origin[a] + b.lo[a] * g.spacing[a] for a in range(3)])
        bhi = np.array([g.origin[a] + b.hi[a] * g.spacing[a] for a in range(3)])
        top = np.array([g.origin[a] + (g.nodes[a] - 1) * g.spacing[a] for a in range(3)])
        for k in range(len(sl) - 1):
            bto.cycle(sl[k], sl[k + 1], c["dt"])
            com.cycle(sl[k], sl[k + 1], c["dt"])
            p = com.pos
            inside = np.all(p >= blo, 1) & np.all(np.where(np.array(b.hi) >= g.nodes[:3], p <= top, p < bhi), 1)
            newly = (~inside) & (first_exit > k) & (com.status == 0)
            first_exit[newly] = k
        ok = bto.status == oracle.VALID
        assert np.array_equal(bto.pos[ok], com.pos[ok])
        assert np.all(bto.status[first_exit < 10 ** 9] != oracle.VALID)
        assert np.all(bto.term_cycle[first_exit < 10 ** 9] <= first_exit[first_exit < 10 ** 9])
        assert ok.sum() + (bto.status == 1).sum() + (bto.status == 2).sum() == bto.n
        # terminated particles keep their pre-step position
        assert np.all(np.isfinite(bto.pos))


def test_eq4_band_never_terminated(abc_small):
    """Eq. 4: a seed farther than sum_c dt max|v| from every internal
    face cannot reach it, so it is never TERM_BOUNDARY."""
    c, sl = abc_small
    g = c["grid"]
    vmax = max(float(np.linalg.norm(V, axis=-1).max()) for V in sl)
    reach = (len(sl) - 1) * c["dt"] * vmax
    for b in L.decompose(g, c["layout"]):
        it = oracle.run_interval(g, b.lo, b.hi, 1, sl, c["dt"])
        faces = []
        for a in range(3):
            if b.lo[a] > 0:
                faces.append((a, g.origin[a] + b.lo[a] * g.spacing[a]))
            if b.hi[a] < g.nodes[a]:
                faces.append((a, g.origin[a] + b.hi[a] * g.spacing[a]))
        dist = np.min([np.abs(it.start[:, a] - x) for a, x in faces], axis=0)
        far = dist > reach * 1.0000001
        assert far.sum() > 0
        assert np.all(it.status[far] != oracle.TERM_BOUNDARY)


def test_single_rank_bto_equals_comm(abc_small):
    """R=1 equivalence: bitwise identical flow maps."""
    c, sl = abc_small
    g = c["grid"]
    a = oracle.run_interval(g, (0, 0, 0), g.nodes, 1, sl, c["dt"], oracle.BTO)
    b = oracle.run_interval(g, (0, 0, 0), g.nodes, 1, sl, c["dt"], oracle.COMM)
    assert np.array_equal(a.pos, b.pos) and np.array_equal(a.status, b.status)


def test_monotone_discard(abc_small):
    """MONOTONE DISCARD: discards after k cycles never exceed those
    after k' > k; and the COMM map only discards global exits."""
    c, sl = abc_small
    g = c["grid"]
    b = L.decompose(g, c["layout"])[0]
    it = oracle.Interval(g, b.lo, b.hi, 1, oracle.BTO)
    prev = 0
    for k in range(len(sl) - 1):
        it.cycle(sl[k], sl[k + 1], c["dt"])
        cur = int((it.status != 0).sum())
        assert cur >= prev
        prev = cur
    assert prev > 0


def test_zero_field_end_equals_seed():
    g = grid3((6, 6, 6))
    V = np.zeros((6, 6, 6, 3), np.float32)
    it = oracle.run_interval(g, (0, 0, 0), (3, 6, 6), 1, [V] * 6, 0.1)
    assert np.array_equal(it.pos, it.start) and np.all(it.status == 0)


# ---------------------------------------------------------------- seeding

def test_seed_counts_and_union():
    g = grid3((64, 64, 64))
    assert oracle.seeds(g, (0, 0, 0), (64, 64, 64), 1).shape[0] == 262144
    assert oracle.seeds(g, (0, 0, 0), (64, 64, 64), 2).shape[0] == 32 ** 3
    g2 = grid3((10, 9, 7))
    for s in (1, 2, 3):
        allg = oracle.seeds(g2, (0, 0, 0), g2.nodes, s)
        parts = np.vstack([oracle.seeds(g2, b.lo, b.hi, s) for b in L.decompose(g2, (3, 2, 2))])
        key = lambda a: set(map(tuple, a.tolist()))
        assert key(allg) == key(parts) and parts.shape[0] == allg.shape[0]


def test_decompose_remainder_rule():
    g = grid3((10, 4, 4))
    b = L.decompose(g, (3, 1, 1))
    assert [x.hi[0] - x.lo[0] for x in b] == [4, 3, 3]


# ---------------------------------------------------------------- metrics (pin 11)

def test_eq6_reproduces_paper_tables():
    """Eq. 6 with C = extent/(N-1), truncated to 0.1, reproduces 33 of the
    paper's 35 printed accuracy cells from the printed L2 cells; the two
    exceptions are the ones DESIGN.md lists."""
    tab = json.load(open(os.path.join(GOLDEN, "paper_tables.json")))
    hits, misses = 0, []
    for r in tab["rows"]:
        C = r["C_num"] / r["C_den"]
        got = metrics.paper_printed_accuracy(r["L"], C)
        if abs(got - r["printed"]) < 1e-9:
            hits += 1
        else:
            misses.append(r["label"])
            assert "exception" in r, r
    assert hits == 33 and sorted(misses) == ["clover 256^3", "nyx i40 1:8"]


def test_eq5_and_folds():
    a = np.random.default_rng(0).normal(size=(100, 3))
    assert metrics.total_avg_l2(a, a) == 0.0
    assert abs(metrics.total_avg_l2(a + np.array([3.0, 4.0, 0.0]), a) - 5.0) < 1e-12
    tab = json.load(open(os.path.join(GOLDEN, "paper_tables.json")))["max_l2_fold"]
    assert metrics.max_l2_stats(tab["maxima"]) == (tab["greatest"], tab["average"])
    assert metrics.accuracy_pct(0.0, 2.0) == 100.0 and metrics.accuracy_pct(2.0, 2.0) == 0.0


def test_eq2_double_interpolation_identity():
    """Eq. 2: interpolating through a filled hole equals direct
    interpolation between its valid neighbours."""
    f = np.array([10.0, -1.0, 30.0, 7.0, 99.0, 2.0])
    valid = np.array([True, False, True, True, False, True])
    x = np.linspace(0, 5, 51)
    got = metrics.grid_fill_1d(f, valid, x)
    direct = np.interp(x, np.nonzero(valid)[0].astype(float), f[valid])
    np.testing.assert_allclose(got, direct, atol=1e-12)
    assert abs(metrics.grid_fill_1d([10.0, 0.0, 30.0], [True, False, True], [0.5])[0] - 15.0) < 1e-12


def test_barycentric_affine_exact():
    """Barycentric interpolation is exact on affine flow maps."""
    rng = np.random.default_rng(5)
    pts = np.stack(np.meshgrid(*[np.arange(5.0)] * 3, indexing="ij"), -1).reshape(-1, 3)
    M = rng.normal(size=(3, 3)); t = rng.normal(size=3)
    q = rng.uniform(0.1, 3.9, (200, 3))
    out, ins = metrics.barycentric_interpolate(pts, pts @ M.T + t, q)
    assert ins.all()
    np.testing.assert_allclose(out, q @ M.T + t, atol=1e-9)


def test_abc_field_origin_value():
    tab = json.load(open(os.path.join(GOLDEN, "paper_tables.json")))["abc_origin"]
    g = grid3((3, 3, 3), h=(1.0, 1.0, 1.0))
    V = L.field_at_nodes(L.FieldSpec("abc", period=1.0), g, 0.0)
    np.testing.assert_allclose(V[0, 0, 0], tab["value"], rtol=1e-7)


def test_bto_update_only_exit_rotation():
    """The updated position is tested too, not only the stage samples.
    Solid-body rotation v = (-(y-cy), x-cx), particle at radius R east of the
    centre: by hand, q2_y = q3_y = y0 + R dt/2, q4_y = y0 + R (dt - dt^3/4) and
    x'_y = y0 + R (dt - dt^3/6).  With the block's upper y-face at y0 + h and
    R (dt - dt^3/4) < h <= R (dt - dt^3/6), every stage sample is inside but
    x' is not -> TERM_BOUNDARY at cycle 0 with the position unchanged."""
    h, dt = 0.5, 0.5
    R = h / 0.474
    assert R * (dt - dt ** 3 / 4) < h <= R * (dt - dt ** 3 / 6)
    g = L.Grid(3, (17, 17, 3), (0.0, 0.0, 0.0), (h, h, h))
    x0, y0 = 4.0, 4.0                      # seed node (8, 8)
    spec = L.FieldSpec("rotation", (1.0, x0 - R, y0))
    V = L.field_at_nodes(spec, g, 0.0)
    it = oracle.Interval(g, (0, 0, 0), (17, 9, 3), 1, oracle.BTO,
                         g_seeds=np.array([[8, 8, 0], [8, 4, 0]]))
    it.cycle(V, V, dt)
    assert it.status[0] == oracle.TERM_BOUNDARY and it.term_cycle[0] == 0
    assert np.array_equal(it.pos[0], [x0, y0, 0.0])
    # the same particle without the block face moves to the closed-form x'_y
    free = oracle.rk4_free(g, V, V, dt, np.array([[x0, y0, 0.0]]))
    assert abs(free[0, 1] - (y0 + R * (dt - dt ** 3 / 6))) < 1e-6


def test_grid_fill_affine_exact_and_eq2():
    """GridFill (Eq. 2) on the seed lattice is exact on affine flow maps and
    along a single lattice line reduces to grid_fill_1d / direct interpolation."""
    rng = np.random.default_rng(9)
    n = 12
    ax = np.arange(n)
    gz, gy, gx = np.meshgrid(ax, ax, ax, indexing="ij")
    lat = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], 1)
    M = rng.normal(size=(3, 3)); t = rng.normal(size=3)
    end = (lat * 0.3) @ M.T + t
    hole = (np.abs(lat[:, 0] - 6) <= 1) & (lat[:, 1] % 3 != 0)
    out, filled = metrics.grid_fill(lat, end, ~hole, hole)
    assert filled[hole].all()
    np.testing.assert_allclose(out[hole], end[hole], atol=1e-12)
    # one lattice line: equals the 1-D Eq. 2 fill
    f = rng.normal(size=n)
    valid = np.ones(n, bool); valid[[3, 4, 8]] = False
    lat1 = np.stack([np.arange(n), np.zeros(n, int)], 1)
    out1, fl1 = metrics.grid_fill(lat1, f[:, None], valid, ~valid)
    np.testing.assert_allclose(out1[~valid, 0], metrics.grid_fill_1d(f, valid, np.arange(n))[~valid], atol=1e-12)


def test_agreement_accepts_an_external_reconstruction():
    """metrics.agreement(recon=...) (used for the CUDA GridFill) gives the same
    numbers as its own GridFill when handed that GridFill's output."""
    import lag_inputs as L
    from oracle import metrics
    g = L.Grid(2, (12, 10, 1), (0.0, 0.0, 0.0), (0.1, 0.1, 1.0))
    gy, gx = np.meshgrid(np.arange(10), np.arange(12), indexing="ij")
    gs = np.stack([gx.ravel(), gy.ravel(), np.zeros(gx.size, int)], 1)
    rng = np.random.default_rng(3)
    end = gs[:, :2] * 0.1 + 0.01 * rng.standard_normal((gs.shape[0], 2))
    bst = np.where((gs[:, 0] == 5) | (gs[:, 0] == 6), 1, 0).astype(np.uint8)
    cst = np.zeros_like(bst)
    cend = end + 1e-3
    ref = metrics.agreement(g, gs, gs[:, :2] * 0.1, end, bst, cend, cst, 1, method="gridfill")
    rec = metrics.grid_fill(gs[:, :2], end, bst == 0, bst != 0)
    got = metrics.agreement(g, gs, gs[:, :2] * 0.1, end, bst, cend, cst, 1, recon=rec)
    assert got == ref
    assert ref["holes"] == 20 and ref["excluded"] == 0


# ---- FTLE (oracle/ftle.py) -----------------------

def _lattice_pts(dims, spacing):
    idx = np.indices(dims[::-1]).reshape(len(dims), -1)[::-1].T
    return idx * np.asarray(spacing, dtype=np.float64)


def test_ftle_identity_translation_and_rotation_are_zero():
    from oracle.ftle import ftle
    dims, sp = (7, 6, 5), (0.1, 0.2, 0.3)
    X = _lattice_pts(dims, sp)
    th = 0.7
    R = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1]])
    for F in (X, X + np.array([0.3, -1.0, 2.0]), X @ R.T + 0.5):
        out, nbad = ftle(F, dims, sp, 2.5)
        assert nbad == 0
        np.testing.assert_allclose(out, 0.0, atol=1e-14)


def test_ftle_diagonal_stretch_is_ln2():
    """SPEC.md:466 example: end = diag(2, 0.5) seed, T = 1 -> ln 2 (every
    node: one-sided differences are exact on linear maps too)."""
    from oracle.ftle import ftle
    dims, sp = (9, 8), (0.25, 0.5)
    X = _lattice_pts(dims, sp)
    out, _ = ftle(X * np.array([2.0, 0.5]), dims, sp, 1.0)
    np.testing.assert_allclose(out, np.log(2.0), rtol=0, atol=1e-14)
    out, _ = ftle(X * np.array([2.0, 0.5]), dims, sp, -4.0)           # |T|
    np.testing.assert_allclose(out, np.log(2.0) / 4.0, rtol=0, atol=1e-14)


def test_ftle_shear_closed_form():
    """F = (x + k y, y, z): lambda_max(C) = 1 + k^2/2 + k sqrt(1 + k^2/4)."""
    from oracle.ftle import ftle
    dims, sp, k, T = (6, 7, 5), (0.3, 0.2, 0.1), 1.7, 3.0
    X = _lattice_pts(dims, sp)
    F = X.copy()
    F[:, 0] += k * X[:, 1]
    out, _ = ftle(F, dims, sp, T)
    lam = 1 + k * k / 2 + k * np.sqrt(1 + k * k / 4)
    np.testing.assert_allclose(out, 0.5 * np.log(lam) / T, rtol=1e-13)


def test_ftle_quadratic_map_interior_central_difference_is_exact():
    """F = X + c X^2 per component: central differences are exact on
    quadratics, so interior nodes match the analytic gradient 1 + 2 c x;
    faces use one-sided differences (1 + c(2x + h))."""
    from oracle.ftle import ftle
    dims, sp, c, T = (8, 6), (0.2, 0.3), np.array([0.4, -0.3]), 1.5
    X = _lattice_pts(dims, sp)
    out, _ = ftle(X + c * X ** 2, dims, sp, T)
    ix = X / np.array(sp)
    g = 1 + 2 * c * X                                                  # interior: diagonal J
    lo = ix == 0
    hi = ix == np.array(dims) - 1
    g = np.where(lo, 1 + c * (2 * X + np.array(sp)), g)
    g = np.where(hi, 1 + c * (2 * X - np.array(sp)), g)
    expect = np.log(np.abs(g).max(axis=1)) / T
    np.testing.assert_allclose(out, expect, rtol=0, atol=1e-12)


def test_ftle_degenerate_tensor_counted_and_nan_propagates():
    from oracle.ftle import ftle
    dims, sp = (4, 4), (1.0, 1.0)
    F = np.zeros((16, 2))                                              # collapsed map: C = 0
    out, nbad = ftle(F, dims, sp, 1.0)
    assert nbad == 16 and (out == 0).all()
    F = _lattice_pts(dims, sp)
    F[5] = np.nan
    out, nbad = ftle(F, dims, sp, 1.0)
    # node 5 feeds the stencils of its 4 neighbours, not its own central difference
    assert np.isnan(out[[1, 4, 6, 9]]).all() and np.isfinite(out[[0, 5, 15]]).all() and nbad == 0


# ---- pathline stitching (oracle/pathline.py; §3.2) -

def _lat(dims, origin, sp):
    idx = np.indices(dims[::-1]).reshape(len(dims), -1)[::-1].T
    return np.asarray(origin) + idx * np.asarray(sp)


def test_kuhn_weights_reproduce_the_point_and_are_convex():
    from oracle.pathline import kuhn_weights
    rng = np.random.default_rng(11)
    for d in (2, 3):
        f = rng.random((500, d))
        f[:20, 0] = f[:20, 1]                               # ties
        f[20:30] = np.round(f[20:30])                       # cube corners
        off, w = kuhn_weights(f)
        assert (w >= 0).all()
        np.testing.assert_allclose(w.sum(1), 1.0, atol=1e-15)
        np.testing.assert_allclose(np.einsum("mj,mjc->mc", w, off), f, atol=1e-15)
        # consecutive vertices differ in exactly one axis (a Kuhn path 0 -> 1...1)
        assert (np.abs(np.diff(off, axis=1)).sum(2) == 1).all()


def test_stitched_affine_maps_compose_exactly():
    """Barycentric interpolation is exact on affine maps, so stitching the
    maps x -> M_k x + b_k equals their composition."""
    from oracle.pathline import stitch
    dims, o, sp = (9, 8, 7), (-1.0, 0.5, 2.0), (0.5, 0.25, 0.3)
    X = _lat(dims, o, sp)
    c = np.array(o) + (np.array(dims) - 1) * np.array(sp) / 2          # lattice centre
    maps = [(np.array([[1.02, 0.05, 0.0], [-0.03, 0.98, 0.02], [0.01, 0.0, 1.01]]), np.array([0.02, -0.01, 0.03])),
            (np.array([[0.99, -0.02, 0.01], [0.04, 1.01, 0.0], [0.0, 0.03, 0.97]]), np.array([-0.05, 0.02, 0.0])),
            (np.eye(3) * 1.01, np.array([0.0, 0.0, -0.02]))]
    ends = np.stack([(X - c) @ M.T + c + b for M, b in maps])
    rng = np.random.default_rng(4)
    q = c + (rng.random((200, 3)) - 0.5) * (np.array(dims) - 1) * np.array(sp) * 0.6
    path, status, samples, _ = stitch(ends, None, dims, o, sp, q)
    assert (status == 0).all() and (samples == 4).all()
    x = q.copy()
    for k, (M, b) in enumerate(maps):
        x = (x - c) @ M.T + c + b
        np.testing.assert_allclose(path[:, k + 1], x, rtol=0, atol=1e-13)


def test_stitch_uniform_flow_example_and_hull_truncation():
    """uniform v = (1,0,0), dt = 0.1, two intervals of 5 cycles,
    seed (0.1, 0.5, 0.5) -> samples (0.6, .5, .5), (1.1, .5, .5); a third
    interval from 1.1 on a [0, 1.5] lattice lands outside the hull and the
    fourth is truncated."""
    from oracle.pathline import stitch, OUT_OF_HULL
    dims, o, sp = (16, 3, 3), (0.0, 0.0, 0.0), (0.1, 0.5, 0.5)
    X = _lat(dims, o, sp)
    ends = np.stack([X + np.array([0.5, 0.0, 0.0])] * 4)
    path, status, samples, _ = stitch(ends, None, dims, o, sp, np.array([[0.1, 0.5, 0.5]]))
    np.testing.assert_allclose(path[0, 1], [0.6, 0.5, 0.5], atol=1e-15)
    np.testing.assert_allclose(path[0, 2], [1.1, 0.5, 0.5], atol=1e-15)
    np.testing.assert_allclose(path[0, 3], [1.6, 0.5, 0.5], atol=1e-15)   # interpolated from inside
    assert status[0] == OUT_OF_HULL and samples[0] == 4 and np.isnan(path[0, 4]).all()


def test_stitch_identity_map_is_stationary_and_invalid_flows_truncate():
    from oracle.pathline import stitch, INVALID_FLOW
    dims, o, sp = (5, 4), (0.0, 0.0), (1.0, 1.0)
    X = _lat(dims, o, sp)
    ends = np.stack([X, X])
    valid = np.ones((2, 20), bool)
    valid[1, 6] = False                                        # node (1, 1)
    q = np.array([[1.0, 2.0], [1.5, 1.25], [2.0, 2.0], [0.5, 2.5], [4.0, 3.0]])   # last: top corner
    path, status, samples, _ = stitch(ends, valid, dims, o, sp, q)
    # (1.5, 1.25) lies in the cube at (1, 1), whose simplex holds node (1, 1)
    # with weight 0.5 > 0, so its second interval is truncated.  Nodes and
    # points whose simplex gives (1, 1) weight 0 are unaffected.
    assert list(status) == [0, INVALID_FLOW, 0, 0, 0]
    np.testing.assert_array_equal(path[[0, 2, 3, 4], 2], q[[0, 2, 3, 4]])
    assert samples[1] == 2


def test_stitch_interpolant_is_continuous_across_simplices_and_cubes():
    """Kuhn simplices conform: for a nonlinear map, the interpolant evaluated
    just either side of simplex facets (f_a = f_b) and of cube faces differs
    by O(eps)."""
    from oracle.pathline import stitch
    dims, o, sp = (6, 6, 6), (0.0, 0.0, 0.0), (1.0, 1.0, 1.0)
    X = _lat(dims, o, sp)
    ends = (X + 0.3 * np.sin(X[:, ::-1]) + 0.1 * X ** 2)[None]
    rng = np.random.default_rng(8)
    base = 1 + 3 * rng.random((300, 3))
    base[:100, 1] = np.floor(base[:100, 1]) + (base[:100, 0] - np.floor(base[:100, 0]))   # f_x = f_y facet
    base[100:200, 2] = np.round(base[100:200, 2])                                        # cube face
    eps = 1e-9
    for ax in range(3):
        dv = np.zeros(3)
        dv[ax] = eps
        a = stitch(ends, None, dims, o, sp, base + dv)[0][:, 1]
        b = stitch(ends, None, dims, o, sp, base - dv)[0][:, 1]
        assert np.abs(a - b).max() < 50 * eps


# ------------------------------------------------ excuse band, sector counter,
# GridFill axis choice, Delaunay tiling (the functions behind the flag-parity
# excuse band, the roofline's algorithmic bytes and the agreement metric)

def _uniform_x(grid, U=1.0):
    V = np.zeros((grid.nodes[2], grid.nodes[1], grid.nodes[0], 3), dtype=np.float32)
    V[..., 0] = U
    return V


def test_face_distance_uniform_flow_closed_form():
    """Reading R14: min over post-seed stage samples and
    committed positions of the distance, in cells, to any block or global
    face.  Uniform flow u = (1,0,0), h = 1, dt = 1/4 (all samples dyadic, exact
    in fp64): a seed at x = g visits g + n/4 + 1/8 (stages 2, 3) and
    g + (n+1)/4 (stage 4 and the committed position), n = 0..I-1.  Block
    x in [0, 8) of N_x = 17 (faces 0, 8, 16); y = z = 4 of N = 9 (distance 4).
    Hand values: g = 2 -> 2.125 (the first stage sample; the seed itself,
    2.0, does not count), g = 3 -> 3.0 (x = 5 at the end, 3 from face 8),
    g = 5 -> 1.0 (x = 7), g = 7 -> 0.0 (stage 4 of cycle 3 lands on face 8 and
    terminates there)."""
    g = grid3((17, 9, 9))
    V = _uniform_x(g)
    seeds = np.array([[2, 4, 4], [3, 4, 4], [5, 4, 4], [7, 4, 4], [0, 4, 4]], dtype=np.int64)
    it = oracle.Interval(g, (0, 0, 0), (8, 9, 9), 1, oracle.BTO, g_seeds=seeds)
    for _ in range(8):
        it.cycle(V, V, 0.25)
    assert it.min_face[:4].tolist() == [2.125, 3.0, 1.0, 0.0]
    assert it.status.tolist() == [0, 0, 0, 1, 0]
    assert it.term_cycle[3] == 3
    # seed 0 sits on the block's lower face and on the global face: its first
    # stage sample is 1/8 away
    assert it.min_face[4] == 0.125
    # far from every x-face the y/z faces decide (4 cells)
    g2 = grid3((41, 9, 9))
    it2 = oracle.Interval(g2, (0, 0, 0), (41, 9, 9), 1, oracle.BTO,
                          g_seeds=np.array([[10, 4, 4]], dtype=np.int64))
    for _ in range(4):
        it2.cycle(_uniform_x(g2), _uniform_x(g2), 0.25)
    assert it2.min_face[0] == 4.0


def test_touched_nodes_exact_set_uniform_flow():
    """The sector counter's node map (scripts/algbytes.py, the roofline's
    algorithmic bytes): bit 0 = nodes of V_t the stage gathers read (stages
    1-3), bit 1 = nodes of V_t1 (stages 2-4).  Uniform flow (1,0,0), dt = 1/4,
    one cycle from node (2,1,1): every stage sample (x = 2, 2.125, 2.125, 2.25)
    lies in cell (2,1,1), so exactly its 8 corners x in {2,3}, y in {1,2},
    z in {1,2} carry both bits.  From the closed top face x = 5 = N-1 moving
    in -x the cell is clamped to 4 (corners {4,5}); stage samples 4.875 stay
    in cell 4."""
    g = grid3((6, 5, 4))
    expected = np.zeros((4, 5, 6), dtype=np.uint8)
    for z in (1, 2):
        for y in (1, 2):
            for x in (2, 3):
                expected[z, y, x] = 3
    V = _uniform_x(g)
    touched = np.zeros((4, 5, 6), dtype=np.uint8)
    it = oracle.Interval(g, (0, 0, 0), (6, 5, 4), 1, oracle.BTO,
                         g_seeds=np.array([[2, 1, 1]], dtype=np.int64))
    it.cycle(V, V, 0.25, touched=touched)
    np.testing.assert_array_equal(touched, expected)
    # the brute-force tent support of every stage sample lies inside the set
    for xs in (2.0, 2.125, 2.25):
        for idx in np.ndindex(4, 5, 6):
            n = idx[::-1]
            w = max(0.0, 1 - abs(xs - n[0])) * max(0.0, 1 - abs(1 - n[1])) * max(0.0, 1 - abs(1 - n[2]))
            if w > 0:
                assert touched[idx] == 3
    # clamped top face
    touched[:] = 0
    Vm = _uniform_x(g, U=-1.0)
    it = oracle.Interval(g, (0, 0, 0), (6, 5, 4), 1, oracle.BTO,
                         g_seeds=np.array([[5, 1, 1]], dtype=np.int64))
    it.cycle(Vm, Vm, 0.25, touched=touched)
    expected[:] = 0
    for z in (1, 2):
        for y in (1, 2):
            for x in (4, 5):
                expected[z, y, x] = 3
    np.testing.assert_array_equal(touched, expected)
    assert it.status[0] == 0 and it.pos[0, 0] == 4.75


def test_grid_fill_takes_the_shortest_bracket():
    """Reading R18: a hole is filled along the lattice axis with
    the shortest valid bracket (ties averaged).  5x5 lattice, holes at
    (2,1), (2,2), (2,3); valid values v = 10 i + j^2 (not affine in j, so the
    axes disagree).  Hole (2,2): x-bracket (1,2)-(3,2), span 2 -> (14 + 34)/2
    = 24; y-bracket (2,0)-(2,4), span 4 -> (20 + 36)/2 = 28.  Hole (2,1):
    x -> (11 + 31)/2 = 21; y (span 4) -> 20 + 16/4 = 24.  The shortest-bracket
    rule gives 24 and 21; averaging both axes would give 26 and
    22.5; the longest bracket 28 and 24."""
    lat = np.array([[i, j] for j in range(5) for i in range(5)], dtype=np.int64)
    vals = (10.0 * lat[:, 0] + lat[:, 1] ** 2)[:, None].astype(np.float64)
    hole = np.zeros(25, dtype=bool)
    for (i, j) in ((2, 1), (2, 2), (2, 3)):
        hole[j * 5 + i] = True
    valid = ~hole
    out, filled = metrics.grid_fill(lat, np.where(valid[:, None], vals, np.nan), valid, hole)
    assert filled.sum() == 3
    assert out[2 * 5 + 2, 0] == 24.0
    assert out[1 * 5 + 2, 0] == 21.0
    assert out[3 * 5 + 2, 0] == (19 + 39) / 2     # x-bracket (1,3)-(3,3)
    # a tie (isolated hole: spans 2 on both axes) averages the two fills
    hole2 = np.zeros(25, dtype=bool)
    hole2[2 * 5 + 2] = True
    out2, _ = metrics.grid_fill(lat, vals, ~hole2, hole2)
    assert out2[12, 0] == ((14 + 34) / 2 + (21 + 29) / 2) / 2


def test_reconstruct_holes_one_interior_hole_and_one_corner():
    """Reading R12 (Delaunay over the valid seeds around each hole tile,
    barycentric end interpolation): on a 7x7 lattice with an affine
    end map, the interior hole (3,3) is reconstructed exactly (barycentric
    interpolation is exact on affine maps) and the corner hole (0,0) lies
    outside the hull of the valid seeds, so it is excluded: exactly 1 of 2.
    The tile triangulates the valid seeds within `margin` lattice steps of its
    holes; with none (margin 0) nothing would be reconstructed."""
    n = 7
    g = np.array([[i, j, 0] for j in range(n) for i in range(n)], dtype=np.int64)
    start = g[:, :2].astype(np.float64)
    M = np.array([[1.1, 0.3], [-0.2, 0.9]])
    end = start @ M.T + np.array([0.25, -0.5])
    hole = np.zeros(n * n, dtype=bool)
    hole[0] = True
    hole[3 * n + 3] = True
    valid = ~hole
    rec, inside = metrics.reconstruct_holes(g, start, np.where(valid[:, None], end, np.nan), valid,
                                            hole, 1, workers=1)
    assert inside.tolist().count(True) == 1 and bool(inside[3 * n + 3]) and not inside[0]
    np.testing.assert_allclose(rec[3 * n + 3], end[3 * n + 3], rtol=0, atol=1e-12)
    # the agreement fold counts it: one hole compared, one excluded
    st = np.where(valid, 0, 1).astype(np.uint8)
    grid = L.Grid(2, (n, n, 1), (0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
    r = metrics.agreement(grid, g, start, np.where(valid[:, None], end, np.nan), st, end,
                          np.zeros(n * n, dtype=np.uint8), 1)
    assert r["holes"] == 2 and r["excluded"] == 1 and r["compared"] == n * n - 1
    assert r["L"] < 1e-12
