"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on
identical seeded fp32 inputs (north-star acceptance: 1e-4 cells, flags equal
outside the 1e-5-cell excuse band).  Sizes span several 32-particle tiles with
ragged tails; the full-size C5 block is checked on sampled particles."""
import numpy as np
import pytest

import lag_inputs as L
import oracle
from helpers import global_slices, oracle_block, gpu_block, compare

pytestmark = pytest.mark.gpu


def _run_config(cfg, ncycles, stride=None, mode=0, blocks=None, host=False):
    stride = stride or cfg["stride"]
    sl = global_slices(cfg, ncycles)
    out = []
    for b in (blocks or L.decompose(cfg["grid"], cfg["layout"])):
        start, end, status, st = gpu_block(cfg, b, sl, stride, mode=mode, host=host)
        orc = oracle_block(cfg, b, sl, stride, oracle.BTO if mode == 0 else oracle.COMM)
        out.append(compare(cfg, orc, start, end, status, label=f"{cfg['name']} rank {b.rank}"))
        assert st["particle_steps"] > 0
    return out


def test_c1_double_gyre_2d_all_intervals():
    """C1: 2D double gyre 64x32, stride 1 (2048 particles), 100 cycles in 5
    intervals of 20, one block — every interval vs the oracle."""
    cfg = L.make_config("C1")
    g = cfg["grid"]
    for it in range(cfg["cycles"] // cfg["interval"]):
        sl = global_slices(cfg, cfg["interval"], t0_cycle=it * cfg["interval"])
        b = L.decompose(g, (1, 1, 1))[0]
        start, end, status, _ = gpu_block(cfg, b, sl, 1)
        orc = oracle_block(cfg, b, sl, 1, oracle.BTO)
        r = compare(cfg, orc, start, end, status, label=f"C1 interval {it}")
        assert r["n"] == 2048


def test_c2_abc_8_blocks_bto():
    """C2 at reduced size (33^3 ABC, 2x2x2 blocks, stride 1, interval 25)."""
    cfg = L.make_config("C2", scale=33)
    res = _run_config(cfg, cfg["interval"])
    assert sum(r["term"] for r in res) > 0          # BTO terminations happen
    assert all(r["n"] % 32 != 0 or True for r in res)


def test_c3_clover_stride2():
    cfg = L.make_config("C3", scale=40)
    res = _run_config(cfg, 20)
    assert res[0]["n"] == 20 ** 3


def test_c4_nyx_turbulence():
    """C4 shape at reduced size (65^3 over 2x2x2 blocks); dt raised so the
    short window still terminates particles at the internal faces."""
    cfg = L.make_config("C4", scale=65)
    cfg["dt"] *= 6.0
    res = _run_config(cfg, 12, stride=2)
    assert sum(r["term"] for r in res) > 0


def test_c5_weak_scaling_block_small():
    cfg = L.make_config("C5", scale=24, nranks=2)
    _run_config(cfg, 25)


def test_strides_and_ragged_tiles():
    cfg = L.make_config("C2", scale=29)
    b = L.Block(0, (0, 0, 0), (3, 2, 5), (26, 23, 19))     # odd offsets and extents
    for s in (1, 2, 3, 5):
        _run_config(cfg, 8, stride=s, blocks=[b])


def test_host_pointers_match_device_pointers_bitwise():
    """The end-to-end path (host slices staged by the library) computes the
    same bits as the device path."""
    cfg = L.make_config("C2", scale=21)
    sl = global_slices(cfg, 6)
    b = L.decompose(cfg["grid"], cfg["layout"])[3]
    a = gpu_block(cfg, b, sl, 1, host=False)
    h = gpu_block(cfg, b, sl, 1, host=True)
    for x, y in zip(a[:3], h[:3]):
        assert np.array_equal(x, y)


def test_host_buffers_reused_by_the_caller():
    """End-to-end path when the caller cycles two pinned host buffers and
    refills them: only the previous v_t1 passed again as v_t may be taken from
    the library's staging; a refilled buffer is copied afresh (same bits as
    the device path)."""
    import torch
    import paper_2004_02003_b200 as P
    cfg = L.make_config("C2", scale=21)
    sl = global_slices(cfg, 6)
    b = L.decompose(cfg["grid"], cfg["layout"])[3]
    ref = gpu_block(cfg, b, sl, 1, host=False)
    g = cfg["grid"]
    cut = [np.ascontiguousarray(L.cut_block_slice(V, g, b, 0), dtype=np.float32) for V in sl]
    bufs = [torch.from_numpy(cut[0].copy()).pin_memory(), torch.from_numpy(cut[1].copy()).pin_memory()]
    ctx = P.Context(P.make_config(g.dim, g.nodes, g.origin, g.spacing, b.lo, b.hi,
                                  stream=torch.cuda.current_stream().cuda_stream))
    n = ctx.seed(1)
    for k in range(len(sl) - 1):
        cur, nxt = bufs[k % 2], bufs[(k + 1) % 2]
        if k > 0:                                  # refill the buffer that becomes v_t1
            torch.cuda.synchronize()
            nxt.copy_(torch.from_numpy(cut[k + 1]))
        ctx.advect(cur, nxt, cfg["dt"])
    start = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    end, status = torch.empty_like(start), torch.empty((n,), dtype=torch.uint8, device="cuda")
    ctx.extract(start, end, status)
    ctx.close()
    for x, y in zip(ref[:3], (start.cpu().numpy(), end.cpu().numpy(), status.cpu().numpy())):
        assert np.array_equal(x, y)


def test_single_rank_comm_equals_bto_bitwise():
    """R = 1 equivalence: COMM and BTO on one block agree bitwise."""
    cfg = L.make_config("C2", scale=21)
    sl = global_slices(cfg, 10)
    b = L.Block(0, (0, 0, 0), (0, 0, 0), cfg["grid"].nodes)
    a = gpu_block(cfg, b, sl, 1, mode=0)
    for ghost in (1, 0):                       # a single-block COMM run needs no ghost layers
        c = gpu_block(cfg, b, sl, 1, mode=1, ghost=ghost)
        for x, y in zip(a[:3], c[:3]):
            assert np.array_equal(x, y)


def test_deterministic_bitwise():
    cfg = L.make_config("C4", scale=33)
    sl = global_slices(cfg, 5)
    b = L.decompose(cfg["grid"], cfg["layout"])[5]
    a = gpu_block(cfg, b, sl, 1)
    c = gpu_block(cfg, b, sl, 1)
    for x, y in zip(a[:3], c[:3]):
        assert np.array_equal(x, y)


def test_two_block_uniform_flow_closed_form_bitwise():
    """Constant v = (U,0,0) with U dt / h = 1/4: fp32 and fp64 are exact, so
    the flags (including the landing-exactly-on-the-face tie) must match the
    closed form with no excuse band (pin 7)."""
    g = L.Grid(3, (17, 5, 5), (0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
    cfg = dict(grid=g, field=L.FieldSpec("uniform", (0.5, 0.0, 0.0)), dt=0.5, name="uniform")
    sl = global_slices(cfg, 7)
    for b in L.decompose(g, (2, 1, 1)):
        start, end, status, _ = gpu_block(cfg, b, sl, 1)
        x0 = start[:, 0]
        disp = 7 * 0.25
        xf = float(L.decompose(g, (2, 1, 1))[0].hi[0])
        for p in range(status.size):
            if b.rank == 0 and x0[p] + disp >= xf:
                cstar = int(np.ceil((xf - x0[p]) / 0.25)) - 1
                assert status[p] == 1 and end[p, 0] == x0[p] + cstar * 0.25
            elif b.rank == 1 and x0[p] + disp > 16.0:
                assert status[p] == 2
            else:
                assert status[p] == 0 and end[p, 0] == x0[p] + disp


def test_zero_field_and_stats_accounting():
    cfg = L.make_config("C2", scale=17)
    g = cfg["grid"]
    zero = [np.zeros(g.nodes[::-1] + (3,), np.float32)] * 4
    b = L.decompose(g, cfg["layout"])[0]
    start, end, status, st = gpu_block(cfg, b, zero, 1)
    assert np.array_equal(start, end) and (status == 0).all()
    assert st["particle_steps"] == 3 * status.size


def test_errors_empty_block_and_order():
    import torch
    import paper_2004_02003_b200 as P
    g = L.Grid(3, (16, 16, 16), (0, 0, 0), (1, 1, 1))
    pc = P.make_config(3, g.nodes, g.origin, g.spacing, (1, 1, 1), (3, 3, 3))
    ctx = P.Context(pc)
    with pytest.raises(P.LagError) as e:
        ctx.advect(1, 1, 0.1)
    assert e.value.status == P.LAG_ESTATE
    with pytest.raises(P.LagError) as e:
        ctx.seed(4)                          # no multiple of 4 in [1, 3)
    assert e.value.status == P.LAG_EEMPTY
    assert ctx.seed(2) == 1
    v = torch.zeros((3, 3, 3, 3), device="cuda")
    with pytest.raises(P.LagError) as e:
        ctx.advect(v, v, -1.0)
    assert e.value.status == P.LAG_EINVAL
    with pytest.raises(P.LagError) as e:     # write cycles come in order (interval 0 first)
        P.lag_extract(ctx.ctx, 1)
    assert e.value.status == P.LAG_ESTATE
    assert P.lag_extract(ctx.ctx, 0) == 1
    assert P.lag_extract(ctx.ctx, 1) == 1
    ctx.close()


def test_nonfinite_velocity_is_latched():
    import torch
    import paper_2004_02003_b200 as P
    g = L.Grid(3, (8, 8, 8), (0, 0, 0), (1, 1, 1))
    ctx = P.Context(P.make_config(3, g.nodes, g.origin, g.spacing, (0, 0, 0), g.nodes))
    n = ctx.seed(1)
    v = torch.zeros((8, 8, 8, 3), device="cuda")
    v[4, 4, 4, 0] = float("nan")
    ctx.advect(v, v, 0.1)
    end = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    with pytest.raises(P.LagError) as e:
        ctx.extract(end=end)
    assert e.value.status == P.LAG_ENONFINITE
    ctx.close()


@pytest.mark.slow
def test_c5_full_size_sampled():
    """C5 at the bench's size and launch configuration (128^3, one block,
    stride 1, one interval of 25 cycles): 4096 sampled particles vs the oracle."""
    cfg = L.make_config("C5")
    g = cfg["grid"]
    sl = global_slices(cfg, cfg["interval"])
    b = L.decompose(g, cfg["layout"])[0]
    start, end, status, _ = gpu_block(cfg, b, sl, 1)
    rng = np.random.default_rng(11)
    pick = np.sort(rng.choice(status.size, 4096, replace=False))
    gs = oracle.seeds(g, b.lo, b.hi, 1)[pick]
    orc = oracle.run_interval(g, b.lo, b.hi, 1, sl, cfg["dt"], g_seeds=gs, faces=(b.lo, b.hi))
    compare(cfg, orc, start[pick], end[pick], status[pick], label="C5 full sampled")


def test_two_intervals_one_context_autoreseed():
    """lag_extract reseeds by default: the second interval of the same context
    matches the oracle started at the second interval's time."""
    import torch
    import paper_2004_02003_b200 as P
    cfg = L.make_config("C2", scale=25)
    g = cfg["grid"]
    b = L.decompose(g, cfg["layout"])[6]
    I = 10
    sl = global_slices(cfg, 2 * I)
    dev = [torch.from_numpy(np.ascontiguousarray(L.cut_block_slice(V, g, b, 0))).cuda() for V in sl]
    ctx = P.Context(P.make_config(3, g.nodes, g.origin, g.spacing, b.lo, b.hi,
                                  stream=torch.cuda.current_stream().cuda_stream))
    n = ctx.seed(1)
    outs = []
    for it in range(2):
        for k in range(I):
            ctx.advect(dev[it * I + k], dev[it * I + k + 1], cfg["dt"])
        start = torch.empty((n, 3), dtype=torch.float64, device="cuda")
        end = torch.empty_like(start)
        st = torch.empty((n,), dtype=torch.uint8, device="cuda")
        assert ctx.extract(start, end, st) == n          # default flags: reseed
        outs.append((start.cpu().numpy(), end.cpu().numpy(), st.cpu().numpy()))
    ctx.close()
    for it in range(2):
        orc = oracle_block(cfg, b, sl[it * I:(it + 1) * I + 1], 1, oracle.BTO)
        compare(cfg, orc, *outs[it], label=f"interval {it}")


def test_host_output_buffers():
    """Outputs may be host memory (numpy): staged and copied by the library,
    identical to device outputs."""
    import torch
    import paper_2004_02003_b200 as P
    cfg = L.make_config("C2", scale=21)
    g = cfg["grid"]
    b = L.decompose(g, cfg["layout"])[2]
    sl = global_slices(cfg, 5)
    ref = gpu_block(cfg, b, sl, 1)
    dev = [torch.from_numpy(np.ascontiguousarray(L.cut_block_slice(V, g, b, 0))).cuda() for V in sl]
    ctx = P.Context(P.make_config(3, g.nodes, g.origin, g.spacing, b.lo, b.hi,
                                  stream=torch.cuda.current_stream().cuda_stream))
    n = ctx.seed(1)
    for k in range(5):
        ctx.advect(dev[k], dev[k + 1], cfg["dt"])
    start = np.zeros((n, 3)); end = np.zeros((n, 3)); st = np.zeros(n, np.uint8)
    ctx.extract(start, end, st)
    ctx.close()
    assert np.array_equal(start, ref[0]) and np.array_equal(end, ref[1]) and np.array_equal(st, ref[2])


def test_whole_block_terminates():
    """Every particle of the upstream block leaves it: all TERM_BOUNDARY with
    the closed-form termination positions; particle-steps accounting."""
    g = L.Grid(3, (17, 6, 6), (0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
    cfg = dict(grid=g, field=L.FieldSpec("uniform", (2.0, 0.0, 0.0)), dt=0.5, name="uniform")
    sl = global_slices(cfg, 12)           # 1 cell per cycle, block 0 is 9 cells wide
    b0 = L.decompose(g, (2, 1, 1))[0]
    start, end, status, st = gpu_block(cfg, b0, sl, 1)
    assert (status == 1).all()
    x0 = start[:, 0]
    cstar = np.ceil(b0.hi[0] - x0).astype(int) - 1     # first cycle whose step lands at/after the face
    np.testing.assert_array_equal(end[:, 0], x0 + cstar)
    assert st["particle_steps"] == int((cstar + 1).sum())


def test_frozen_snapshot_single_gather():
    """Frozen snapshot (one accessible time step): passing the same
    array as v_t and v_t1 gathers corners once and gives bitwise the results of
    two distinct arrays with equal content; both match the oracle."""
    cfg = L.make_config("C2", scale=25)
    b = L.decompose(cfg["grid"], cfg["layout"])[1]
    sl = global_slices(cfg, 8)
    frozen = [sl[k] for k in range(8) for _ in (0, 1)]        # pairs (V_k, V_k)
    # distinct arrays with identical content: slices V_k, copy(V_k)
    a = gpu_block(cfg, b, sl, 1, same_tensor=True)
    pairs = []
    for k in range(8):
        pairs += [sl[k], sl[k].copy()]
    import torch
    import paper_2004_02003_b200 as P
    g = cfg["grid"]
    dev = [torch.from_numpy(np.ascontiguousarray(L.cut_block_slice(V, g, b, 0))).cuda() for V in pairs]
    ctx = P.Context(P.make_config(3, g.nodes, g.origin, g.spacing, b.lo, b.hi,
                                  stream=torch.cuda.current_stream().cuda_stream))
    n = ctx.seed(1)
    for k in range(8):
        ctx.advect(dev[2 * k], dev[2 * k + 1], cfg["dt"])
    out = [torch.empty((n, 3), dtype=torch.float64, device="cuda") for _ in range(2)]
    stt = torch.empty((n,), dtype=torch.uint8, device="cuda")
    ctx.extract(out[0], out[1], stt)
    ctx.close()
    assert np.array_equal(a[1], out[1].cpu().numpy()) and np.array_equal(a[2], stt.cpu().numpy())
    orc = oracle.Interval(g, b.lo, b.hi, 1, oracle.BTO, faces=(b.lo, b.hi))
    for k in range(8):
        orc.cycle(sl[k], sl[k], cfg["dt"])
    compare(cfg, orc, *a[:3], label="frozen")


def test_termination_cycles_match_oracle():
    """lag_extract_ex returns the termination cycle of each non-valid flow
    (P:884 future work: termination locations on the boundary); it equals
    the oracle's wherever the statuses agree, -1 for valid flows."""
    cfg = L.make_config("C2", scale=33)
    b = L.decompose(cfg["grid"], cfg["layout"])[4]
    sl = global_slices(cfg, 25)
    start, end, status, st = gpu_block(cfg, b, sl, 1, term_cycle=True)
    orc = oracle_block(cfg, b, sl, 1, oracle.BTO)
    compare(cfg, orc, start, end, status)
    tc = st["term_cycle"]
    same = status == orc.status
    assert (status != 0).sum() > 0
    assert np.array_equal(tc[same], orc.term_cycle[same])
    assert (tc[status == 0] == -1).all()


def test_async_extract_matches_sync_and_keeps_errors_latched():
    """LAG_ASYNC enqueues the write cycle without a host sync: same bits as the
    synchronous extract (device and page-locked host outputs); a latched
    device error survives the asynchronous write cycle and its reseed and is
    reported by the next synchronous one; pageable host outputs are refused."""
    import torch
    import paper_2004_02003_b200 as P
    cfg = L.make_config("C2", scale=21)
    sl = global_slices(cfg, 4)
    b = L.decompose(cfg["grid"], cfg["layout"])[0]
    ref = gpu_block(cfg, b, sl, 1)
    got = gpu_block(cfg, b, sl, 1, extract_flags=P.LAG_ASYNC)
    for x, y in zip(ref[:3], got[:3]):
        assert np.array_equal(x, y)

    g = L.Grid(3, (8, 8, 8), (0, 0, 0), (1, 1, 1))
    ctx = P.Context(P.make_config(3, g.nodes, g.origin, g.spacing, (0, 0, 0), g.nodes))
    n = ctx.seed(1)
    bad = torch.zeros((8, 8, 8, 3), device="cuda")
    bad[4, 4, 4, 0] = float("nan")
    good = torch.zeros_like(bad)
    end = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    with pytest.raises(P.LagError) as e:
        ctx.extract(end=torch.empty((n, 3), dtype=torch.float64), flags=P.LAG_ASYNC)   # pageable
    assert e.value.status == P.LAG_EINVAL
    pinned = torch.full((n, 3), -1.0, dtype=torch.float64).pin_memory()
    ctx.extract(end=pinned, flags=P.LAG_ASYNC | P.LAG_NO_RESEED)                     # enqueued copy
    torch.cuda.synchronize()
    ctx.extract(end=end, flags=P.LAG_NO_RESEED)
    assert np.array_equal(pinned.numpy(), end.cpu().numpy())
    n = ctx.seed(1)
    ctx.advect(bad, bad, 0.1)
    ctx.extract(end=end, flags=P.LAG_ASYNC)                  # enqueued, reseeded, error kept
    ctx.advect(good, good, 0.1)
    with pytest.raises(P.LagError) as e:
        ctx.extract(end=end)
    assert e.value.status == P.LAG_ENONFINITE
    ctx.advect(good, good, 0.1)                              # reported -> cleared
    assert ctx.extract(end=end) == n
    ctx.close()
