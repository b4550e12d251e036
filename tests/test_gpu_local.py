"""COMM baseline on ONE GPU: the blocks of a decomposition as LAG_XCHG_LOCAL
contexts of one process (lag_local_group).  The exchange (ghost layers from
the neighbours' slice arrays, hand-offs appended from their slots, return to
origin at the write cycle) runs through the same advect kernel, append and
scatter code as the NCCL/peer transports, so this covers the COMM rows
(halo fill, particle hand-off, return to origin) on the
driver's 1-GPU box:

  * COMM over all blocks == the single-block run of the whole domain,
    BITWISE (decomposition invariance), with the ghost layers
    poisoned with NaN until the exchange fills them;
  * the single-block run vs the fp64 oracle (north-star rule);
  * hand-offs happen (sent == received > 0) and every seed comes back to its
    origin block at the write cycle, over several intervals (deferred reseed);
  * padded rows (row_pitch_bytes) give bitwise the dense result.
"""
import numpy as np
import pytest

import lag_inputs as L
import oracle
from helpers import global_slices, gpu_block, compare

pytestmark = pytest.mark.gpu


def poisoned_block_slice(V, g, b, ghost, pad=0):
    """Block slice with `ghost` layers, ghost nodes NaN (only the exchange may
    fill them), rows padded by `pad` NaN nodes (row_pitch_bytes)."""
    s = np.array(L.cut_block_slice(V, g, b, ghost), dtype=np.float32)
    if ghost:
        for ax in range(g.dim):
            nax = s.ndim - 2 - ax
            for k in list(range(ghost)) + list(range(s.shape[nax] - ghost, s.shape[nax])):
                idx = [slice(None)] * s.ndim
                idx[nax] = k
                s[tuple(idx)] = np.nan
    if pad:
        shape = list(s.shape)
        shape[-2] += pad
        p = np.full(shape, np.nan, dtype=np.float32)
        p[..., :s.shape[-2], :] = s
        s = p
    return s


def run_local(cfg, layout, slices_per_interval, stride, pad=0, frozen=False, reseed_mid=None,
              streams=False):
    """All blocks of `layout` as one LAG_XCHG_LOCAL group on cuda:0 (one
    stream, or one stream per block).  Returns, per interval, per block
    (start, end, status) and the group's stats."""
    import torch
    import paper_2004_02003_b200 as P
    g = cfg["grid"]
    blocks = L.decompose(g, layout)
    cfgs = []
    own = [torch.cuda.Stream() for _ in blocks] if streams else None
    for b in blocks:
        s = own[b.rank] if streams else torch.cuda.current_stream()
        ext = L.block_slice_extent(g, b, 1)
        pitch = (ext[0] + pad) * g.dim * 4 if pad else 0
        cfgs.append(P.make_config(g.dim, g.nodes, g.origin, g.spacing, b.lo, b.hi, mode=P.LAG_COMM,
                                  ghost=1, rank=b.rank, nranks=len(blocks), layout=layout,
                                  stream=s.cuda_stream, exchange=P.LAG_XCHG_LOCAL,
                                  row_pitch_bytes=pitch))
    grp = P.LocalGroup(cfgs)
    results, stats = [], []
    try:
        ns = grp.seed(stride)
        for it, sl in enumerate(slices_per_interval):
            dev = [[torch.from_numpy(poisoned_block_slice(V, g, b, 1, pad)).cuda() for b in blocks] for V in sl]
            for k in range(len(sl) - 1):
                if reseed_mid is not None and it == 0 and k == reseed_mid:
                    grp.seed(stride)                # mid-interval reseed: in-flight hand-offs dropped
                    break
                grp.advect(dev[k], dev[k] if frozen else dev[k + 1], cfg["dt"])
            if reseed_mid is not None and it == 0:
                continue
            outs = [(torch.empty((n, g.dim), dtype=torch.float64, device="cuda"),
                     torch.empty((n, g.dim), dtype=torch.float64, device="cuda"),
                     torch.empty((n,), dtype=torch.uint8, device="cuda")) for n in ns]
            if streams:                             # the outputs were allocated on the current stream
                torch.cuda.synchronize()
            stats.append(grp.stats())               # before the write cycle: hand-offs in flight
            grp.extract(outs)
            torch.cuda.synchronize()
            results.append([tuple(x.cpu().numpy() for x in o) for o in outs])
    finally:
        grp.close()
    return blocks, results, stats


def assemble(g, blocks, per_block, stride):
    """Scatter per-block flow maps into the global seed order."""
    gs = oracle.seeds(g, (0, 0, 0), g.nodes, stride)
    key = {tuple(x): i for i, x in enumerate(gs.tolist())}
    n = gs.shape[0]
    start = np.full((n, g.dim), np.nan)
    end = np.full((n, g.dim), np.nan)
    status = np.full(n, 255, dtype=np.uint8)
    for b, (s, e, st) in zip(blocks, per_block):
        idx = np.array([key[tuple(x)] for x in oracle.seeds(g, b.lo, b.hi, stride).tolist()])
        start[idx], end[idx], status[idx] = s, e, st
    return start, end, status


@pytest.mark.parametrize("config,scale,layout,cycles,dtmul", [
    ("C2", 33, (2, 2, 2), 25, 4.0),
    ("C5", 20, (2, 1, 1), 25, 4.0),
    ("C1", 0, (2, 2, 1), 20, 0.25),
    ("C4", 65, (2, 2, 2), 10, 4.0),
])
def test_local_comm_equals_single_block_and_oracle(config, scale, layout, cycles, dtmul):
    cfg = L.make_config(config, scale=scale or None, nranks=int(np.prod(layout)))
    cfg["dt"] *= dtmul                                # more hand-offs per interval
    g = cfg["grid"]
    stride = 2 if config == "C4" else cfg["stride"]
    sl = global_slices(cfg, cycles)
    blocks, res, stats = run_local(cfg, layout, [sl], stride)
    whole = L.Block(0, (0, 0, 0), (0, 0, 0), g.nodes)
    single = gpu_block(cfg, whole, sl, stride)
    got = assemble(g, blocks, res[0], stride)
    for a, b in zip(got, single[:3]):
        assert np.array_equal(a, b)                   # bitwise decomposition invariance
    orc = oracle.run_interval(g, (0, 0, 0), g.nodes, stride, sl, cfg["dt"], mode=oracle.BTO,
                              faces=((0, 0, 0), g.nodes))
    compare(cfg, orc, *single[:3], label=f"{config} single/comm")
    sent = sum(s["sent"] for s in stats[0])
    recv = sum(s["received"] for s in stats[0])
    assert sent > 0 and recv > 0
    assert all(s["device_error"] == 0 for s in stats[0])


def test_local_comm_several_intervals_return_to_origin():
    """Three intervals on one group: the write cycle returns every particle to
    its origin block, the group reseeds after its last extract, and each
    interval equals a fresh single-block run bitwise."""
    cfg = L.make_config("C2", scale=29, nranks=8)
    cfg["dt"] *= 4.0
    g = cfg["grid"]
    I = 12
    allsl = global_slices(cfg, 3 * I)
    per = [allsl[i * I:(i + 1) * I + 1] for i in range(3)]
    blocks, res, _ = run_local(cfg, (2, 2, 2), per, 1, streams=True)     # blocks run concurrently
    whole = L.Block(0, (0, 0, 0), (0, 0, 0), g.nodes)
    for it in range(3):
        single = gpu_block(cfg, whole, per[it], 1)
        got = assemble(g, blocks, res[it], 1)
        for a, b in zip(got, single[:3]):
            assert np.array_equal(a, b), f"interval {it}"
        moved = np.abs(got[1] - got[0]).max()
        assert moved > 2 * min(g.spacing)              # particles crossed block faces


def test_local_comm_padded_rows_and_frozen_snapshot():
    cfg = L.make_config("C2", scale=33, nranks=8)
    cfg["dt"] *= 4.0
    sl = global_slices(cfg, 10)
    blocks, dense, _ = run_local(cfg, (2, 2, 2), [sl], 1)
    _, padded, _ = run_local(cfg, (2, 2, 2), [sl], 1, pad=3)
    for a, b in zip(dense[0], padded[0]):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    # frozen snapshot (v_t1 = v_t): equals the single block
    g = cfg["grid"]
    _, fz, _ = run_local(cfg, (2, 2, 2), [sl], 1, frozen=True)
    whole = L.Block(0, (0, 0, 0), (0, 0, 0), g.nodes)
    single = gpu_block(cfg, whole, sl, 1, same_tensor=True)
    for a, b in zip(assemble(g, blocks, fz[0], 1), single[:3]):
        assert np.array_equal(a, b)


def test_local_comm_mid_interval_reseed_drops_in_flight_particles():
    """lag_seed on every block in the middle of an interval discards the
    particles in flight: the next interval equals a fresh run bitwise."""
    cfg = L.make_config("C2", scale=25, nranks=8)
    cfg["dt"] *= 4.0
    g = cfg["grid"]
    sl = global_slices(cfg, 16)
    blocks, res, _ = run_local(cfg, (2, 2, 2), [sl[:9], sl[8:]], 1, reseed_mid=6)
    single = gpu_block(cfg, L.Block(0, (0, 0, 0), (0, 0, 0), g.nodes), sl[8:], 1)
    for a, b in zip(assemble(g, blocks, res[0], 1), single[:3]):
        assert np.array_equal(a, b)


def test_local_comm_errors():
    import torch
    import paper_2004_02003_b200 as P
    cfg = L.make_config("C2", scale=17, nranks=2)
    g = cfg["grid"]
    blocks = L.decompose(g, (2, 1, 1))
    s = torch.cuda.current_stream()
    cfgs = [P.make_config(3, g.nodes, g.origin, g.spacing, b.lo, b.hi, mode=P.LAG_COMM, ghost=1,
                          rank=b.rank, nranks=2, layout=(2, 1, 1), stream=s.cuda_stream,
                          exchange=P.LAG_XCHG_LOCAL) for b in blocks]
    # wrong rank order
    c0, c1 = P.Context(cfgs[0]), P.Context(cfgs[1])
    with pytest.raises(P.LagError) as e:
        P.lag_local_group([c1.ctx, c0.ctx])
    assert e.value.status == P.LAG_EINVAL
    with pytest.raises(P.LagError) as e:           # seed without a group
        c0.seed(1)
    assert e.value.status == P.LAG_ESTATE
    c0.close(); c1.close()
    grp = P.LocalGroup(cfgs)
    ns = grp.seed(1)
    vs = [torch.zeros(tuple(reversed(L.block_slice_extent(g, b, 1))) + (3,), device="cuda") for b in blocks]
    grp.blocks[0].advect(vs[0], vs[0], 0.01)
    with pytest.raises(P.LagError) as e:           # twice in one group cycle
        grp.blocks[0].advect(vs[0], vs[0], 0.01)
    assert e.value.status == P.LAG_ESTATE
    with pytest.raises(P.LagError) as e:           # host slice
        grp.blocks[1].advect(vs[1].cpu(), vs[1].cpu(), 0.01)
    assert e.value.status == P.LAG_EINVAL
    grp.blocks[1].advect(vs[1], vs[1], 0.01)        # completes the cycle
    out0 = [torch.empty((ns[0], 3), dtype=torch.float64, device="cuda") for _ in range(2)]
    grp.blocks[0].extract(out0[0], out0[1])
    with pytest.raises(P.LagError) as e:           # block 1 has not extracted yet
        grp.blocks[0].advect(vs[0], vs[0], 0.01)
    assert e.value.status == P.LAG_ESTATE
    with pytest.raises(P.LagError) as e:           # interval index out of order
        P.lag_extract(grp.blocks[1].ctx, 5)
    assert e.value.status == P.LAG_ESTATE
    grp.blocks[1].extract()
    grp.advect(vs, vs, 0.01)                        # the group reseeded: a new interval runs
    grp.close()


@pytest.mark.slow
def test_local_comm_c2_full_size():
    """configs[1] at full size on one GPU, in bench.py's launch configuration
    (8 blocks of 128^3, one stream per block, stride 1, one interval of 25
    cycles at the config's dt): the COMM group equals the single-block run
    bitwise, and 4096 sampled seeds of that run match the oracle."""
    cfg = L.make_config("C2")
    g = cfg["grid"]
    sl = global_slices(cfg, cfg["interval"])
    blocks, res, stats = run_local(cfg, cfg["layout"], [sl], 1, streams=True)
    assert sum(s["sent"] for s in stats[0]) > 0
    whole = L.Block(0, (0, 0, 0), (0, 0, 0), g.nodes)
    single = gpu_block(cfg, whole, sl, 1)
    got = assemble(g, blocks, res[0], 1)
    for a, b in zip(got, single[:3]):
        assert np.array_equal(a, b)
    gs = oracle.seeds(g, (0, 0, 0), g.nodes, 1)
    pick = np.unique(np.random.default_rng(11).choice(gs.shape[0], 4096, replace=False))
    orc = oracle.run_interval(g, (0, 0, 0), g.nodes, 1, sl, cfg["dt"], mode=oracle.BTO, g_seeds=gs[pick],
                              faces=((0, 0, 0), g.nodes))
    compare(cfg, orc, single[0][pick], single[1][pick], single[2][pick], label="C2 full single/comm")


def test_cuda_graph_replay_equals_direct_calls():
    """bench.py replays captured intervals (CUDA graphs): a captured interval
    (seed | cycles | asynchronous write cycle), replayed twice, gives the same
    flow maps as direct calls — for a BTO context and for a LAG_XCHG_LOCAL
    group with one stream per block."""
    import torch
    import paper_2004_02003_b200 as P
    cfg = L.make_config("C2", scale=33, nranks=8)
    cfg["dt"] *= 4.0
    g = cfg["grid"]
    I = 8
    sl = global_slices(cfg, I)
    blocks = L.decompose(g, cfg["layout"])
    direct = assemble(g, blocks, run_local(cfg, cfg["layout"], [sl], 1, streams=True)[1][0], 1)
    cap = torch.cuda.Stream()
    streams = [torch.cuda.Stream() for _ in blocks]
    cfgs = [P.make_config(3, g.nodes, g.origin, g.spacing, b.lo, b.hi, mode=P.LAG_COMM, ghost=1, rank=b.rank,
                          nranks=8, layout=cfg["layout"], stream=st.cuda_stream, exchange=P.LAG_XCHG_LOCAL)
            for b, st in zip(blocks, streams)]
    grp = P.LocalGroup(cfgs)
    ns = grp.seed(1)
    dev = [[torch.from_numpy(poisoned_block_slice(V, g, b, 1)).cuda() for b in blocks] for V in sl]
    outs = [(torch.empty((n, 3), dtype=torch.float64, device="cuda"), torch.empty((n, 3), dtype=torch.float64, device="cuda"),
             torch.empty((n,), dtype=torch.uint8, device="cuda")) for n in ns]
    torch.cuda.synchronize()

    def interval():
        ev = torch.cuda.Event()
        ev.record(cap)
        for st in streams:
            st.wait_event(ev)
        grp.seed(1)
        for k in range(I):
            grp.advect(dev[k], dev[k + 1], cfg["dt"])
        grp.extract(outs, flags=P.LAG_NO_RESEED | P.LAG_ASYNC)
        for st in streams:
            e = torch.cuda.Event()
            e.record(st)
            cap.wait_event(e)

    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=cap):
        interval()
    for _ in range(2):
        for o in outs:
            for x in o:
                x.fill_(0)
        torch.cuda.synchronize()
        gr.replay()
        torch.cuda.synchronize()
        got = assemble(g, blocks, [tuple(x.cpu().numpy() for x in o) for o in outs], 1)
        for a, b in zip(got, direct):
            assert np.array_equal(a, b)
    grp.close()
    # a BTO context: the captured interval equals direct calls
    b = L.Block(0, (0, 0, 0), (0, 0, 0), g.nodes)
    ref = gpu_block(cfg, b, sl, 1)
    ctx = P.Context(P.make_config(3, g.nodes, g.origin, g.spacing, b.lo, b.hi, stream=cap.cuda_stream))
    n = ctx.seed(1)
    d1 = [torch.from_numpy(np.ascontiguousarray(L.cut_block_slice(V, g, b, 0))).cuda() for V in sl]
    o = (torch.empty((n, 3), dtype=torch.float64, device="cuda"), torch.empty((n, 3), dtype=torch.float64, device="cuda"),
         torch.empty((n,), dtype=torch.uint8, device="cuda"))
    torch.cuda.synchronize()
    gr2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr2, stream=cap):
        ctx.seed(1)
        for k in range(I):
            ctx.advect(d1[k], d1[k + 1], cfg["dt"])
        ctx.extract(*o, flags=P.LAG_NO_RESEED | P.LAG_ASYNC)
    gr2.replay()
    torch.cuda.synchronize()
    for x, y in zip(o, ref[:3]):
        assert np.array_equal(x.cpu().numpy(), y)
    ctx.close()


def test_bto_padded_rows_equal_dense():
    """row_pitch_bytes: BTO on slices whose rows carry NaN
    padding nodes gives bitwise the dense result (padding is never read)."""
    import torch
    import paper_2004_02003_b200 as P
    cfg = L.make_config("C2", scale=29, nranks=8)
    g = cfg["grid"]
    sl = global_slices(cfg, 6)
    b = L.decompose(g, cfg["layout"])[3]
    ref = gpu_block(cfg, b, sl, 1)
    ext = L.block_slice_extent(g, b, 0)
    pad = 5
    dev = [torch.from_numpy(poisoned_block_slice(V, g, b, 0, pad)).cuda() for V in sl]
    ctx = P.Context(P.make_config(3, g.nodes, g.origin, g.spacing, b.lo, b.hi,
                                  stream=torch.cuda.current_stream().cuda_stream,
                                  row_pitch_bytes=(ext[0] + pad) * 12))
    n = ctx.seed(1)
    for k in range(len(dev) - 1):
        ctx.advect(dev[k], dev[k + 1], cfg["dt"])
    out = (torch.empty((n, 3), dtype=torch.float64, device="cuda"), torch.empty((n, 3), dtype=torch.float64, device="cuda"),
           torch.empty((n,), dtype=torch.uint8, device="cuda"))
    ctx.extract(*out)
    assert ctx.stats()["device_error"] == 0
    for x, y in zip(out, ref[:3]):
        assert np.array_equal(x.cpu().numpy(), y)
    ctx.close()


def test_local_comm_cfl_above_one_latches_ghost_error():
    """A stage sample more than one ghost layer outside the block (CFL >= 1)
    cannot be interpolated from the exchanged data: the particle stops and
    LAG_EGHOST is latched and reported by the write cycle (include/lag.h)."""
    import torch
    import paper_2004_02003_b200 as P
    cfg = L.make_config("C2", scale=17, nranks=2)
    cfg["dt"] *= 20.0                                    # CFL ~ 3 cells per cycle
    g = cfg["grid"]
    blocks = L.decompose(g, (2, 1, 1))
    sl = global_slices(cfg, 2)
    cfgs = [P.make_config(3, g.nodes, g.origin, g.spacing, b.lo, b.hi, mode=P.LAG_COMM, ghost=1, rank=b.rank,
                          nranks=2, layout=(2, 1, 1), stream=torch.cuda.current_stream().cuda_stream,
                          exchange=P.LAG_XCHG_LOCAL) for b in blocks]
    grp = P.LocalGroup(cfgs)
    grp.seed(1)
    dev = [[torch.from_numpy(poisoned_block_slice(V, g, b, 1)).cuda() for b in blocks] for V in sl]
    grp.advect(dev[0], dev[1], cfg["dt"])
    st = grp.stats()
    assert any(s["device_error"] == P.LAG_EGHOST for s in st)
    with pytest.raises(P.LagError) as e:
        for b in grp.blocks:
            b.extract()
    assert e.value.status == P.LAG_EGHOST
    grp.close()
