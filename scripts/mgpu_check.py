"""Multi-GPU parity check (launch with torchrun, one rank per GPU).

  torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/mgpu_check.py [config] [scale]

Per rank: one block of the layout (weak layout for C3/C5, 2x2x2-style split
otherwise).  Checks, on rank 0:
  * COMM (NCCL halo fill + particle hand-off + return-to-origin) flow maps of
    all ranks == the single-block GPU run of the whole domain, BITWISE
    (decomposition invariance);
  * COMM vs the fp64 oracle (global integration) within the north-star rule;
  * BTO per rank vs the oracle per block;
  * sent == received over all ranks, and >0 (the exchange really happened).
Prints one JSON line with the outcome; exit code 0 iff everything passed.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import lag_inputs as L  # noqa: E402
import paper_2004_02003_b200 as P  # noqa: E402


def run_block(cfg, block, layout, rank, world, mode, slices, stride, nccl_id=None, exchange=0,
              reseed_mid=None, second=False):
    g = cfg["grid"]
    ghost = 1 if mode == P.LAG_COMM else 0
    lo = [block.lo[a] - ghost if a < g.dim else 0 for a in range(3)]
    ext = L.block_slice_extent(g, block, ghost)
    bs = [np.array(L.cut_block_slice(V, g, block, ghost), dtype=np.float32) for V in slices]
    if ghost:
        # ghost layers arrive only through the exchange: poison them, so a
        # gather that runs before its halo is filled shows up as a latched
        # non-finite velocity (unused ghosts at global faces stay NaN)
        for b in bs:
            for ax in range(g.dim):
                idx = [slice(None)] * b.ndim
                nax = b.ndim - 2 - ax                 # arrays are [z][y][x][comp] (3-D) / [y][x][comp]
                for k in (0, b.shape[nax] - 1):
                    idx[nax] = k
                    b[tuple(idx)] = np.nan
    dev = [torch.from_numpy(np.ascontiguousarray(b)).cuda() for b in bs]
    s = torch.cuda.current_stream()
    pc = P.make_config(g.dim, g.nodes, g.origin, g.spacing, block.lo, block.hi, mode=mode,
                       ghost=ghost, device=torch.cuda.current_device(), rank=rank,
                       nranks=world if mode == P.LAG_COMM else 1,
                       layout=layout if mode == P.LAG_COMM else (1, 1, 1),
                       nccl_id=nccl_id, stream=s.cuda_stream, exchange=exchange)
    ctx = P.Context(pc)
    n = ctx.seed(stride)
    if reseed_mid:
        # a reseed in the middle of an interval (no write cycle): the hand-offs
        # in flight must be dropped, so the interval that follows is a fresh one
        for k in range(reseed_mid):
            ctx.advect(dev[k], dev[k + 1], cfg["dt"])
        n = ctx.seed(stride)
    if second:
        # a whole interval with its write cycle first (the last cycle's
        # hand-offs flushed, particles returned to their origin): the
        # interval that follows must equal a fresh context's
        for k in range(len(dev) - 1):
            ctx.advect(dev[k], dev[k + 1], cfg["dt"])
        o = [torch.empty((n, g.dim), dtype=torch.float64, device="cuda") for _ in range(2)]
        ctx.extract(o[0], o[1], torch.empty((n,), dtype=torch.uint8, device="cuda"), flags=P.LAG_NO_RESEED)
        n = ctx.seed(stride)
    for k in range(len(dev) - 1):
        ctx.advect(dev[k], dev[k + 1], cfg["dt"])
    start = torch.empty((n, g.dim), dtype=torch.float64, device="cuda")
    end = torch.empty_like(start)
    status = torch.empty((n,), dtype=torch.uint8, device="cuda")
    ctx.extract(start, end, status, flags=P.LAG_NO_RESEED)
    st_mid = ctx.stats()        # after extract: the last cycle's hand-offs were flushed
    ctx.close()
    return start.cpu().numpy(), end.cpu().numpy(), status.cpu().numpy(), st_mid


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "C2"
    scale = int(sys.argv[2]) if len(sys.argv) > 2 else 33
    ncyc = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    cfg = L.make_config(config, scale=scale or None, nranks=world)
    if config.upper() in ("C3", "C5"):
        layout = cfg["layout"]
    else:
        layout = L.layout_for(world, dim=cfg["grid"].dim)
    g = cfg["grid"]
    # more hand-offs per interval (the 2-D gyre already runs near CFL 1.5 in y)
    cfg["dt"] = cfg["dt"] * (0.25 if config.upper() == "C1" else 4.0)
    blocks = L.decompose(g, layout)
    me = blocks[rank]
    slices = [L.field_at_nodes(cfg["field"], g, k * cfg["dt"]) for k in range(ncyc + 1)]
    stride = cfg["stride"] if config.upper() != "C4" else 2
    obj = [P.lag_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    t0 = time.time()
    comm = run_block(cfg, me, layout, rank, world, P.LAG_COMM, slices, stride, nccl_id=obj[0])
    obj2 = [P.lag_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj2, src=0)
    peer = run_block(cfg, me, layout, rank, world, P.LAG_COMM, slices, stride, nccl_id=obj2[0],
                     exchange=P.LAG_XCHG_PEER)
    obj3 = [P.lag_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj3, src=0)
    ovl = run_block(cfg, me, layout, rank, world, P.LAG_COMM, slices, stride, nccl_id=obj3[0],
                    exchange=P.LAG_XCHG_PEER_OVERLAP)
    obj4 = [P.lag_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj4, src=0)
    rsd = run_block(cfg, me, layout, rank, world, P.LAG_COMM, slices, stride, nccl_id=obj4[0],
                    exchange=P.LAG_XCHG_PEER, reseed_mid=5)
    sec = []
    for xch in (P.LAG_XCHG_PEER, P.LAG_XCHG_PEER_OVERLAP):
        o5 = [P.lag_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(o5, src=0)
        sec.append(run_block(cfg, me, layout, rank, world, P.LAG_COMM, slices, stride, nccl_id=o5[0],
                             exchange=xch, second=True))
    bto = run_block(cfg, me, layout, rank, world, P.LAG_BTO, slices, stride)
    sec_all = []
    for x in sec:
        xa = [None] * world
        dist.all_gather_object(xa, x)
        sec_all.append(xa)
    comm_all = [None] * world
    bto_all = [None] * world
    peer_all = [None] * world
    dist.all_gather_object(comm_all, comm)
    dist.all_gather_object(peer_all, peer)
    dist.all_gather_object(bto_all, bto)
    ovl_all = [None] * world
    dist.all_gather_object(ovl_all, ovl)
    rsd_all = [None] * world
    dist.all_gather_object(rsd_all, rsd)
    ok = True
    report = dict(config=config, scale=scale, world=world, layout=list(layout), cycles=ncyc)
    if rank == 0:
        import oracle
        from helpers import compare
        whole = L.Block(0, (0, 0, 0), (0, 0, 0), g.nodes)
        single = run_block(cfg, whole, (1, 1, 1), 0, 1, P.LAG_BTO, slices, stride)
        gs = oracle.seeds(g, (0, 0, 0), g.nodes, stride)
        key = {tuple(x): i for i, x in enumerate(gs.tolist())}
        mism = 0
        sent = sum(int(c[3]["sent"]) for c in comm_all)
        recv = sum(int(c[3]["received"]) for c in comm_all)
        for b, c in zip(blocks, comm_all):
            idx = np.array([key[tuple(x)] for x in oracle.seeds(g, b.lo, b.hi, stride).tolist()])
            for arr_c, arr_s in zip(c[:3], single[:3]):
                if not np.array_equal(arr_c, arr_s[idx]):
                    mism += 1
        report["comm_vs_single_bitwise_mismatching_arrays"] = mism
        pm = sum(int(not np.array_equal(x, y)) for c, pz in zip(comm_all, peer_all) for x, y in zip(c[:3], pz[:3]))
        psent = sum(int(c[3]["sent"]) for c in peer_all)
        precv = sum(int(c[3]["received"]) for c in peer_all)
        report["peer_vs_nccl_bitwise_mismatching_arrays"] = pm
        report["peer_sent"] = psent
        report["peer_received"] = precv
        ok &= pm == 0 and psent == precv and psent == sent
        om = sum(int(not np.array_equal(x, y)) for c, oz in zip(comm_all, ovl_all) for x, y in zip(c[:3], oz[:3]))
        report["overlap_vs_nccl_bitwise_mismatching_arrays"] = om
        report["overlap_sent"] = sum(int(c[3]["sent"]) for c in ovl_all)
        ok &= om == 0 and report["overlap_sent"] == sent
        rm = sum(int(not np.array_equal(x, y)) for c, rz in zip(peer_all, rsd_all) for x, y in zip(c[:3], rz[:3]))
        report["peer_mid_reseed_vs_fresh_mismatching_arrays"] = rm
        ok &= rm == 0
        # second interval after a write cycle == the first interval of a fresh context
        sm = [sum(int(not np.array_equal(x, y)) for c, z in zip(peer_all, xa) for x, y in zip(c[:3], z[:3]))
              for xa in sec_all]
        report["second_interval_vs_fresh_mismatching_arrays"] = {"peer": sm[0], "peer_overlap": sm[1]}
        ok &= sum(sm) == 0
        report["sent"] = sent
        report["received"] = recv
        ok &= mism == 0 and sent == recv and sent > 0
        # oracle: global COMM (decomposition-free) and per-block BTO
        orc_c = oracle.run_interval(g, (0, 0, 0), g.nodes, stride, slices, cfg["dt"], mode=oracle.BTO,
                                    faces=((0, 0, 0), g.nodes))
        report["comm_vs_oracle"] = compare(cfg, orc_c, *single[:3], label="single/comm")
        for b, bt in zip(blocks, bto_all):
            orc_b = oracle.run_interval(g, b.lo, b.hi, stride, slices, cfg["dt"], faces=(b.lo, b.hi))
            r = compare(cfg, orc_b, *bt[:3], label=f"bto rank {b.rank}")
            report.setdefault("bto_term", 0)
            report["bto_term"] += r["term"]
        report["ok"] = bool(ok)
        report["seconds"] = time.time() - t0
        print(json.dumps(report), flush=True)
    okt = torch.tensor([1 if ok else 0])
    dist.broadcast(okt, src=0)
    dist.destroy_process_group()
    sys.exit(0 if okt.item() == 1 else 1)


if __name__ == "__main__":
    main()
