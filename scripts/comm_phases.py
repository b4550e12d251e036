"""Per-phase device time of one lag_advect_cycle (LAG_PHASE_TIMING=1):
pre-advect exchange, advect kernel, post-advect signal — BTO and COMM over
both transports, C5 per GPU, L2 flushed before every cycle (as bench.py).
  torchrun --nproc-per-node N scripts/comm_phases.py [--no-flush]"""
import json
import os
import sys

os.environ["LAG_PHASE_TIMING"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import lag_inputs as L  # noqa: E402
import paper_2004_02003_b200 as P  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    cfg = L.make_config("C5", nranks=world)
    flush = None if "--no-flush" in sys.argv else torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    out = {}
    for name, mode, xch in [("bto", P.LAG_BTO, 0), ("comm_nccl", P.LAG_COMM, P.LAG_XCHG_NCCL),
                            ("comm_peer", P.LAG_COMM, P.LAG_XCHG_PEER),
                            ("comm_peer_overlap", P.LAG_COMM, P.LAG_XCHG_PEER_OVERLAP)]:
        nid = bench.broadcast_bytes(P.lag_nccl_unique_id() if rank == 0 else None, world, rank)
        arm = bench.Arm(cfg, rank, world, mode, nccl_id=nid, exchange=xch)
        bench.run_arm(arm, 2, flush)
        st0 = arm.ctx.stats()
        t_adv, t_other, ps = bench.run_arm(arm, 4, flush)
        st1 = arm.ctx.stats()
        cyc = 4 * arm.interval
        ph = [(b - a) * 1e3 / cyc for a, b in zip(st0["phase_ms"], st1["phase_ms"])]
        if xch == P.LAG_XCHG_PEER_OVERLAP and mode == P.LAG_COMM:   # phases of the fused cycle
            r = {"us_per_cycle_event": 1e3 * sum(t_adv) / cyc, "snapshot_us": ph[0],
                 "pass1_exchange_and_ghost_free_us": ph[1], "pass2_deferred_and_arrivals_us": ph[2],
                 "sent": st1["sent"]}
        else:
            r = {"us_per_cycle_event": 1e3 * sum(t_adv) / cyc, "pre_exchange_us": ph[0], "advect_us": ph[1],
                 "post_us": ph[2], "sent": st1["sent"]}
        allr = [None] * world
        dist.all_gather_object(allr, r)
        out[name] = {k: max(x[k] for x in allr) for k in r}
        arm.ctx.close()
    if rank == 0:
        print(json.dumps({"world": world, "flush": flush is not None, "max_over_ranks": out}, indent=1))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
