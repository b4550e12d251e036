"""Host-side cost of one lag_advect_cycle call (time the call returns, no
sync) vs the device period per cycle, for BTO (and COMM arms under torchrun).
  python scripts/host_overhead.py            (1 GPU, BTO)
  torchrun --nproc-per-node 2 scripts/host_overhead.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import lag_inputs as L  # noqa: E402
import paper_2004_02003_b200 as P  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    cfg = L.make_config("C5", nranks=world)
    arms = [("bto", P.LAG_BTO, 0)]
    if world > 1:
        arms += [("comm_nccl", P.LAG_COMM, 0), ("comm_peer", P.LAG_COMM, 1)]
    for name, mode, xch in arms:
        nid = bench.broadcast_bytes(P.lag_nccl_unique_id() if rank == 0 else None, world, rank) if world > 1 else None
        arm = bench.Arm(cfg, rank, world, mode, nccl_id=nid, exchange=xch)
        bench.run_arm(arm, 2, None)
        s = arm.stream
        host = []
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(arm.interval + 1)]
        arm.ctx.seed(arm.cfg["stride"])
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev[0].record(s)
        for c in range(arm.interval):
            t0 = time.perf_counter()
            arm.ctx.advect(arm.slices[c], arm.slices[c + 1], arm.cfg["dt"])
            host.append(time.perf_counter() - t0)
            ev[c + 1].record(s)
        torch.cuda.synchronize()
        per = [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(arm.interval)]
        host.sort()
        per.sort()
        print(f"rank {rank} {name}: host call median {1e6 * host[len(host) // 2]:.1f} us "
              f"(min {1e6 * host[0]:.1f}), device period median {per[len(per) // 2]:.1f} us", flush=True)
        arm.ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
