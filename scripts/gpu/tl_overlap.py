"""Timeline of the overlapped COMM cycle (LAG_XCHG_PEER_OVERLAP) from the
liblag_TL2.so build (scripts/gpu/tl_build2.py), C5 at N ranks.
  LAG_LIB=paper_2004_02003_b200/liblag_TL2.so torchrun --nproc-per-node 2 scripts/gpu/tl_overlap.py"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import lag_inputs as L  # noqa: E402
import paper_2004_02003_b200 as P  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    lib = ctypes.CDLL(os.environ["LAG_LIB"])
    cfg = L.make_config("C5", nranks=world)
    flushbuf = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    nid = bench.broadcast_bytes(P.lag_nccl_unique_id() if rank == 0 else None, world, rank)
    arm = bench.Arm(cfg, rank, world, P.LAG_COMM, nccl_id=nid, exchange=P.LAG_XCHG_PEER_OVERLAP)
    res = {}
    for fl in ("flush", "noflush"):
        bench.run_arm(arm, 2, flushbuf if fl == "flush" else None)
        torch.cuda.synchronize()
        a = np.zeros(64 * 16, dtype=np.uint64)
        assert lib.lag_tl2_read(a.ctypes.data_as(ctypes.c_void_p)) == 0
        t = a.reshape(64, 16).astype(np.int64)[: arm.interval]
        rows = []
        for c in range(1, arm.interval):
            r = t[c]
            p1 = max(r[1], r[2])
            nxt = t[c + 1][0] if c + 1 < arm.interval else 0
            rows.append([(r[1] - r[0]) / 1e3, (r[5] - r[0]) / 1e3, (r[2] - r[0]) / 1e3, (r[3] - p1) / 1e3,
                         (r[4] - r[3]) / 1e3, ((nxt - r[4]) / 1e3) if nxt else float("nan")])
        med = np.nanmedian(np.array(rows), axis=0).tolist()
        allr = [None] * world
        dist.all_gather_object(allr, med)
        res[fl] = allr
    arm.ctx.close()
    if rank == 0:
        print("median us per cycle [exchange CTAs end, pass-1 advect start, pass-1 advect end, gap to pass 2, pass 2, gap to next pass 1] per rank (from pass-1 entry)")
        print(json.dumps(res, indent=1))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
