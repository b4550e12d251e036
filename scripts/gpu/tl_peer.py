"""Device timeline of the peer-transport COMM cycle (experiment; needs the
liblag_TL.so variant built by /tmp/tl_subs.py-style substitutions that stamp
%globaltimer at: exchange entry (0), halo signalled (1), wait done (2), ghost
pulled (3), appended (4), advect entry (5), advect's last-warp signal (6)).
  LAG_LIB=paper_2004_02003_b200/liblag_TL.so torchrun --nproc-per-node 2 scripts/gpu/tl_peer.py"""
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


def read(lib):
    a = np.zeros(1024 * 16, dtype=np.uint64)
    b = np.zeros(1024 * 16, dtype=np.uint64)
    assert lib.lag_tl_read_api(a.ctypes.data_as(ctypes.c_void_p)) == 0
    assert lib.lag_tl_read_peer(b.ctypes.data_as(ctypes.c_void_p)) == 0
    return np.maximum(a, b).reshape(1024, 16)       # stamps live in one of the two copies


def host_probe(arm, P, n=3):
    """host enqueue time per advect call (no sync inside the interval) and
    wall time per cycle including the device drain"""
    import time
    out = []
    for _ in range(n):
        arm.ctx.seed(arm.cfg["stride"])
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for c in range(arm.interval):
            arm.ctx.advect(arm.slices[c], arm.slices[c + 1], arm.cfg["dt"])
        t1 = time.perf_counter()
        arm.ctx.extract(arm.start, arm.end, arm.status, flags=P.LAG_NO_RESEED | P.LAG_ASYNC)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        out.append((1e6 * (t1 - t0) / arm.interval, 1e6 * (t2 - t0) / arm.interval))
    return out


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    lib = ctypes.CDLL(os.environ["LAG_LIB"])
    cfg = L.make_config("C5", nranks=world)
    flushbuf = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    res = {}
    for xname, xch in [("peer", P.LAG_XCHG_PEER), ("nccl", P.LAG_XCHG_NCCL)]:
        nid = bench.broadcast_bytes(P.lag_nccl_unique_id() if rank == 0 else None, world, rank)
        arm = bench.Arm(cfg, rank, world, P.LAG_COMM, nccl_id=nid, exchange=xch)
        allr = [None] * world
        dist.all_gather_object(allr, host_probe(arm, P))
        res[f"{xname}_host"] = allr
        for fl in ("flush", "noflush"):
            bench.run_arm(arm, 1, flushbuf if fl == "flush" else None)
            torch.cuda.synchronize()
            before = read(lib)
            t_adv, _, _ = bench.run_arm(arm, 2, flushbuf if fl == "flush" else None)
            torch.cuda.synchronize()
            after = read(lib)
            rows = np.nonzero((after != before).any(axis=1))[0]
            tl = {int(r): [int(v) for v in after[r]] for r in rows}
            allr = [None] * world
            dist.all_gather_object(allr, {"tl": tl, "us_per_cycle": 1e3 * sum(t_adv) / (2 * arm.interval)})
            res[f"{xname}_{fl}"] = allr
        arm.ctx.close()
    arm = bench.Arm(cfg, rank, world, P.LAG_BTO)
    bench.run_arm(arm, 1, None)
    bench.run_arm(arm, 1, None)
    torch.cuda.synchronize()
    allr = [None] * world
    dist.all_gather_object(allr, {"tl": {int(r): [int(v) for v in read(lib)[r]] for r in range(512, 512 + arm.interval)}})
    res["bto_tl"] = allr
    allr = [None] * world
    dist.all_gather_object(allr, host_probe(arm, P))
    res["bto_host"] = allr
    arm.ctx.close()
    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        json.dump(res, open(os.path.join(ROOT, "gpurun_out", f"tl_peer_n{world}.json"), "w"))
        for k, allr in res.items():
            if k.endswith("_host"):
                print(k, "host us/call, wall us/cycle", allr)
            else:
                print(k, "us/cycle", [round(r["us_per_cycle"], 1) for r in allr])
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
