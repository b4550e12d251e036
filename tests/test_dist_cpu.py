"""World-size-2 gloo test (CPU) of the multi-rank host logic of bench.py:
max-over-ranks timing, sums of particle-steps, broadcast of the NCCL unique-id
bytes, and the weak-scaling block layout each rank picks."""
import os
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import lag_inputs as L
    mx = bench.allreduce_max(float(rank + 1) * 1.5, world)
    sm = bench.allreduce_sum(float(rank + 1), world)
    idb = bench.broadcast_bytes(b"\x07" * 128 if rank == 0 else None, world, rank)
    cfg = L.make_config("C5", nranks=world)
    blk = L.decompose(cfg["grid"], cfg["layout"])[rank]
    q.put((rank, mx, sm, idb, blk.lo, blk.hi, cfg["layout"]))
    dist.destroy_process_group()


def test_two_rank_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29511
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, sm, idb, lo, hi, lay in res:
        assert mx == 3.0 and sm == 3.0 and idb == b"\x07" * 128
        assert lay == (2, 1, 1)
    assert res[0][4] == (0, 0, 0) and res[0][5] == (128, 128, 128)
    assert res[1][4] == (128, 0, 0) and res[1][5] == (256, 128, 128)
