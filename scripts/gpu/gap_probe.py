"""Kernel-to-kernel gaps on one GPU (experiment; liblag_TL.so variant):
stamps of %globaltimer at CTA 0 entry (5) and the last warp exit (10) of
(a) back-to-back BTO advect launches of C5, (b) the same captured in a CUDA
graph, (c) an empty kernel of the same grid.
  LAG_LIB=paper_2004_02003_b200/liblag_TL.so python scripts/gpu/gap_probe.py"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import lag_inputs as L  # noqa: E402
import paper_2004_02003_b200 as P  # noqa: E402


def read(lib):
    a = np.zeros(1024 * 16, dtype=np.uint64)
    assert lib.lag_tl_read_api(a.ctypes.data_as(ctypes.c_void_p)) == 0
    return a.reshape(1024, 16).astype(np.int64)


def gaps(t, lo, n):
    adv = [(t[lo + i][10] - t[lo + i][5]) / 1e3 for i in range(n)]
    gap = [(t[lo + i + 1][5] - t[lo + i][10]) / 1e3 for i in range(n - 1)]
    return {"kernel_us_med": float(np.median(adv)), "gap_us_med": float(np.median(gap)),
            "gap_us": [round(g, 2) for g in gap[:10]]}


def main():
    lib = ctypes.CDLL(os.environ["LAG_LIB"])
    torch.cuda.set_device(0)
    cfg = L.make_config("C5", nranks=1)
    arm = bench.Arm(cfg, 0, 1, P.LAG_BTO)
    s = arm.stream
    out = {}
    bench.run_arm(arm, 2, None)
    # (a) stream launches
    with torch.cuda.stream(s):
        arm.ctx.seed(cfg["stride"])
        for c in range(arm.interval):
            arm.ctx.advect(arm.slices[c], arm.slices[c + 1], cfg["dt"])
    torch.cuda.synchronize()
    out["stream"] = gaps(read(lib), 512, arm.interval)
    # (b) graph of one interval's cycles (a context on a capture stream)
    gs = torch.cuda.Stream()
    gr = cfg["grid"]
    ctx = P.Context(P.make_config(gr.dim, gr.nodes, gr.origin, gr.spacing, (0, 0, 0), gr.nodes, mode=P.LAG_BTO,
                                  stream=gs.cuda_stream))
    g = torch.cuda.CUDAGraph()
    ctx.seed(cfg["stride"])
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=gs):
        for c in range(arm.interval):
            ctx.advect(arm.slices[c], arm.slices[c + 1], cfg["dt"])
    torch.cuda.synchronize()
    for _ in range(2):
        ctx.seed(cfg["stride"])
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
    out["graph"] = gaps(read(lib), 512, arm.interval)
    # (d) bench conditions: L2 flush before every cycle, one event pair per cycle
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for fl in (flush, None):
        ev = []
        with torch.cuda.stream(s):
            arm.ctx.seed(cfg["stride"])
            for c in range(arm.interval):
                if fl is not None:
                    fl.zero_()
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(s)
                arm.ctx.advect(arm.slices[c], arm.slices[c + 1], cfg["dt"])
                a1.record(s)
                ev.append((a0, a1))
        torch.cuda.synchronize()
        t = read(lib)
        r = gaps(t, 512, arm.interval)
        r["event_us_med"] = float(np.median([a.elapsed_time(b) * 1e3 for a, b in ev]))
        r["event_us"] = [round(a.elapsed_time(b) * 1e3, 2) for a, b in ev[:10]]
        r["kernel_us"] = [round((t[512 + i][10] - t[512 + i][5]) / 1e3, 2) for i in range(10)]
        out["events_flush" if fl is not None else "events_noflush"] = r
    # (c) empty kernels, same grid
    blocks = 148 * 4
    lib.lag_tl_empty(ctypes.c_int(50), ctypes.c_int(blocks), ctypes.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    out["empty_592x128"] = gaps(read(lib), 600, 50)
    lib.lag_tl_empty(ctypes.c_int(50), ctypes.c_int(1), ctypes.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    out["empty_1x128"] = gaps(read(lib), 600, 50)
    print(json.dumps(out, indent=1))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "gap_probe.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
