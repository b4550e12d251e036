"""Per-cycle advect timing for kernel experiments (CUDA events, L2 flushed
before every cycle).  LAG_LIB=<path> selects a library variant.
usage: python scripts/time_advect.py [config] [intervals]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import lag_inputs as L  # noqa: E402
import paper_2004_02003_b200 as P  # noqa: E402


def main(config="C5", intervals=3, stride=None, flush_l2=True, frozen=False):
    cfg = L.make_config(config)
    g = cfg["grid"]
    b = L.decompose(g, cfg["layout"])[0]
    ext = L.block_slice_extent(g, b, 0)
    hi = [b.lo[a] + ext[a] for a in range(3)]
    I = cfg["interval"]
    sl = [L.field_at_nodes(cfg["field"], g, k * cfg["dt"], lo=b.lo, hi=hi, device="cuda",
                           backend="torch").contiguous() for k in range(I + 1)]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    ctx = P.Context(P.make_config(g.dim, g.nodes, g.origin, g.spacing, b.lo, b.hi, stream=s.cuda_stream))
    times = []
    for it in range(intervals + 1):
        ctx.seed(stride or cfg["stride"])
        for c in range(I):
            if flush_l2:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ctx.advect(sl[c], sl[c] if frozen else sl[c + 1], cfg["dt"])
            e1.record(s)
            if it > 0 or intervals == 0:
                times.append((e0, e1))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in times]
    st = ctx.stats()
    us = 1e3 * sum(ms) / len(ms)
    print(f"{os.environ.get('LAG_LIB', 'default')}: {config} {'flushed' if flush_l2 else 'warm-L2'}{' frozen' if frozen else ''} {us:.1f} us/cycle "
          f"(first {1e3 * ms[0]:.1f}, last {1e3 * ms[I - 1]:.1f}), "
          f"{st['particle_steps'] / (intervals + 1) / I / us * 1e-3:.2f} G p-steps/s")
    ctx.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C5", int(sys.argv[2]) if len(sys.argv) > 2 else 3,
         flush_l2="--warm" not in sys.argv, frozen="--frozen" in sys.argv)
