"""Short C5 run for ncu: seed + a few advect cycles of the bench's workload
(same launch configuration as bench.py), no timing of its own."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import lag_inputs as L  # noqa: E402
import paper_2004_02003_b200 as P  # noqa: E402


def main(config="C5", cycles=8):
    cycles = int(cycles)
    cfg = L.make_config(config)
    g = cfg["grid"]
    b = L.decompose(g, cfg["layout"])[0]
    ext = L.block_slice_extent(g, b, 0)
    hi = [b.lo[a] + ext[a] for a in range(3)]
    sl = [L.field_at_nodes(cfg["field"], g, k * cfg["dt"], lo=b.lo, hi=hi, device="cuda",
                           backend="torch").contiguous() for k in range(cycles + 1)]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    ctx = P.Context(P.make_config(g.dim, g.nodes, g.origin, g.spacing, b.lo, b.hi,
                                  stream=s.cuda_stream))
    ctx.seed(cfg["stride"])
    for c in range(cycles):
        flush.zero_()
        ctx.advect(sl[c], sl[c + 1], cfg["dt"])
    torch.cuda.synchronize()
    print("ok", ctx.stats())
    ctx.close()


if __name__ == "__main__":
    main(*(sys.argv[1:3] or ["C5"]))
