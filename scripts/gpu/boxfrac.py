import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import lag_inputs as L
import paper_2004_02003_b200 as P
for config in ("C5", "C3"):
    cfg = L.make_config(config)
    g = cfg["grid"]; b = L.decompose(g, cfg["layout"])[0]
    ext = L.block_slice_extent(g, b, 0); hi = [b.lo[a] + ext[a] for a in range(3)]
    I = cfg["interval"]
    sl = [L.field_at_nodes(cfg["field"], g, k * cfg["dt"], lo=b.lo, hi=hi, device="cuda", backend="torch").contiguous() for k in range(I + 1)]
    ctx = P.Context(P.make_config(3, g.nodes, g.origin, g.spacing, b.lo, b.hi, stream=torch.cuda.current_stream().cuda_stream))
    n = ctx.seed(cfg["stride"])
    prev = 0
    row = []
    for c in range(I):
        ctx.advect(sl[c], sl[c + 1], cfg["dt"])
        st = ctx.stats()
        boxed = st["phase_ms"][2]
        row.append(round((boxed - prev) / ((n + 31) // 32), 3))
        prev = boxed
    print(config, "box-staged fraction of tiles per cycle:", row)
    ctx.close()
