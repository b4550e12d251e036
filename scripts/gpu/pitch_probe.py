"""C5 per-cycle advect time vs slice layout: ghost layers and row pitch
(BTO and COMM at N=1).  L2 flushed before every cycle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import lag_inputs as L
import paper_2004_02003_b200 as P

cfg = L.make_config("C5")
g = cfg["grid"]; b = L.decompose(g, cfg["layout"])[0]; I = cfg["interval"]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()

def run(mode, ghost, pitch_nodes=None, reps=3):
    ext = L.block_slice_extent(g, b, ghost)
    lo = [b.lo[a] - ghost for a in range(3)]
    hi = [lo[a] + ext[a] for a in range(3)]
    sl = []
    for k in range(I + 1):
        v = L.field_at_nodes(cfg["field"], g, k * cfg["dt"], lo=lo, hi=hi, device="cuda", backend="torch")
        if pitch_nodes:
            p = torch.zeros((ext[2], ext[1], pitch_nodes, 3), device="cuda")
            p[:, :, :ext[0]] = v
            v = p
        sl.append(v.contiguous())
    pc = P.make_config(3, g.nodes, g.origin, g.spacing, b.lo, b.hi, mode=mode, ghost=ghost,
                       stream=s.cuda_stream, row_pitch_bytes=12 * pitch_nodes if pitch_nodes else 0)
    ctx = P.Context(pc)
    ms = []
    for it in range(reps + 1):
        ctx.seed(1)
        for c in range(I):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); ctx.advect(sl[c], sl[c + 1], cfg["dt"]); e1.record(s)
            if it:
                ms.append((e0, e1))
    torch.cuda.synchronize()
    t = [a.elapsed_time(b_) * 1e3 for a, b_ in ms]
    ctx.close()
    return sum(t) / len(t)

for mode, ghost, pitch in [(0, 0, None), (0, 0, 129), (0, 0, 132), (0, 1, None), (0, 1, 136), (1, 1, None), (1, 1, 136), (0, 0, None)]:
    print(f"mode {'COMM' if mode else 'BTO'} ghost {ghost} pitch {pitch or 'dense'}: {run(mode, ghost, pitch):.1f} us/cycle", flush=True)
