"""Time lag_gridfill on a BTO-like hole pattern (bands next to block faces of
a 2x2x2 decomposition) on a dims^3 lattice; prints µs per call and effective
GB/s over the algorithmic bytes (read values+valid once, write out+filled)."""
import sys
import numpy as np
import torch
import paper_2004_02003_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
w = int(sys.argv[2]) if len(sys.argv) > 2 else 3          # hole band half-width (seeds)
dims = (n, n, n)
x = torch.arange(n, device="cuda")
near = ((x - n // 2).abs() < w)
ok = ~(near[None, None, :] | near[None, :, None] | near[:, None, None])
valid = ok.reshape(-1).to(torch.uint8).contiguous()
vals = torch.randn((n ** 3, 3), dtype=torch.float64, device="cuda")
out = torch.empty_like(vals)
filled = torch.empty_like(valid)
for _ in range(3):
    P.lag_gridfill(vals, valid, dims, out, filled)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    P.lag_gridfill(vals, valid, dims, out, filled)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
byts = n ** 3 * (3 * 8 * 2 + 2)
print(f"gridfill {n}^3 holes={int((valid == 0).sum())} {us:.1f} us/call "
      f"(incl. sync) {byts / us / 1e3:.1f} GB/s algorithmic")
