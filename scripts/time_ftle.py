"""Time lag_ftle on an n^3 lattice of a smooth random map; prints µs per call
(kernel + launch + sync) and GB/s over the algorithmic bytes (each end
position read once, 24 B, + 8 B written per node)."""
import sys
import torch
import paper_2004_02003_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dims = (n, n, n)
ends = torch.rand((n ** 3, 3), dtype=torch.float64, device="cuda")
out = torch.empty((n ** 3,), dtype=torch.float64, device="cuda")
for _ in range(3):
    P.lag_ftle(ends, dims, (0.1, 0.1, 0.1), 1.0, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    P.lag_ftle(ends, dims, (0.1, 0.1, 0.1), 1.0, out)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
print(f"ftle {n}^3 {us:.1f} us/call {n ** 3 * 32 / us / 1e3:.1f} GB/s algorithmic")
