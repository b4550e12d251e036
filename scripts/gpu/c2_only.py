import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
print(json.dumps(bench.measure_c2(int(sys.argv[1]) if len(sys.argv) > 1 else 3, 2, flush), indent=1))
