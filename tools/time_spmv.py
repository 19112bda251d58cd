"""Device time of one CSR SpMV with the device-built U of grid nx^2 (K1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_08186_b200 as q
from paper_2406_08186_b200 import coined as CO
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
eng = q.init_engine("b200")
g = q.graphs.grid(nx, nx)
u = CO.device_operator(eng, g, "flipflop")
n = u.n_rows
xa = torch.full((n,), 1.0 / np.sqrt(n), dtype=torch.complex128, device="cuda")
xb = torch.empty_like(xa)
for _ in range(5):
    q.backend.spmv_device(eng, u, xa, xb)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    q.backend.spmv_device(eng, u, xa, xb)
b.record()
torch.cuda.synchronize()
us = a.elapsed_time(b) * 1e3 / 50
print(f"nx {nx}: {us:.1f} us/spmv, {120 * n / us / 1e3:.0f} GB/s (120 B/arc)")
