"""Device time per coined step of the torus path (runner.advance), no checks:
for kernel experiments.  usage: time_lattice.py [nx] [steps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_08186_b200 as q
from paper_2406_08186_b200 import coined as CO
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 240
eng = q.init_engine("b200")
spec = q.CoinedSpec(q.graphs.grid(nx, nx))
r = CO._LatticeRunner(eng, spec)
r.a.fill_(1.0 / np.sqrt(4 * nx * nx))
for _ in range(3):
    r.advance(steps)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    r.advance(steps)
b.record()
torch.cuda.synchronize()
us = a.elapsed_time(b) * 1e3 / (5 * steps)
print(f"nx {nx}: {us:.2f} us/step, {4 * nx * nx / us / 1e3:.1f} G arc-updates/s")
