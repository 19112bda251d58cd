"""CSR Taylor term timing: CTQW on grid(nx, nx) (degree 4, H built on the
device as CSR), gamma = 0.25, marked {0}; one evolve of t = 1."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2406_08186_b200 as q
from paper_2406_08186_b200 import ctqw as CT

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
eng = q.init_engine("b200")
cs = q.CtqwSpec(q.graphs.grid(nx, nx), 0.25, 1.0, frozenset({0}))
op = CT._Operator(eng, cs)
n = nx * nx
x = torch.full((n,), 1.0 / np.sqrt(n), dtype=torch.complex128, device="cuda")
nnz = 4 * n + 1
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    terms = op.evolve(x, 1.0, 1e-12)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    per = dt / sum(terms)
    b = 64 * n + nnz * 20 + 8 * n   # term r/w + acc RMW + values/cols + row offsets
    print(f"grid {nx}^2 CSR H: {dt*1e3:.2f} ms, terms {terms}, {per*1e6:.1f} us/term, "
          f"{b / per / 1e9:.0f} GB/s algorithmic ({b / n:.0f} B/vertex-term)")
q.stop_engine(eng)
