"""C3 phase timing: grid 4096^2, centre marked, uniform psi0, T = 16707 steps
with p(marked) every step and distributions every 4096 steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2406_08186_b200 as q
from paper_2406_08186_b200 import coined as CO

nx = 4096
eng = q.init_engine("b200")
g = q.graphs.grid(nx, nx)
c = nx // 2 + nx * (nx // 2)
spec = q.CoinedSpec(g, "flipflop", "grover", frozenset({c}), "minus_identity")
arcs = 4 * nx * nx
T = 16707
psi = q.WalkState(q.graphs.arc_basis(g), np.full(arcs, 2.0 ** -13, dtype=np.complex128))
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    basis, x = CO._upload_initial(eng, spec, psi)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = CO._LatticeRunner(eng, spec)
    r.load(x)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    tr = torch.empty((T + 1, 1), dtype=torch.float64, device="cuda")
    r.advance(T, tr, (c,))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    del r, x
    t4 = time.perf_counter()
    trace, dists = CO.search_trace(eng, spec, T, psi, 4096)
    t5 = time.perf_counter()
    print(f"upload+norm {1e3*(t1-t0):.1f} ms, runner+planes {1e3*(t2-t1):.1f} ms, "
          f"{T} traced steps {1e3*(t3-t2):.1f} ms ({1e6*(t3-t2)/T:.1f} us/step); "
          f"search_trace total {1e3*(t5-t4):.1f} ms")
q.stop_engine(eng)
