"""C3 first-call timing in a fresh process (what bench.py's c3 line sees):
search_trace on grid 4096^2, centre marked, uniform psi0, 16,707 steps,
distributions every 4096 steps.  usage: c3_first_call.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_08186_b200 as q
from paper_2406_08186_b200 import coined as CO
nx = 4096
eng = q.init_engine("b200")
g = q.graphs.grid(nx, nx)
c = nx // 2 + nx * (nx // 2)
spec = q.CoinedSpec(g, "flipflop", "grover", frozenset({c}), "minus_identity")
psi = q.WalkState(q.graphs.arc_basis(g), np.full(4 * nx * nx, 2.0 ** -13, dtype=np.complex128))
for rep in range(2):
    t0 = time.perf_counter()
    trace, dists = CO.search_trace(eng, spec, 16707, psi, 4096)
    print(f"rep {rep}: search_trace {1e3 * (time.perf_counter() - t0):.1f} ms "
          f"({os.environ.get('QWB_SNAPSHOT_HOST', 'default')})", flush=True)
