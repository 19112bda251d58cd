"""Device time per coined step on a 4096^2 torus with different marked sets
(tile kernel, no trace): for the marked-variant cost.  usage: time_marked.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_08186_b200 as q
from paper_2406_08186_b200 import coined as CO
nx = 4096
c = nx // 2 + nx * (nx // 2)
eng = q.init_engine("b200")
for label, marked in (("none", ()), ("centre", (c,)), ("corner 0", (0,)), ("8 vertices", tuple(c + 37 * k for k in range(8)))):
    spec = q.CoinedSpec(q.graphs.grid(nx, nx), "flipflop", "grover", frozenset(marked),
                        "minus_identity" if marked else "none")
    r = CO._LatticeRunner(eng, spec)
    r.a.fill_(2.0 ** -13)
    r.advance(960); torch.cuda.synchronize()
    t0 = time.perf_counter(); r.advance(960); torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter() - t0) / 960 * 1e6:.2f} us/step", flush=True)
    del r
