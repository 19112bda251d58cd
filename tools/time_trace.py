"""Device time per coined step with and without the fused p(marked) trace:
torus nx^2, centre marked, 4096 steps.  usage: time_trace.py [nx]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_08186_b200 as q
from paper_2406_08186_b200 import coined as CO
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
c = nx // 2 + nx * (nx // 2)
eng = q.init_engine("b200")
spec = q.CoinedSpec(q.graphs.grid(nx, nx), "flipflop", "grover", frozenset({c}), "minus_identity")
r = CO._LatticeRunner(eng, spec)
r.a.fill_(2.0 ** -13)
trace = torch.empty((4097, 1), dtype=torch.float64, device="cuda")
def tm(label, fn):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"nx {nx} {label}: {dt / 4096 * 1e6:.1f} us/step", flush=True)
tm("no trace", lambda: r.advance(4096))
tm("trace", lambda: r.advance(4096, trace, (c,)))
