"""First-call cost of coined.search_trace at C3 (4096^2): the function's
phases replayed with a synchronize after each, in a fresh process, twice."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_08186_b200 as q
from paper_2406_08186_b200 import coined as CO
from paper_2406_08186_b200.backend import SnapshotPipe
nx = 4096
eng = q.init_engine("b200")
g = q.graphs.grid(nx, nx)
c = nx // 2 + nx * (nx // 2)
spec = q.CoinedSpec(g, "flipflop", "grover", frozenset({c}), "minus_identity")
psi = q.WalkState(q.graphs.arc_basis(g), np.full(4 * nx * nx, 2.0 ** -13, dtype=np.complex128))
for rep in range(2):
    t = [time.perf_counter()]
    def mark():
        torch.cuda.synchronize(); t.append(time.perf_counter())
    marked = spec.active_marked
    basis, x = CO._upload_initial(eng, spec, psi); mark()
    r = CO._LatticeRunner(eng, spec); r.load(x); mark()
    trace = torch.empty((16708, 1), dtype=torch.float64, device="cuda")
    pipe = SnapshotPipe(eng, g.n, 4, dtype=torch.float64, pinned=False); mark()
    r.advance(16, trace, marked); mark()
    r.advance(4096 - 16, trace[16:], marked); mark()
    pipe.capture(r.probability); mark()
    r.advance(4096, trace[4096:], marked); mark()
    pipe.capture(r.probability); mark()
    res = pipe.results(); mark()
    d = np.diff(t) * 1e3
    print(f"rep {rep}: upload {d[0]:.1f}, runner {d[1]:.1f}, pipe init {d[2]:.1f}, first 16 steps {d[3]:.1f}, "
          f"4080 steps {d[4]:.1f}, capture {d[5]:.1f}, 4096 steps {d[6]:.1f}, capture {d[7]:.1f}, results {d[8]:.1f} ms",
          flush=True)
