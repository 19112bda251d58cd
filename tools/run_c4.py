"""C4 workload driver for profiling: hypercube(22) CTQW, gamma = 1/22,
marked {0}, one evolve of t = 1 (2 sub-steps x ~12 Taylor terms)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_08186_b200 as q
from paper_2406_08186_b200 import ctqw as CT

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 22
eng = q.init_engine("b200")
marked = frozenset() if os.environ.get("C4_UNMARKED") else frozenset({0})
cs = q.CtqwSpec(q.graphs.hypercube(dim), 1.0 / dim, 1.0, marked)
op = CT._Operator(eng, cs)
n = 1 << dim
x = torch.full((n,), 1.0 / np.sqrt(n), dtype=torch.complex128, device="cuda")
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    terms = op.evolve(x, 1.0, 1e-12)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"dim {dim}: {dt*1e3:.2f} ms, terms {terms}, {dt/sum(terms)*1e6:.1f} us/term")
q.stop_engine(eng)
