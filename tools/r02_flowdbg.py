"""Per-phase cycle counters of the lattice kernels (experiment build with
-DQWB_EXP_TIMING): usage flowdbg.py nx steps"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_08186_b200 as q
from paper_2406_08186_b200 import coined as CO, _native as N
nx = int(sys.argv[1]); steps = int(sys.argv[2])
eng = q.init_engine("b200")
r = CO._LatticeRunner(eng, q.CoinedSpec(q.graphs.grid(nx, nx)))
r.a.fill_(1.0 / np.sqrt(4 * nx * nx))
lib = N.load()
buf = (C.c_ulonglong * 16)()
r.advance(steps); torch.cuda.synchronize()
lib.qwb_exp_dbg(buf, 1)
r.advance(steps); torch.cuda.synchronize()
lib.qwb_exp_dbg(buf, 1)
for k, name in ((0, "tile"), (1, "flow")):
    v = list(buf[8 * k:8 * k + 8])
    n = v[3]
    if n:
        print(f"{name}: items {n}, per item cycles (tid 0): wait {v[0]/n:.0f}, lds+bar {v[1]/n:.0f}, steps+store {v[2]/n:.0f}, storing warp steps+store {v[4]/n:.0f}, not-ready {v[5]}, prefetch section {v[6]/n:.0f}")
