"""Launch-boundary timeline of the lattice tile kernel (experiment build with
-DQWB_EXP_TIMING exporting qwb_exp_timeline): per launch and CTA, globaltimer
at entry, after griddepcontrol.wait, when the first tile's stage is ready, at
exit.  usage: r02_timeline.py nx"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_08186_b200 as q
from paper_2406_08186_b200 import coined as CO, _native as N
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
eng = q.init_engine("b200")
r = CO._LatticeRunner(eng, q.CoinedSpec(q.graphs.grid(nx, nx)))
r.a.fill_(1.0 / np.sqrt(4 * nx * nx))
lib = N.load()
buf = (C.c_ulonglong * (64 * 160 * 4))()
r.advance(600); torch.cuda.synchronize()
lib.qwb_exp_timeline(buf, 1)
r.advance(6 * 60); torch.cuda.synchronize()
lib.qwb_exp_timeline(buf, 0)
t = np.array(buf, dtype=np.float64).reshape(64, 160, 4)
g = min(148, t.shape[1])
t = t[:, :g, :]
rows = []
for L in range(2, 58):
    a = t[L]
    if (a == 0).any():
        continue
    nxt = t[L + 1]
    rows.append(dict(
        entry_spread=(a[:, 0].max() - a[:, 0].min()) / 1e3,
        wait_min=(a[:, 1].min() - t[L - 1][:, 3].max()) / 1e3,     # after the previous grid's last exit
        ready_after_wait=np.median(a[:, 2] - a[:, 1]) / 1e3,
        exit_spread=(a[:, 3].max() - a[:, 3].min()) / 1e3,
        launch=(a[:, 3].max() - t[L - 1][:, 3].max()) / 1e3,
        compute=(a[:, 3].max() - a[:, 2].min()) / 1e3,
        gap=(nxt[:, 2].min() - a[:, 3].max()) / 1e3))
keys = list(rows[0])
print(f"{nx}^2: {len(rows)} launches, medians (us):")
for k in keys:
    print(f"  {k:18s} {np.median([r_[k] for r_ in rows]):8.2f}")
