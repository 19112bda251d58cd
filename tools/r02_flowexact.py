"""Debug: flow kernel vs per-launch kernel on a localized start (2304 x 256),
differences per step count (run each in its own process via env)."""
import os, subprocess, sys
import numpy as np
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2406_08186_b200 as q
nx, ny, steps = 2304, 256, int(sys.argv[2])
eng = q.init_engine("b200")
g = q.graphs.grid(nx, ny); b = q.graphs.arc_basis(g)
c = nx // 2 + nx * (ny // 2)
psi = np.zeros(b.size, complex)
for w in (c - 1, c + 1, c - nx, c + nx): psi[q.graphs.arc_index(b, c, w)] = 0.5
out = q.coined.simulate(eng, q.CoinedSpec(g), (steps, steps + 1, 1), q.WalkState(b, psi))[0].amplitudes
np.save(sys.argv[3], out)
'''
for steps in [int(x) for x in sys.argv[1:]]:
    res = {}
    for flow in ("2", "0"):
        f = f"/tmp/fx_{flow}_{steps}.npy"
        subprocess.run([sys.executable, "-c", code, root, str(steps), f], env=dict(os.environ, QWB_LATTICE_FLOW=flow), check=True)
        res[flow] = np.load(f)
    d = res["2"] != res["0"]
    print(steps, "differ", int(d.sum()), "max abs", float(np.abs(res["2"] - res["0"]).max()), "norm flow", float(np.linalg.norm(res["2"])), flush=True)
