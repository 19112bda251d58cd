"""Time the pieces of coined.simulate(engine, spec, (1000, 1001, 1), psi0) on
grid 2048^2 (the bench's e2e call): H2D, norm check, layout conversion, the
1000 steps, conversion back, D2H."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_08186_b200 as q
from paper_2406_08186_b200 import coined as CO, backend as B

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
eng = q.init_engine("b200")
g = q.graphs.grid(nx, nx)
spec = q.CoinedSpec(g)
rng = np.random.default_rng(0)
psi = rng.normal(size=g.num_arcs) + 1j * rng.normal(size=g.num_arcs)
psi /= np.linalg.norm(psi)
psi0 = q.WalkState(q.graphs.arc_basis(g), psi)

def t(label, fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    print(f"{label:28s} {(time.perf_counter() - t0) / reps * 1e3:8.2f} ms", flush=True)
    return r

x = t("H2D (to_device)", lambda: B.to_device(eng, psi0.amplitudes))
t("device_norm", lambda: B.device_norm(eng, x))
r = CO._LatticeRunner(eng, spec)
t("to_planes", lambda: r.load(x))
t("advance(1000)", lambda: r.advance(1000), reps=2)
t("from_planes", lambda: r.store(x))
t("D2H (to_host pinned)", lambda: B.to_host(x, pinned=True))
t("simulate (1000,1001,1)", lambda: CO.simulate(eng, spec, (1000, 1001, 1), psi0))
t("arc_basis + basis check", lambda: q.graphs.arc_basis(g) == psi0.basis)
hp = torch.empty(g.num_arcs, dtype=torch.complex128, pin_memory=True)
hpage = torch.empty(g.num_arcs, dtype=torch.complex128)
print("psi0 pinned:", torch.from_numpy(np.ascontiguousarray(psi0.amplitudes)).is_pinned())
t("H2D torch pinned tensor", lambda: x.copy_(hp))
t("H2D torch pageable", lambda: x.copy_(hpage))
t("D2H torch pinned tensor", lambda: hp.copy_(x))
t("D2H torch pageable", lambda: hpage.copy_(x))
t("pinned alloc 268MB", lambda: torch.empty(g.num_arcs, dtype=torch.complex128, pin_memory=True))
t("simulate (0,1001,100) 11 snaps", lambda: CO.simulate(eng, spec, (0, 1001, 100), psi0), reps=2)
t("simulate (0,10001,1000) 11 snaps", lambda: CO.simulate(eng, spec, (0, 10001, 1000), psi0), reps=1)
