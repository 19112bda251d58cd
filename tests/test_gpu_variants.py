"""The lattice kernels' launch forms, each forced through its environment
switch in a fresh process (the switches are read once per process), against
the CPU oracle, bitwise: the persistent dataflow kernel (QWB_LATTICE_FLOW=2)
and the per-launch tile kernel (QWB_LATTICE_FLOW=0) on lattices where the
default would pick the other one, with marked vertices, both shifts, wrap
tiles narrower than the halo, and a localized start run into the subnormal
range; and the hypercube term kernels' forms (QWB_HC_STREAM)."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2406_08186_b200 as q
from oracle import qwalk_oracle as O
nx, ny, steps, shift, localized = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5], sys.argv[6] == "1"
marked = tuple(int(v) for v in sys.argv[7].split(",") if v)
eng = q.init_engine("b200")
g = q.graphs.grid(nx, ny)
spec = q.CoinedSpec(g, shift, "grover", frozenset(marked), "minus_identity" if marked else "none")
b = q.graphs.arc_basis(g)
if localized:
    c = nx // 2 + nx * (ny // 2)
    psi = np.zeros(b.size, complex)
    for w in (c - 1, c + 1, c - nx, c + nx):
        psi[q.graphs.arc_index(b, c, w)] = 0.5
else:
    rng = np.random.default_rng(nx + ny)
    psi = rng.normal(size=b.size) + 1j * rng.normal(size=b.size)
    psi /= np.linalg.norm(psi)
got = q.coined.simulate(eng, spec, (steps, steps + 1, 1), q.WalkState(b, psi))[0].amplitudes
offs, cols = O.grid_adjacency(nx, ny)
u = O.evolution_operator(offs, cols, shift, marked, "grid", (nx, ny, True))
mv = O.Matvec(O.default_threads())
ref = O.coined_simulate(u, psi, [steps], mv)[0]
mv.close()
bad = int(np.count_nonzero(got != ref))
print("differ", bad)
sys.exit(1 if bad else 0)
'''


@pytest.mark.parametrize("flow", ["2", "0"])
@pytest.mark.parametrize("nx,ny,steps,shift,localized,marked", [
    (2048, 2048, 41, "flipflop", False, ""),                        # flow forced on (default: per-launch)
    (1024, 1024, 40, "persistent", False, "5,524800"),              # per-launch forced on (default: flow)
    (1018, 290, 33, "flipflop", False, "0,1017,294000"),            # last tile column 10 wide, row 10 high
    (290, 1022, 26, "persistent", False, "145"),                    # last tile column 2 wide (< T)
    (2304, 256, 1100, "flipflop", True, ""),                        # front into subnormals
    (1024, 1024, 40, "flipflop", False, "525311,308221"),           # marked at x = nx - 1 and nx - 3, interior
                                                                    # rows: halo columns of the x0 = 0 tiles
])
def test_lattice_launch_forms(flow, nx, ny, steps, shift, localized, marked, tmp_path):
    env = dict(os.environ, QWB_LATTICE_FLOW=flow)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(nx), str(ny), str(steps), shift,
                        "1" if localized else "0", marked], capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr


HC_SCRIPT = r'''
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2406_08186_b200 as q
from oracle import qwalk_oracle as O
dim = int(sys.argv[2])
marked = tuple(int(v) for v in sys.argv[3].split(",") if v)
n = 1 << dim
rng = np.random.default_rng(dim + 1)
psi = rng.normal(size=n) + 1j * rng.normal(size=n)
psi /= np.linalg.norm(psi)
eng = q.init_engine("b200")
spec = q.CtqwSpec(q.graphs.hypercube(dim), 1.0 / dim, 0.75, frozenset(marked))
got = q.ctqw.simulate(eng, spec, (0, 2, 1), q.WalkState(q.VertexBasis(n), psi))[-1].amplitudes
offs, cols = O.hypercube_adjacency(dim)
ref = O.evolve_state(O.hamiltonian(offs, cols, 1.0 / dim, marked), psi, 0.75)
bad = int(np.count_nonzero(got != ref))
print("differ", bad)
sys.exit(1 if bad else 0)
'''


@pytest.mark.parametrize("variant", ["52", "51", "42", "21202", "21201", "21002"])
@pytest.mark.parametrize("dim,marked", [(14, "0,777,16383"), (13, "5,8191")])
def test_hypercube_term_kernel_forms(variant, dim, marked):
    """The hypercube term kernels forced through QWB_HC_STREAM (paired ring:
    NSP * 10 + PROD; single ring: CONS/256 * 10000 + NS * 100 + PROD; odd
    partner counts always take the single ring), bitwise against the oracle."""
    env = dict(os.environ, QWB_HC_STREAM=variant)
    r = subprocess.run([sys.executable, "-c", HC_SCRIPT, ROOT, str(dim), marked], capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def _fuzz_case(seed):
    """A random torus, step count, shift and marked set (biased to the torus
    edges, the halo columns that wrap, and to more than 8 vertices: the
    bitmap path)."""
    import numpy as np
    rng = np.random.default_rng(1000 + seed)
    nx, ny = (int(v) for v in rng.integers(64, 600, size=2))
    steps = int(rng.integers(1, 40))
    shift = ("flipflop", "persistent")[seed % 2]
    k = int(rng.choice([0, 1, 3, 9]))
    xs = [int(v) for v in rng.choice([0, 1, 5, nx - 1, nx - 3, nx - 6, nx // 2, int(rng.integers(0, nx))], size=k)]
    ys = [int(v) for v in rng.choice([0, 1, 7, ny - 1, ny - 2, ny // 2, int(rng.integers(0, ny))], size=k)]
    marked = sorted({y * nx + x for x, y in zip(xs, ys)})
    return nx, ny, steps, shift, ",".join(str(v) for v in marked)


@pytest.mark.parametrize("form", ["launch", "flow"])
@pytest.mark.parametrize("seed", range(int(os.environ.get("QWB_FUZZ_CASES", "8"))))
def test_lattice_fuzz(seed, form):
    """Random tori, step counts, shifts and marked sets through the lattice
    kernels, bitwise against the oracle."""
    nx, ny, steps, shift, marked = _fuzz_case(seed)
    env = dict(os.environ, QWB_LATTICE_FLOW={"launch": "0", "flow": "2"}[form])
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(nx), str(ny), str(steps), shift, "0", marked],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, f"{nx}x{ny} {steps} {shift} marked {marked}: " + r.stdout + r.stderr
