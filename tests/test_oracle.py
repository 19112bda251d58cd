"""Pin the CPU oracle to the reference: golden fixtures (always) and the live
reference (only where /root/reference is mounted, i.e. the build container).

Everything here is bit-exact (`np.array_equal`) unless stated otherwise: the
oracle uses the same numpy primitives in the same order as the reference.
"""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC, golden_group, load_golden
from oracle import qwalk_oracle as O

GRAPH_BUILDERS = {
    "cycle": lambda p: O.cycle_adjacency(int(p[0])),
    "line": lambda p: O.line_adjacency(int(p[0])),
    "grid": lambda p: O.grid_adjacency(int(p[0]), int(p[1]), bool(p[2])),
    "hypercube": lambda p: O.hypercube_adjacency(int(p[0])),
}


def _adj(rec):
    kind = str(rec["kind"])
    if kind in GRAPH_BUILDERS:
        return GRAPH_BUILDERS[kind](rec["params"])
    return rec["offs"], rec["cols"]


def test_graph_families_and_arc_order():
    z = load_golden("graphs")
    for name in z["names"]:
        rec = golden_group(z, str(name))
        offs, cols = _adj(rec)
        assert np.array_equal(offs, rec["offs"]), name
        assert np.array_equal(cols, rec["cols"]), name
        assert np.array_equal(O.arcs(offs, cols), rec["arcs"]), name
        assert np.array_equal(O.reverse_arcs(offs, cols), rec["flipflop"]), name
        if "persistent" in rec:
            t = O.persistent_targets(str(rec["kind"]), tuple(int(x) for x in rec["params"]), offs, cols)
            assert np.array_equal(t, rec["persistent"]), name


def test_known_answers():
    # cycle(3) arcs (reference tests/test_graphs.py:107-112)
    offs, cols = O.cycle_adjacency(3)
    assert [tuple(a) for a in O.arcs(offs, cols)] == [(0, 1), (0, 2), (1, 0), (1, 2), (2, 0), (2, 1)]
    # S[2,0] = 1 on cycle(3) (tests/test_coined.py:31-36)
    assert O.reverse_arcs(offs, cols)[0] == 2
    # cycle(4): U|0,1> = |3,0> (tests/test_coined.py:189-198)
    offs, cols = O.cycle_adjacency(4)
    u = O.evolution_operator(offs, cols)
    amp = np.zeros(8, complex)
    amp[0] = 1.0
    out = O.csr_rows(u, amp, 0, 8)
    assert out[O.arc_positions(offs, cols, [3], [0])[0]] == 1.0 and np.abs(out).sum() == 1.0
    # hypercube slot order: N(5) in dim 4 = [1, 4, 7, 13]
    offs, cols = O.hypercube_adjacency(4)
    assert list(cols[offs[5]:offs[6]]) == [1, 4, 7, 13]


def test_coined_operator_and_trajectories_bitwise():
    z = load_golden("coined")
    for name in z["cases"]:
        rec = golden_group(z, str(name))
        kind = str(rec["kind"])
        offs, cols = rec["offs"], rec["cols"]
        if kind in GRAPH_BUILDERS:
            o2, c2 = GRAPH_BUILDERS[kind](rec["params"])
            assert np.array_equal(o2, offs) and np.array_equal(c2, cols)
        u = O.evolution_operator(offs, cols, str(rec["shift"]), rec["marked"], kind,
                                 tuple(int(x) for x in rec["params"]))
        assert np.array_equal(u.row_offsets, rec["u_offs"]), name
        assert np.array_equal(u.col_indices, rec["u_cols"]), name
        assert np.array_equal(u.values, rec["u_vals"]), name
        if "states" in rec:
            r = rec["range"]
            states = O.coined_simulate(u, rec["psi0"], range(*r))
            assert np.array_equal(np.stack(states), rec["states"]), name
            probs = np.stack([O.coined_probability(offs, s) for s in states])
            assert np.array_equal(probs, rec["probs"]), name


def test_threaded_matvec_is_bitwise_serial():
    offs, cols = O.grid_adjacency(40, 30)
    u = O.evolution_operator(offs, cols, marked=(5, 77))
    rng = np.random.default_rng(3)
    x = rng.normal(size=u.n_rows) + 1j * rng.normal(size=u.n_rows)
    mv = O.Matvec(4)
    try:
        assert np.array_equal(mv(u, x), O.csr_rows(u, x, 0, u.n_rows))
    finally:
        mv.close()


def test_ctqw_bitwise():
    z = load_golden("ctqw")
    for name in z["cases"]:
        rec = golden_group(z, str(name))
        kind = str(rec["kind"])
        offs, cols = rec["offs"], rec["cols"]
        if kind in GRAPH_BUILDERS:
            o2, c2 = GRAPH_BUILDERS[kind](rec["params"])
            assert np.array_equal(o2, offs) and np.array_equal(c2, cols)
        h = O.hamiltonian(offs, cols, float(rec["gamma"]), rec["marked"])
        assert np.array_equal(h.row_offsets, rec["h_offs"]), name
        assert np.array_equal(h.col_indices, rec["h_cols"]), name
        assert np.array_equal(h.values, rec["h_vals"]), name
        assert O.inf_norm(h) == float(rec["inf_norm"]), name
        ev = O.evolve_state(h, rec["psi0"], float(rec["t_evolve"]))
        assert np.array_equal(ev, rec["evolved"]), name
        states = O.ctqw_simulate(h, rec["psi0"], range(*rec["range"]), float(rec["delta_t"]))
        assert np.array_equal(np.stack(states), rec["states"]), name
        assert np.array_equal(np.stack([O.ctqw_probability(s) for s in states]), rec["probs"]), name


def test_series_not_converged():
    offs, cols = O.cycle_adjacency(8)
    h = O.hamiltonian(offs, cols, 1.0)
    psi = np.zeros(8, complex)
    psi[0] = 1
    with pytest.raises(O.SeriesNotConverged):
        O.evolve_state(h, psi, 1.0, max_terms=3)


def test_numpy_summation_model_pinned():
    """The pairwise order the CUDA kernels implement against
    numpy's own reduceat on the golden probes."""
    from tests_support_pairwise import pairwise_reduceat
    z = load_golden("numerics")
    for k in (1, 2, 3, 4, 5, 8, 9, 13, 22, 23, 64, 65, 66, 100, 200, 300):
        x = z[f"x{k}"]
        ref = z[f"sum{k}"][0]
        got = pairwise_reduceat(x)
        assert got.real == ref.real and got.imag == ref.imag, k
        assert np.add.reduceat(x, [0])[0] == ref


def test_numpy_cmul_model_pinned():
    from tests_support_pairwise import cmul_fma
    z = load_golden("numerics")
    a, b, ab = z["mul_a"], z["mul_b"], z["mul_ab"]
    for i in range(a.shape[0]):
        got = cmul_fma(a[i], b[i])
        assert got.real == ab[i].real and got.imag == ab[i].imag


# --------------------------------------------------------------------------
# live reference (build container only)
# --------------------------------------------------------------------------

needs_ref = pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference not mounted")


def _ref():
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    from qwalk import backend as B, coined as CO, ctqw as CT, graphs as G
    spec = importlib.util.spec_from_file_location(
        "ref_conftest", "/root/reference/pkg/tests/conftest.py")
    conf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(conf)
    return B, CO, CT, G, conf


@needs_ref
def test_live_reference_random_graphs_coined():
    B, CO, CT, G, conf = _ref()
    eng = B.init_engine("serial")
    rng = np.random.default_rng(4096)
    for _ in range(40):
        g = conf.random_graph_with_arc_bound(rng, max_arcs=64)
        marked = {int(rng.integers(0, g.n))} if rng.random() < 0.5 else set()
        spec = CO.CoinedSpec(g, "flipflop", "grover", frozenset(marked),
                             "minus_identity" if marked else "none")
        u_ref = CO.evolution_operator(eng, spec)
        u = O.evolution_operator(g.adjacency.row_offsets, g.adjacency.col_indices, marked=marked)
        assert np.array_equal(u.row_offsets, u_ref.row_offsets)
        assert np.array_equal(u.col_indices, u_ref.col_indices)
        assert np.array_equal(u.values, u_ref.values)
        x = conf.random_unit_vector(rng, u.n_rows)
        assert np.array_equal(O.csr_rows(u, x, 0, u.n_rows), B._csr_rows(u_ref, x, 0, u.n_rows))
    B.stop_engine(eng)


@needs_ref
def test_live_reference_grid_sizes():
    B, CO, CT, G, conf = _ref()
    for nx, ny in ((3, 3), (3, 4), (5, 3), (2, 5), (9, 2), (12, 12)):
        for periodic in (True, False):
            g = G.grid(nx, ny, periodic)
            offs, cols = O.grid_adjacency(nx, ny, periodic)
            assert np.array_equal(offs, g.adjacency.row_offsets)
            assert np.array_equal(cols, g.adjacency.col_indices)
    for d in (1, 2, 5, 8):
        g = G.hypercube(d)
        offs, cols = O.hypercube_adjacency(d)
        assert np.array_equal(cols, g.adjacency.col_indices)
