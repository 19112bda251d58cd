"""Session façade (`Coined`, `ContinuousTime`, `Lattice`, ..., `set_marked`):
the paper-style API named by the north star (TS
frontend/src/session.ts:60-170).  CPU tests cover construction, kets and
validation on generic graphs (family graphs are generated on the device);
GPU tests check that the sessions return the oracle's states bit for bit."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2


def _cycle_adj(n):
    a = np.zeros((n, n))
    for i in range(n):
        a[i, (i + 1) % n] = a[(i + 1) % n, i] = 1
    return a


def test_session_construction_and_kets():
    import paper_2406_08186_b200 as q
    a = _cycle_adj(6)
    w = q.Coined(a, shift="flipflop", coin="grover", marked=[3])
    assert w.spec.marked == frozenset({3}) and w.spec.marked_policy == "minus_identity"
    s = 2 ** -0.5
    psi = s * w.ket(0, 1) + s * w.ket(0, 5)
    assert abs(psi.norm() - 1) < 1e-15
    assert psi.amplitudes[0] == s and psi.amplitudes[1] == s     # arcs (0,1), (0,5)
    w.set_marked([])
    assert w.spec.marked == frozenset() and w.spec.marked_policy == "none"
    w.set_marked(2)
    assert w.get_marked() == [2]
    c = q.ContinuousTime(a, gamma=0.35, time=0.03, marked=[1, 4])
    assert c.get_marked() == [1, 4] and c.get_gamma() == 0.35 and c.get_time() == 0.03
    phi = s * (c.ket(2) + 1j * c.ket(4))
    assert phi.amplitudes[4] == 1j * s
    c.set_marked(None)
    assert c.get_marked() == []


def test_session_validation_matches_core():
    import paper_2406_08186_b200 as q
    a = _cycle_adj(5)
    with pytest.raises(ValueError):
        q.Coined(a, coin="hadamard")          # reference: COINS = ("grover",)
    with pytest.raises(q.errors.MarkedVertexOutOfRange):
        q.Coined(a, marked=[7])
    with pytest.raises(q.errors.UnsupportedGraphForPersistentShift):
        q.Coined(a, shift="persistent")       # generic graph
    with pytest.raises(ValueError):
        q.ContinuousTime(a, gamma=-1.0, time=1.0)
    with pytest.raises(ValueError):
        q.Coined(a).simulate(range=3)         # state missing


@pytest.mark.gpu
def test_coined_session_lattice_bitwise(oracle):
    import paper_2406_08186_b200 as q
    nx = 24
    c = 12 + nx * 12
    with q.Coined(q.Lattice(nx), marked=[c]) as w:
        psi0 = w.uniform_state()
        states = w.simulate(range=(0, 30, 7), state=psi0)
        probs = w.probability_distribution(states)
        offs, cols = oracle.grid_adjacency(nx, nx)
        u = oracle.evolution_operator(offs, cols, "flipflop", (c,))
        ref = oracle.coined_simulate(u, psi0.amplitudes, range(0, 30, 7))
        for st, r, p in zip(states, ref, probs):
            assert np.array_equal(st.amplitudes, r)
            assert np.max(np.abs(p - oracle.coined_probability(offs, r))) <= 1e-12
        # set_marked rebuilds the oracle for the next simulate
        w.set_marked([])
        s2 = w.simulate(range=5, state=psi0)
        ref2 = oracle.coined_simulate(oracle.evolution_operator(offs, cols), psi0.amplitudes, range(5))
        assert all(np.array_equal(a.amplitudes, b) for a, b in zip(s2, ref2))
        u_dev = w.get_evolution()
        u_ref = oracle.evolution_operator(offs, cols)
        assert np.array_equal(u_dev.row_offsets, u_ref.row_offsets) and np.array_equal(u_dev.values, u_ref.values)


@pytest.mark.gpu
def test_continuous_time_session_cycle101(oracle):
    """PAPER.md Fig. 1: cycle(101), walker departing from vertex 50."""
    import paper_2406_08186_b200 as q
    with q.ContinuousTime(q.Cycle(101), gamma=0.5, time=5.0) as ct:
        psi0 = ct.ket(50)
        states = ct.simulate(range=11, state=psi0)
        probs = ct.probability_distribution(states)
        offs, cols = oracle.cycle_adjacency(101)
        h = oracle.hamiltonian(offs, cols, 0.5)
        ref = oracle.ctqw_simulate(h, psi0.amplitudes, range(11), 5.0)
        for st, r, p in zip(states, ref, probs):
            assert rel_l2(st.amplitudes, r) <= 1e-10
            assert np.max(np.abs(p - np.abs(r) ** 2)) <= 1e-12
        # mirror symmetry about the start vertex (tests/test_acceptance.py:86-102)
        p = probs[-1]
        assert np.max(np.abs(p[50 - np.arange(50)] - p[50 + np.arange(50)])) <= 1e-10
        ct.set_marked([50])
        h2 = ct.get_hamiltonian()
        assert h2.nnz == h.nnz + 1
