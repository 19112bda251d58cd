"""The reference package itself (installed unmodified in baseline/_ref) with
the B200 core plugged in as engine kind "b200" (paper_2406_08186_b200.bridge):
the reference's own coined.simulate / ctqw.evolve_state / ctqw.simulate run
through libqwb200 and reproduce the golden fixtures the reference wrote.
Skipped when baseline/_ref is absent (it is installed per checkout,
DESIGN.md §5)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden_group, load_golden, rel_l2

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def qwalk():
    if not os.path.isdir(os.path.join(REF, "qwalk")):
        pytest.skip("baseline/_ref (the installed reference) is absent")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import qwalk
    if not os.path.abspath(qwalk.__file__).startswith(REF):
        pytest.skip("another qwalk copy was imported first in this process")
    from paper_2406_08186_b200 import bridge
    bridge.install(qwalk)
    return qwalk


def _graph(qw, rec):
    kind = str(rec["kind"])
    p = [int(x) for x in rec["params"]]
    if kind == "cycle":
        return qw.graphs.cycle(p[0])
    if kind == "line":
        return qw.graphs.line(p[0])
    if kind == "grid":
        return qw.graphs.grid(p[0], p[1], bool(p[2]))
    if kind == "hypercube":
        return qw.graphs.hypercube(p[0])
    offs, cols = rec["offs"], rec["cols"]
    a = qw.CsrMatrix(offs.shape[0] - 1, offs.shape[0] - 1, offs, cols, np.ones(cols.shape[0], complex))
    return qw.graph_from_adjacency(a)


def test_cpu_engines_untouched(qwalk):
    """The bridge leaves the reference's own engines on their own code."""
    g = qwalk.graphs.cycle(16)
    spec = qwalk.coined.CoinedSpec(g)
    psi = qwalk.coined.ket(spec, 0, 1)
    for kind in ("serial", "parallel"):
        eng = qwalk.init_engine(kind, 2)
        assert eng.kind.value == kind
        st = qwalk.coined.simulate(eng, spec, (0, 5, 1), psi)
        assert len(st) == 5 and abs(st[-1].norm() - 1.0) < 1e-12
        qwalk.stop_engine(eng)


def test_b200_kind_fails_loudly_without_gpu(qwalk):
    from conftest import have_gpu
    if have_gpu():
        pytest.skip("a GPU is visible")
    with pytest.raises(Exception) as ei:
        qwalk.init_engine("b200")
    assert "DeviceError" in type(ei.value).__name__ or "device" in str(ei.value).lower()


@pytest.mark.gpu
def test_reference_coined_simulate_on_b200(qwalk):
    z = load_golden("coined")
    eng = qwalk.init_engine("b200")
    try:
        for name in z["cases"]:
            rec = golden_group(z, str(name))
            if "states" not in rec:
                continue
            g = _graph(qwalk, rec)
            marked = frozenset(int(v) for v in rec["marked"])
            spec = qwalk.coined.CoinedSpec(g, str(rec["shift"]), "grover", marked,
                                           "minus_identity" if marked else "none")
            psi0 = qwalk.WalkState(qwalk.arc_basis(g), rec["psi0"])
            states = qwalk.coined.simulate(eng, spec, tuple(int(x) for x in rec["range"]), psi0)
            got = np.stack([s.amplitudes for s in states])
            assert np.array_equal(got, rec["states"]), name
            probs = qwalk.coined.probability_distribution(spec, states)
            assert np.array_equal(np.stack(probs), rec["probs"]), name
    finally:
        qwalk.stop_engine(eng)


@pytest.mark.gpu
def test_reference_ctqw_on_b200(qwalk):
    z = load_golden("ctqw")
    eng = qwalk.init_engine("b200")
    try:
        for name in z["cases"]:
            rec = golden_group(z, str(name))
            g = _graph(qwalk, rec)
            spec = qwalk.ctqw.CtqwSpec(g, float(rec["gamma"]), float(rec["delta_t"]),
                                       frozenset(int(v) for v in rec["marked"]))
            h = qwalk.ctqw.build_hamiltonian(spec)
            psi0 = qwalk.WalkState(qwalk.VertexBasis(g.n), rec["psi0"])
            ev = qwalk.ctqw.evolve_state(eng, h, psi0, float(rec["t_evolve"]))
            assert rel_l2(ev.amplitudes, rec["evolved"]) <= 1e-10, name
            assert np.array_equal(ev.amplitudes, rec["evolved"]), name
            states = qwalk.ctqw.simulate(eng, spec, tuple(int(x) for x in rec["range"]), psi0)
            assert np.array_equal(np.stack([s.amplitudes for s in states]), rec["states"]), name
    finally:
        qwalk.stop_engine(eng)


@pytest.mark.gpu
def test_reference_errors_through_b200(qwalk):
    """Operand checks keep the reference's exception classes."""
    from qwalk import errors as RE
    eng = qwalk.init_engine("b200")
    other = qwalk.init_engine("serial")
    try:
        v = qwalk.move_to_device(eng, qwalk.ComplexVector(np.ones(4, complex)))
        m = qwalk.move_to_device(eng, qwalk.csr_from_triplets(3, 3, [0, 1, 2], [0, 1, 2], np.ones(3, complex)))
        with pytest.raises(RE.DimensionMismatch):
            qwalk.matvec_mul(eng, v, m)
        with pytest.raises(RE.NonFiniteEntry):
            qwalk.move_to_device(eng, qwalk.ComplexVector(np.array([1.0, np.nan], complex)))
        w = qwalk.move_to_device(other, qwalk.ComplexVector(np.ones(3, complex)))
        with pytest.raises(RE.NotOnDevice):
            qwalk.matvec_mul(eng, w, m)
        qwalk.stop_engine(eng)
        with pytest.raises(RE.EngineStopped):
            qwalk.move_to_device(eng, qwalk.ComplexVector(np.ones(3, complex)))
        with pytest.raises(RE.AlreadyStopped):
            qwalk.stop_engine(eng)
    finally:
        if eng.state == "initialized":
            qwalk.stop_engine(eng)
        qwalk.stop_engine(other)
