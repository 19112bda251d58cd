"""CPU-only tests: the C-ABI library builds, loads and exports every symbol the
header declares; host-side logic (ranges, states, specs, error mapping)
behaves like the reference.  No kernel is launched here."""

from __future__ import annotations

import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def _header_functions():
    text = open(os.path.join(ROOT, "include", "qwb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qwb_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2406_08186_b200 import _build
    return _build.build()


def test_library_exports_every_header_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (qwb_[a-z0-9_]+)", out))
    declared = set(_header_functions())
    assert declared, "header parse failed"
    assert declared <= exported, sorted(declared - exported)


def test_ctypes_signatures_cover_header(lib_path):
    from paper_2406_08186_b200 import _native as N
    assert set(_header_functions()) == set(N.exported_symbols())
    lib = N.load()
    for name in N.exported_symbols():
        assert hasattr(lib, name)
    assert lib.qwb_version().decode().startswith("qwb200")


def test_library_is_sm100a_only(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", "")), out


def test_status_codes_map_to_reference_exceptions():
    from paper_2406_08186_b200 import _native as N, errors as E
    assert N.STATUS_TO_EXC[1] is E.DimensionMismatch
    assert N.STATUS_TO_EXC[7] is E.SeriesNotConverged
    assert N.STATUS_TO_EXC[8] is E.MarkedVertexOutOfRange
    for exc in N.STATUS_TO_EXC.values():
        assert issubclass(exc, (E.QuantumWalkError, ValueError))
    with pytest.raises(E.SeriesNotConverged):
        N.check(7)


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2406_08186_b200 as q
    with pytest.raises(q.errors.DeviceError):
        q.init_engine("b200")
    with pytest.raises(q.errors.UnsupportedEngineKind):
        q.init_engine("serial")


def test_simrange_and_walkstate():
    from paper_2406_08186_b200.state import SimRange, VertexBasis, WalkState
    assert list(SimRange.coerce(3).indices()) == [0, 1, 2]
    assert list(SimRange.coerce((2, 9, 3)).indices()) == [2, 5, 8]
    for bad in ((3, 1, 1), (0, 5, 0), (-1, 2, 1)):
        with pytest.raises(ValueError):
            SimRange.coerce(bad)
    st = WalkState(VertexBasis(3), [1, 0, 0])
    with pytest.raises(AttributeError):
        st.basis = None
    with pytest.raises(ValueError):
        st.amplitudes[0] = 2
    s2 = (st + st) / 2
    assert np.array_equal(s2.amplitudes, st.amplitudes)


def test_specs_validate_like_reference():
    import paper_2406_08186_b200 as q
    g = q.graphs.cycle(4)
    with pytest.raises(ValueError, match="shift"):
        q.CoinedSpec(g, shift="bogus")
    with pytest.raises(ValueError, match="coin"):
        q.CoinedSpec(g, coin="hadamard")
    with pytest.raises(ValueError, match="marked_policy"):
        q.CoinedSpec(g, marked=frozenset({1}), marked_policy="none")
    with pytest.raises(q.errors.MarkedVertexOutOfRange):
        q.CoinedSpec(g, marked=frozenset({7}), marked_policy="minus_identity")
    with pytest.raises(q.errors.UnsupportedGraphForPersistentShift):
        q.CoinedSpec(q.graphs.hypercube(2), shift="persistent")
    with pytest.raises(ValueError):
        q.CtqwSpec(g, 0.0, 1.0)
    with pytest.raises(q.errors.SizeTooSmall):
        q.graphs.grid(1, 5)
    # family graphs need no GPU until their adjacency is requested
    t = q.graphs.grid(8192, 8192)
    assert t.is_torus and t.num_arcs == 4 * 8192 * 8192


def test_host_csr_from_triplets_matches_oracle(oracle):
    import paper_2406_08186_b200 as q
    rng = np.random.default_rng(13)
    r = rng.integers(0, 40, 500)
    c = rng.integers(0, 30, 500)
    v = rng.normal(size=500) + 1j * rng.normal(size=500)
    a = q.csr_from_triplets(40, 30, r, c, v)
    b = oracle.csr_from_triplets(40, 30, r, c, v)
    assert np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert np.array_equal(a.values, b.values)
    g = q.graphs.graph_from_edges(5, [(0, 1), (1, 2), (3, 4)])
    assert list(g.adjacency.col_indices) == [1, 0, 2, 1, 4, 3]
    with pytest.raises(q.errors.NotSymmetric):
        q.graphs.graph_from_adjacency([[0, 1], [0, 0]])
    with pytest.raises(q.errors.SelfLoopPresent):
        q.graphs.graph_from_adjacency([[1, 1], [1, 0]])
    with pytest.raises(q.errors.WeightedAdjacency):
        q.graphs.graph_from_adjacency([[0, 2], [2, 0]])


def test_family_closed_forms_match_oracle():
    """arc_index / neighbors / degree on the regular families without the
    adjacency (closed forms, graphs.py:115-159 semantics) equal the oracle's
    CSR for every vertex of small instances; no device is touched."""
    from oracle import qwalk_oracle as O
    import paper_2406_08186_b200 as q
    cases = [(q.graphs.grid(5, 7), O.grid_adjacency(5, 7)), (q.graphs.grid(3, 3), O.grid_adjacency(3, 3)),
             (q.graphs.cycle(9), O.cycle_adjacency(9)), (q.graphs.line(6), O.line_adjacency(6)),
             (q.graphs.hypercube(5), O.hypercube_adjacency(5))]
    for g, (offs, cols) in cases:
        b = q.graphs.arc_basis(g)
        for v in range(g.n):
            nb = cols[offs[v]:offs[v + 1]]
            assert np.array_equal(q.graphs.neighbors(g, v), nb), (g, v)
            assert q.graphs.degree(g, v) == len(nb)
            for j, w in enumerate(nb):
                assert q.graphs.arc_index(b, v, int(w)) == offs[v] + j
        with pytest.raises(q.errors.NotAnArc):
            q.graphs.arc_index(b, 0, 0)
        assert g._adjacency is None          # nothing was materialised
    # a huge torus: an arc index is O(1) and needs no adjacency
    big = q.graphs.grid(8192, 8192)
    c = 4096 + 8192 * 4096
    assert q.graphs.arc_index(q.graphs.arc_basis(big), c, c + 1) == 4 * c + 2
    assert big._adjacency is None


def test_bench_refuses_more_gpus_than_visible():
    """`bench.py --gpus N` re-execs itself under torchrun when N > 1 and no
    WORLD_SIZE is set, but only when N GPUs are visible: here (no GPU) it must
    fail loudly instead of measuring one GPU and reporting it as N."""
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1",
                        "--warmup", "3", "--no-extras", "--no-cpu"], capture_output=True, text=True, env=env,
                       timeout=300)
    assert r.returncode != 0
    assert "2 requested but 0 CUDA device" in r.stderr
    # a torchrun world that disagrees with --gpus is refused as well
    env.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr
