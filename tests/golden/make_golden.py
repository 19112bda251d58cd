"""Generate golden fixtures by running the REAL reference (`qwalk` 0.1.0).

Run in the build container (where /root/reference is mounted):

    python tests/golden/make_golden.py

It imports the reference from /root/reference/pkg/src (read-only; nothing is
copied) and writes `tests/golden/*.npz`.  The fixtures are what the oracle and
the GPU product are pinned to on the GPU box, where /root/reference does not
exist.  Regenerating must be deterministic: every input is seeded.
"""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
OUT = os.path.dirname(os.path.abspath(__file__))


def _load_reference():
    sys.path.insert(0, REF_SRC)
    import qwalk  # noqa: F401  (reference package)
    from qwalk import backend as B, coined as CO, ctqw as CT, graphs as G
    from qwalk.state import VertexBasis, WalkState
    spec = importlib.util.spec_from_file_location("ref_conftest", os.path.join(REF_TESTS, "conftest.py"))
    conf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(conf)
    return B, CO, CT, G, VertexBasis, WalkState, conf


def _graph_record(prefix, g, G, CO, out):
    a = g.adjacency
    b = G.arc_basis(g)
    out[prefix + "offs"] = a.row_offsets
    out[prefix + "cols"] = a.col_indices
    out[prefix + "arcs"] = np.asarray(b.arcs)
    out[prefix + "flipflop"] = _targets_of(CO.flip_flop_shift(b))
    if g.kind in ("cycle", "line") or (g.kind == "grid" and g.params[2] and min(g.params[:2]) >= 3):
        out[prefix + "persistent"] = _targets_of(CO.persistent_shift(b))


def _targets_of(perm_csr):
    """Permutation CSR (row targets[j], col j) -> targets array."""
    rows = np.repeat(np.arange(perm_csr.n_rows), np.diff(perm_csr.row_offsets))
    t = np.empty(perm_csr.n_cols, dtype=np.int64)
    t[perm_csr.col_indices] = rows
    return t


def main():
    B, CO, CT, G, VertexBasis, WalkState, conf = _load_reference()
    eng = B.init_engine("serial")

    # ---------------- graphs: adjacency, arc order, shift targets ----------
    graphs = {
        "k2": G.graph_from_adjacency([[0, 1], [1, 0]]),
        "cycle3": G.cycle(3),
        "cycle7": G.cycle(7),
        "line5": G.line(5),
        "grid5x5": G.grid(5, 5),
        "grid4x3": G.grid(4, 3),
        "grid2x3": G.grid(2, 3),
        "grid3x2": G.grid(3, 2),
        "grid2x2": G.grid(2, 2),
        "grid4x4open": G.grid(4, 4, periodic=False),
        "grid7x5": G.grid(7, 5),
        "hypercube4": G.hypercube(4),
        "star": G.graph_from_edges(6, [(0, 1), (0, 2), (0, 3), (1, 2), (4, 5)]),
    }
    rng = np.random.default_rng(8192)
    for i in range(6):
        graphs[f"rand{i}"] = conf.random_graph_with_arc_bound(rng, max_arcs=80)
    rng = np.random.default_rng(2024)
    for i in range(4):
        graphs[f"conn{i}"] = conf.random_connected_graph(rng, max_n=24)
    g_out = {}
    names = sorted(graphs)
    for name in names:
        _graph_record(name + "/", graphs[name], G, CO, g_out)
        g_out[name + "/kind"] = np.array(graphs[name].kind)
        g_out[name + "/params"] = np.array(graphs[name].params if graphs[name].params else (), dtype=np.int64)
    g_out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "graphs.npz"), **g_out)

    # ---------------- coined operators U and trajectories ------------------
    u_out = {}
    cases = []

    def add_case(name, g, shift="flipflop", marked=(), psi0=None, rng_=None, steps=()):
        spec = CO.CoinedSpec(g, shift, "grover", frozenset(marked),
                             "minus_identity" if marked else "none")
        u = CO.evolution_operator(eng, spec)
        b = G.arc_basis(g)
        p = name + "/"
        u_out[p + "offs"] = g.adjacency.row_offsets
        u_out[p + "cols"] = g.adjacency.col_indices
        u_out[p + "kind"] = np.array(g.kind)
        u_out[p + "params"] = np.array(g.params if g.params else (), dtype=np.int64)
        u_out[p + "shift"] = np.array(shift)
        u_out[p + "marked"] = np.array(sorted(marked), dtype=np.int64)
        u_out[p + "u_offs"] = u.row_offsets
        u_out[p + "u_cols"] = u.col_indices
        u_out[p + "u_vals"] = u.values
        if psi0 is None:
            amp = conf.random_unit_vector(rng_, b.size)
        else:
            amp = psi0
        st0 = WalkState(b, amp)
        if steps:
            states = CO.simulate(eng, spec, steps, st0)
            u_out[p + "psi0"] = amp
            u_out[p + "range"] = np.array(steps, dtype=np.int64)
            u_out[p + "states"] = np.stack([s.amplitudes for s in states])
            u_out[p + "probs"] = np.stack(CO.probability_distribution(g, states))
        cases.append(name)

    r = np.random.default_rng(7)
    add_case("k2", graphs["k2"], rng_=r, steps=(0, 4, 1))
    add_case("cycle5", G.cycle(5), rng_=r, steps=(0, 12, 3))
    add_case("cycle9_persistent_marked", G.cycle(9), "persistent", {2}, rng_=r, steps=(0, 20, 5))
    add_case("line6_persistent", G.line(6), "persistent", rng_=r, steps=(0, 15, 7))
    add_case("grid5x5", G.grid(5, 5), rng_=r, steps=(0, 30, 10))
    add_case("grid6x6_persistent", G.grid(6, 6), "persistent", rng_=r, steps=(0, 25, 8))
    add_case("grid16_marked", G.grid(16, 16), "flipflop", {0, 37}, rng_=r, steps=(0, 40, 13))
    add_case("grid33_marked2", G.grid(33, 33), "flipflop", {5, 600}, rng_=r, steps=(3, 50, 23))
    add_case("grid7x5_persistent_marked", G.grid(7, 5), "persistent", {34}, rng_=r, steps=(0, 21, 10))
    add_case("grid2x3", G.grid(2, 3), rng_=r, steps=(0, 10, 3))
    add_case("grid4x4open", G.grid(4, 4, periodic=False), rng_=r, steps=(0, 10, 3))
    add_case("hypercube4_marked", G.hypercube(4), "flipflop", {3}, rng_=r, steps=(0, 10, 2))
    add_case("star", graphs["star"], rng_=r, steps=(0, 9, 4))
    # C1: cycle(1024), psi0 = (|512,513> + i|512,511>)/sqrt 2, range (0, 501, 1) -> keep a few
    g1024 = G.cycle(1024)
    b1024 = G.arc_basis(g1024)
    amp = np.zeros(b1024.size, dtype=complex)
    amp[G.arc_index(b1024, 512, 513)] = 1 / np.sqrt(2)
    amp[G.arc_index(b1024, 512, 511)] = 1j / np.sqrt(2)
    add_case("c1_cycle1024", g1024, psi0=amp, steps=(0, 501, 100))
    # grid 64^2, center 4-arc state (pattern of tests/test_acceptance.py:147-157)
    nx = 64
    g64 = G.grid(nx, nx)
    b64 = G.arc_basis(g64)
    c = 32 + nx * 32
    amp = np.zeros(b64.size, dtype=complex)
    for w in (c + 1, c - 1, c + nx, c - nx):
        amp[G.arc_index(b64, c, w)] = 0.5
    add_case("grid64_center", g64, psi0=amp, steps=(0, 65, 16))
    add_case("grid21_persistent_center", G.grid(21, 21), "persistent",
             psi0=_center_state(G, 21), steps=(60, 61, 1))
    rr = np.random.default_rng(41)
    for i in range(6):
        g = conf.random_graph_with_arc_bound(rr, max_arcs=64)
        add_case(f"rand41_{i}", g, rng_=rr, steps=(0, int(rr.integers(2, 40)), 3))
    u_out["cases"] = np.array(cases)
    np.savez_compressed(os.path.join(OUT, "coined.npz"), **u_out)

    # ---------------- CTQW: H, inf-norm, evolve, simulate ------------------
    c_out = {}
    ccases = []

    def add_ctqw(name, g, gamma, delta_t, marked, psi0, rng_idx, t_evolve):
        spec = CT.CtqwSpec(g, gamma, delta_t, frozenset(marked))
        h = CT.build_hamiltonian(spec)
        p = name + "/"
        c_out[p + "offs"] = g.adjacency.row_offsets
        c_out[p + "cols"] = g.adjacency.col_indices
        c_out[p + "kind"] = np.array(g.kind)
        c_out[p + "params"] = np.array(g.params if g.params else (), dtype=np.int64)
        c_out[p + "gamma"] = np.array(gamma)
        c_out[p + "delta_t"] = np.array(delta_t)
        c_out[p + "marked"] = np.array(sorted(marked), dtype=np.int64)
        c_out[p + "h_offs"] = h.row_offsets
        c_out[p + "h_cols"] = h.col_indices
        c_out[p + "h_vals"] = h.values
        c_out[p + "inf_norm"] = np.array(CT._inf_norm(h))
        st0 = WalkState(VertexBasis(g.n), psi0)
        c_out[p + "psi0"] = psi0
        c_out[p + "t_evolve"] = np.array(t_evolve)
        c_out[p + "evolved"] = CT.evolve_state(eng, h, st0, t_evolve).amplitudes
        states = CT.simulate(eng, spec, rng_idx, st0)
        c_out[p + "range"] = np.array(rng_idx, dtype=np.int64)
        c_out[p + "states"] = np.stack([s.amplitudes for s in states])
        c_out[p + "probs"] = np.stack(CT.probability_distribution(states))
        ccases.append(name)

    r = np.random.default_rng(31)
    add_ctqw("k2", graphs["k2"], 1.0, np.pi / 2, (), np.array([1.0, 0.0], complex), (0, 3, 1), np.pi / 2)
    add_ctqw("cycle8", G.cycle(8), 0.5, 0.7, (), conf.random_unit_vector(r, 8), (0, 6, 2), 2.3)
    add_ctqw("cycle101", G.cycle(101), 0.35, 5.0, (50,), _vertex(101, 50), (0, 11, 5), 50.0)
    add_ctqw("hypercube6_marked", G.hypercube(6), 1.0 / 6, 1.0, (0,),
             np.full(64, 1 / 8, dtype=complex), (0, 4, 1), 1.0)
    add_ctqw("hypercube10_marked", G.hypercube(10), 1.0 / 10, 1.0, (0,),
             np.full(1024, 1 / 32, dtype=complex), (0, 3, 2), 1.0)
    add_ctqw("grid8x8", G.grid(8, 8), 0.25, 0.9, (3, 17), conf.random_unit_vector(r, 64), (1, 5, 2), 1.7)
    rr = np.random.default_rng(2024)
    for i in range(4):
        g = conf.random_connected_graph(rr, max_n=20)
        add_ctqw(f"rand2024_{i}", g, float(rr.uniform(0.1, 2.0)), float(rr.uniform(0.1, 1.5)),
                 (int(rr.integers(0, g.n)),), conf.random_unit_vector(rr, g.n), (0, 4, 1),
                 float(rr.uniform(0.1, 3.0)))
    c_out["cases"] = np.array(ccases)
    np.savez_compressed(os.path.join(OUT, "ctqw.npz"), **c_out)

    # ---------------- numpy summation-order probes (backend.py:400-403) ----
    s_out = {}
    rng = np.random.default_rng(5)
    for k in (1, 2, 3, 4, 5, 8, 9, 13, 22, 23, 64, 65, 66, 100, 200, 300):
        x = (rng.normal(size=k) + 1j * rng.normal(size=k)) * 10.0 ** rng.integers(-6, 6, size=k)
        s_out[f"x{k}"] = x
        s_out[f"sum{k}"] = np.add.reduceat(x, [0])
    a = rng.normal(size=257) + 1j * rng.normal(size=257)
    b = rng.normal(size=257) + 1j * rng.normal(size=257)
    s_out["mul_a"], s_out["mul_b"], s_out["mul_ab"] = a, b, a * b
    np.savez_compressed(os.path.join(OUT, "numerics.npz"), **s_out)
    B.stop_engine(eng)
    print("golden fixtures written to", OUT)


def _vertex(n, v):
    a = np.zeros(n, dtype=complex)
    a[v] = 1.0
    return a


def _center_state(G, nx):
    g = G.grid(nx, nx)
    b = G.arc_basis(g)
    c = nx // 2 + nx * (nx // 2)
    amp = np.zeros(b.size, dtype=complex)
    for w in (c + 1, c - 1, c + nx, c - nx):
        amp[G.arc_index(b, c, w)] = 0.5
    return amp


if __name__ == "__main__":
    main()
