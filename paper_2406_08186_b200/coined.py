"""Coined discrete-time walk on the B200 (mirrors qwalk.coined, coined.py:38-294).

One step applies U = S C (Grover coin, then the flip-flop or persistent shift;
marked vertices get the -I coin block).  Three device paths, chosen per graph:

* torus (`grid(nx, ny, periodic=True)`, nx, ny >= 3): matrix-free fused
  coin+shift+oracle kernel on the direction-plane layout (lattice.cu) — U is
  never materialised, 32 B of HBM traffic per arc per step;
* any other graph: U built on the device as int32/complex128 CSR
  (builders.cu) and stepped with the CSR SpMV (spmv.cu); operators whose state
  fits in shared memory run the whole snapshot loop in one persistent CTA.

All paths reproduce the reference's numpy arithmetic bit for bit.  States stay
in HBM between snapshots; only requested snapshots are copied back.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .backend import (
    CsrMatrix,
    DeviceCsr,
    Engine,
    SnapshotPipe,
    builder_engine,
    csr_from_triplets,
    device_norm,
    empty_z,
    to_device,
    to_host,
)
from .errors import (
    BasisMismatch,
    MarkedVertexOutOfRange,
    UnnormalizedInitialState,
    UnsupportedGraphForPersistentShift,
)
from .graphs import ArcBasis, Graph, arc_basis, arc_index
from .state import SimRange, WalkState

__all__ = [
    "CoinedSpec", "SHIFTS", "COINS", "MARKED_POLICIES", "flip_flop_shift", "persistent_shift",
    "grover_coin", "apply_marked_policy", "evolution_operator", "ket", "simulate",
    "probability_distribution", "simulate_probabilities", "search_trace",
]

SHIFTS = ("flipflop", "persistent")
COINS = ("grover",)
MARKED_POLICIES = ("minus_identity", "none")

_SNAPSHOT_BUDGET_BYTES = 1 << 30


@dataclass(frozen=True)
class CoinedSpec:
    """Parameters of a coined walk (coined.py:58-87)."""

    graph: Graph
    shift: str = "flipflop"
    coin: str = "grover"
    marked: frozenset = frozenset()
    marked_policy: str = "none"

    def __post_init__(self):
        if self.shift not in SHIFTS:
            raise ValueError(f"shift: unknown shift {self.shift!r} (expected one of {SHIFTS})")
        if self.coin not in COINS:
            raise ValueError(f"coin: unknown coin {self.coin!r} (expected one of {COINS})")
        if self.marked_policy not in MARKED_POLICIES:
            raise ValueError(f"marked_policy: unknown policy {self.marked_policy!r}"
                             f" (expected one of {MARKED_POLICIES})")
        object.__setattr__(self, "marked", frozenset(int(v) for v in self.marked))
        for v in self.marked:
            if not (0 <= v < self.graph.n):
                raise MarkedVertexOutOfRange(f"marked vertex {v} not in 0..{self.graph.n - 1}")
        if self.marked and self.marked_policy == "none":
            raise ValueError("marked_policy: must be 'minus_identity' when vertices are marked")
        if self.shift == "persistent" and self.graph.kind not in ("cycle", "line", "grid"):
            raise UnsupportedGraphForPersistentShift(
                f"persistent shift is undefined on {self.graph.kind!r} graphs")

    @property
    def active_marked(self) -> tuple:
        return tuple(sorted(self.marked)) if self.marked_policy == "minus_identity" else ()


def _family_args(g: Graph):
    fam = N.FAMILY.get(g.kind, 0)
    if g.kind == "grid":
        nx, ny, periodic = g.params
        return fam, N.i64_array((nx, ny, 1 if periodic else 0))
    if g.kind in ("cycle", "line", "hypercube") and g.params:
        return fam, N.i64_array((g.params[0],))
    return 0, N.i64_array((0,))


def _marked_tensor(engine: Engine, marked):
    import torch
    if not marked:
        return None
    return torch.tensor(sorted(marked), dtype=torch.int64, device=engine.torch_device)


def _shift_sources(engine: Engine, g: Graph, shift: str):
    import torch
    offs, col = g.device_adjacency(engine)
    fam, params = _family_args(g)
    src = torch.empty(max(1, g.num_arcs), dtype=torch.int64, device=engine.torch_device)
    engine.call("qwb_shift_sources", g.n, N.ptr(offs), N.ptr(col), N.SHIFT[shift], fam, params,
                N.ptr(src), engine.stream())
    return src[: g.num_arcs]


def _permutation_from_sources(src) -> CsrMatrix:
    s = src.cpu().numpy()
    n = s.shape[0]
    return CsrMatrix(n, n, np.arange(n + 1, dtype=np.int64), s, np.ones(n, dtype=np.complex128))


def flip_flop_shift(basis: ArcBasis) -> CsrMatrix:
    """Arc-reversal permutation (coined.py:96-101), built on the device."""
    return _permutation_from_sources(_shift_sources(builder_engine(), basis.graph, "flipflop"))


def persistent_shift(basis: ArcBasis) -> CsrMatrix:
    """Direction-preserving shift (coined.py:149-161), built on the device."""
    if basis.graph.kind not in ("cycle", "line", "grid"):
        raise UnsupportedGraphForPersistentShift(
            f"persistent shift is undefined on {basis.graph.kind!r} graphs")
    return _permutation_from_sources(_shift_sources(builder_engine(), basis.graph, "persistent"))


def device_operator(engine: Engine, g: Graph, shift: str, marked=()) -> DeviceCsr:
    """U = S C (or C alone for shift "none") as device CSR (coined.py:164-238)."""
    import torch
    offs, col = g.device_adjacency(engine)
    n_arcs = g.num_arcs
    fam, params = _family_args(g)
    mk = _marked_tensor(engine, marked)
    uoffs = torch.empty(n_arcs + 1, dtype=torch.int64, device=engine.torch_device)
    nnz = C.c_int64(0)
    args = (g.n, N.ptr(offs), N.ptr(col), N.ptr(mk), len(marked), N.SHIFT[shift], fam, params)
    engine.call("qwb_coined_operator", *args, N.ptr(uoffs), None, None, C.byref(nnz), engine.stream())
    ucol = torch.empty(max(1, nnz.value), dtype=torch.int32, device=engine.torch_device)
    uval = torch.empty(max(1, nnz.value), dtype=torch.complex128, device=engine.torch_device)
    engine.call("qwb_coined_operator", *args, N.ptr(uoffs), N.ptr(ucol), N.ptr(uval), None,
                engine.stream())
    return DeviceCsr(n_arcs, n_arcs, uoffs, ucol[: nnz.value], uval[: nnz.value])


def grover_coin(basis: ArcBasis) -> CsrMatrix:
    """Block-diagonal Grover coin, exact zeros dropped (coined.py:164-185)."""
    return device_operator(builder_engine(), basis.graph, "none").to_host()


def apply_marked_policy(coin: CsrMatrix, basis: ArcBasis, marked, policy: str = "minus_identity") -> CsrMatrix:
    """Replace marked vertices' coin blocks by -I (coined.py:188-219).

    Host CSR surgery on a caller-supplied coin (the walk itself folds the
    oracle into the device builder instead)."""
    if policy == "none" or not marked:
        return coin
    if policy != "minus_identity":
        raise ValueError(f"marked_policy: unknown policy {policy!r}")
    marked = frozenset(int(v) for v in marked)
    for v in marked:
        if not (0 <= v < basis.graph.n):
            raise MarkedVertexOutOfRange(f"marked vertex {v} not in 0..{basis.graph.n - 1}")
    offs = basis.tail_offsets
    in_span = np.zeros(basis.size, dtype=bool)
    for v in marked:
        in_span[offs[v]: offs[v + 1]] = True
    rows = np.repeat(np.arange(coin.n_rows), np.diff(coin.row_offsets))
    keep = ~in_span[rows]
    diag = np.concatenate([np.arange(offs[v], offs[v + 1], dtype=np.int64) for v in sorted(marked)])
    r = np.concatenate([rows[keep], diag])
    c = np.concatenate([coin.col_indices[keep], diag])
    vals = np.concatenate([coin.values[keep], np.full(diag.shape[0], -1.0 + 0j)])
    return csr_from_triplets(coin.n_rows, coin.n_cols, r, c, vals)


def evolution_operator(engine: Engine, spec: CoinedSpec) -> CsrMatrix:
    """U = S C as a host CsrMatrix (coined.py:230-238), assembled on the GPU."""
    engine._require_running()
    return device_operator(engine, spec.graph, spec.shift, spec.active_marked).to_host()


def ket(spec, v: int, w: int) -> WalkState:
    """|v, w> (coined.py:241-247)."""
    g = spec if isinstance(spec, Graph) else spec.graph
    basis = arc_basis(g)
    amp = np.zeros(basis.size, dtype=np.complex128)
    amp[arc_index(basis, v, w)] = 1.0
    return WalkState(basis, amp)


# ---------------------------------------------------------------------------
# device runners
# ---------------------------------------------------------------------------

class _LatticeRunner:
    """Matrix-free torus path; state kept as 4 direction planes."""

    def __init__(self, engine: Engine, spec: CoinedSpec):
        import torch
        self.engine = engine
        g = spec.graph
        self.nx, self.ny = int(g.params[0]), int(g.params[1])
        self.n = self.nx * self.ny
        self.shift = N.SHIFT[spec.shift]
        self.bits = None
        marked = spec.active_marked
        self.marked = tuple(marked)
        self.marked_arr = N.i64_array(marked)
        if marked:
            self.bits = torch.empty((self.n + 31) // 32, dtype=torch.int32, device=engine.torch_device)
            mk = _marked_tensor(engine, marked)
            engine.call("qwb_marked_bitmap", self.n, N.ptr(mk), len(marked), N.ptr(self.bits),
                        engine.stream())
        self.a = empty_z(engine, 4 * self.n)
        self.b = empty_z(engine, 4 * self.n)

    def load(self, arcs):
        self.engine.call("qwb_lattice_to_planes", self.nx, self.ny, N.ptr(arcs), N.ptr(self.a),
                         self.engine.stream())

    def advance(self, steps: int, trace=None, trace_vertices=()):
        if steps <= 0:
            return
        flag = C.c_int(0)
        tv = N.i64_array(trace_vertices)
        self.engine.call("qwb_lattice_run", self.nx, self.ny, self.shift, N.ptr(self.bits),
                         self.marked_arr, len(self.marked), N.ptr(self.a), N.ptr(self.b), int(steps), tv,
                         len(trace_vertices), N.ptr(trace), C.byref(flag), self.engine.stream())
        if flag.value:
            self.a, self.b = self.b, self.a

    def store(self, arcs):
        self.engine.call("qwb_lattice_from_planes", self.nx, self.ny, N.ptr(self.a), N.ptr(arcs),
                         self.engine.stream())

    def probability(self, out):
        self.engine.call("qwb_lattice_probability", self.nx, self.ny, N.ptr(self.a), N.ptr(out),
                         self.engine.stream())


class _CsrRunner:
    """Device-built U stepped by the CSR SpMV."""

    def __init__(self, engine: Engine, spec: CoinedSpec):
        self.engine = engine
        self.graph = spec.graph
        self.u = device_operator(engine, spec.graph, spec.shift, spec.active_marked)
        self.n = self.u.n_rows
        self.cur = empty_z(engine, self.n)
        self.scratch = empty_z(engine, 2 * self.n + 1)

    def load(self, arcs):
        self.cur.copy_(arcs)

    def run_snapshots(self, counts):
        """U^c cur for each cumulative count c; returns (n_snap, n) tensor; cur advances."""
        import torch
        k = N.i64_array(counts)
        out = torch.empty((len(counts), self.n), dtype=torch.complex128, device=self.engine.torch_device)
        u = self.u
        self.engine.call("qwb_csr_run", self.n, N.ptr(u.row_offsets), N.ptr(u.col), N.ptr(u.values),
                         N.ptr(self.cur), k, len(counts), N.ptr(out), N.ptr(self.scratch),
                         self.engine.stream())
        self.cur.copy_(out[-1])
        return out


def _runner(engine: Engine, spec: CoinedSpec):
    if spec.graph.is_torus:
        return _LatticeRunner(engine, spec)
    return _CsrRunner(engine, spec)


def _upload_initial(engine: Engine, spec: CoinedSpec, psi0: WalkState):
    basis = arc_basis(spec.graph)
    if not isinstance(psi0.basis, ArcBasis) or psi0.basis != basis:
        raise BasisMismatch("initial state must be in the arc basis of the graph")
    x = to_device(engine, psi0.amplitudes)
    nrm = device_norm(engine, x)
    if abs(nrm - 1.0) > 1e-8:
        raise UnnormalizedInitialState(f"initial state norm {nrm} is not 1")
    return basis, x


def simulate(engine: Engine, spec: CoinedSpec, sim_range, psi0: WalkState) -> list[WalkState]:
    """States U^k psi0 for each k in the range (coined.py:250-272).

    The state lives in HBM for the whole run; each snapshot is advanced from
    the previous one on the device and copied back once."""
    engine._require_running()
    rng = SimRange.coerce(sim_range)
    basis, x = _upload_initial(engine, spec, psi0)
    ks = list(rng.indices())
    runner = _runner(engine, spec)
    runner.load(x)
    states: list[WalkState] = []
    if isinstance(runner, _LatticeRunner):
        pipe = SnapshotPipe(engine, x.numel(), len(ks))
        cur = 0
        for k in ks:
            runner.advance(k - cur)
            cur = k
            if len(ks) == 1:
                runner.store(x)
                pipe.capture(None, src=x)
            else:
                pipe.capture(runner.store)
        for arr, owner in pipe.results():
            states.append(WalkState._adopt(basis, arr, owner))
        return states
    n = runner.n
    per = max(1, _SNAPSHOT_BUDGET_BYTES // (16 * n))
    cur = 0
    for i in range(0, len(ks), per):
        chunk = ks[i: i + per]
        snaps = runner.run_snapshots([k - cur for k in chunk])
        cur = chunk[-1]
        host, owner = to_host(snaps, pinned=True)
        for j in range(len(chunk)):
            states.append(WalkState._adopt(basis, host[j], owner))
    return states


def simulate_probabilities(engine: Engine, spec: CoinedSpec, sim_range, psi0: WalkState) -> list[np.ndarray]:
    """probability_distribution(spec, simulate(...)) without copying states
    back: the vertex marginals are reduced on the device at each snapshot."""
    engine._require_running()
    rng = SimRange.coerce(sim_range)
    g = spec.graph
    basis, x = _upload_initial(engine, spec, psi0)
    runner = _runner(engine, spec)
    runner.load(x)
    import torch
    p = torch.empty(g.n, dtype=torch.float64, device=engine.torch_device)
    out = []
    cur = 0
    for k in rng.indices():
        if isinstance(runner, _LatticeRunner):
            runner.advance(k - cur)
            runner.probability(p)
        else:
            runner.run_snapshots([k - cur])
            offs, _ = g.device_adjacency(engine)
            engine.call("qwb_prob_arcs", g.n, N.ptr(offs), N.ptr(runner.cur), N.ptr(p), engine.stream())
        cur = k
        out.append(to_host(p).copy())
    return out


def search_trace(engine: Engine, spec: CoinedSpec, steps: int, psi0: WalkState,
                 distribution_every: int = 0):
    """Spatial-search run: p(marked) after every step 0..steps, fused into the
    step kernels, plus full distributions every `distribution_every` steps.

    Returns (trace float64[steps+1, n_marked], {k: p_k}).  Torus only.
    """
    import torch
    engine._require_running()
    g = spec.graph
    if not g.is_torus:
        raise ValueError("search_trace: only the periodic lattice path fuses the trace")
    marked = spec.active_marked
    if not marked or len(marked) > 8:
        raise ValueError("search_trace: needs 1..8 marked vertices")
    basis, x = _upload_initial(engine, spec, psi0)
    r = _LatticeRunner(engine, spec)
    r.load(x)
    trace = torch.empty((steps + 1, len(marked)), dtype=torch.float64, device=engine.torch_device)
    p = torch.empty(g.n, dtype=torch.float64, device=engine.torch_device)
    done = 0
    every = distribution_every if distribution_every > 0 else steps + 1
    # saved distributions download beside the steps that follow them
    keys = list(range(every, steps + 1, every))
    # pageable results through bounce buffers: 4096 steps between distributions
    # leave ample time for the host copies, and nothing is page-locked
    pipe = SnapshotPipe(engine, g.n, max(2, len(keys)), dtype=torch.float64, pinned=False)
    while done < steps:
        chunk = min(steps - done, every - (done % every))
        r.advance(chunk, trace[done:], marked)
        done += chunk
        if done % every == 0:
            pipe.capture(r.probability)
    dists = {k: arr for k, (arr, _owner) in zip(keys, pipe.results())}
    # p(marked) of the final state
    r.probability(p)
    last = p[list(marked)]
    trace[steps].copy_(last)
    return to_host(trace), dists


def probability_distribution(spec, states) -> list[np.ndarray]:
    """p[v] = sum over v's arcs of |amplitude|^2 (coined.py:275-294), on the GPU."""
    import torch
    g = spec if isinstance(spec, Graph) else spec.graph
    eng = builder_engine()
    offs, _ = g.device_adjacency(eng)
    out = []
    p = torch.empty(g.n, dtype=torch.float64, device=eng.torch_device)
    for st in states:
        if not isinstance(st.basis, ArcBasis):
            raise BasisMismatch("expected arc-basis states")
        if st.dim != g.num_arcs:
            raise BasisMismatch(f"state dim {st.dim} does not match the graph's {g.num_arcs} arcs")
        x = to_device(eng, st.amplitudes)
        eng.call("qwb_prob_arcs", g.n, N.ptr(offs), N.ptr(x), N.ptr(p), eng.stream())
        out.append(to_host(p).copy())
    return out
