"""Continuous-time walk on the B200 (mirrors qwalk.ctqw, ctqw.py:43-212).

H = -gamma A - sum_M |v><v| is applied through the sub-stepped truncated
Taylor series of exp(-iHt) (ctqw.py:123-171) with one fused kernel per term
(taylor.cu).  Hypercube graphs use the matrix-free operator; every other graph
uses H as device CSR built by `qwb_hamiltonian`.  Sub-step count, tau and the
stop floor are computed exactly as the reference does (ctqw.py:149-152), with
||H||_inf reduced on the device in numpy's summation order.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .backend import (
    CsrMatrix,
    DeviceCsr,
    Engine,
    SnapshotPipe,
    builder_engine,
    device_norm,
    empty_z,
    to_device,
    to_host,
    upload_csr,
)
from .errors import (
    BasisMismatch,
    DimensionMismatch,
    MarkedVertexOutOfRange,
    UnnormalizedInitialState,
)
from .graphs import Graph
from .state import SimRange, VertexBasis, WalkState, vertex_state

__all__ = [
    "CtqwSpec", "build_hamiltonian", "get_hamiltonian", "ket", "evolve_state", "simulate",
    "probability_distribution", "DEFAULT_TOLERANCE",
]

DEFAULT_TOLERANCE = 1e-12
_MAX_SERIES_TERMS = 1000   # ctqw.py:57; module-level so tests can monkeypatch it


@dataclass(frozen=True)
class CtqwSpec:
    """Parameters of a continuous-time walk (ctqw.py:60-81)."""

    graph: Graph
    gamma: float
    delta_t: float
    marked: frozenset = frozenset()

    def __post_init__(self):
        if not (self.gamma > 0):
            raise ValueError("gamma must be positive")
        if not (self.delta_t > 0):
            raise ValueError("delta_t (time) must be positive")
        object.__setattr__(self, "marked", frozenset(int(v) for v in self.marked))
        for v in self.marked:
            if not (0 <= v < self.graph.n):
                raise MarkedVertexOutOfRange(f"marked vertex {v} not in 0..{self.graph.n - 1}")


def device_hamiltonian(engine: Engine, spec: CtqwSpec) -> DeviceCsr:
    """H as device CSR (ctqw.py:84-98)."""
    import torch
    g = spec.graph
    offs, col = g.device_adjacency(engine)
    marked = sorted(spec.marked)
    mk = torch.tensor(marked, dtype=torch.int64, device=engine.torch_device) if marked else None
    nnz = g.num_arcs + len(marked)
    hoffs = torch.empty(g.n + 1, dtype=torch.int64, device=engine.torch_device)
    hcol = torch.empty(max(1, nnz), dtype=torch.int32, device=engine.torch_device)
    hval = torch.empty(max(1, nnz), dtype=torch.complex128, device=engine.torch_device)
    engine.call("qwb_hamiltonian", g.n, N.ptr(offs), N.ptr(col), float(spec.gamma), N.ptr(mk), len(marked),
                N.ptr(hoffs), N.ptr(hcol), N.ptr(hval), engine.stream())
    return DeviceCsr(g.n, g.n, hoffs, hcol[:nnz], hval[:nnz])


def build_hamiltonian(spec: CtqwSpec) -> CsrMatrix:
    """Host CsrMatrix of H, assembled on the GPU (ctqw.py:84-98)."""
    return device_hamiltonian(builder_engine(), spec).to_host()


def get_hamiltonian(spec: CtqwSpec) -> CsrMatrix:
    return build_hamiltonian(spec)


def ket(spec, v: int) -> WalkState:
    n = spec.n if isinstance(spec, Graph) else spec.graph.n
    return vertex_state(n, v)


def _inf_norm_csr(engine: Engine, h: DeviceCsr) -> float:
    r = C.c_double(0.0)
    if h.nnz == 0:
        return 0.0
    engine.call("qwb_inf_norm", h.n_rows, N.ptr(h.row_offsets), N.ptr(h.values), C.byref(r), engine.stream())
    return float(r.value)


def _inf_norm_hypercube(engine: Engine, dim: int, gamma: float, marked) -> float:
    """||H||_inf of the hypercube H without building it: the distinct row
    patterns (unmarked: dim x |-gamma|; marked v: the -1 diagonal at sorted
    position popcount(v)) reduced by the same device kernel."""
    rows = []
    if len(marked) < (1 << dim):
        rows.append([gamma] * dim)
    for p in sorted({bin(v).count("1") for v in marked}):
        rows.append([gamma] * p + [1.0] + [gamma] * (dim - p))
    offs = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum([len(r) for r in rows], out=offs[1:])
    vals = np.concatenate([np.asarray(r, dtype=np.complex128) for r in rows])
    import torch
    h = DeviceCsr(len(rows), dim + 1, to_device(engine, offs),
                  torch.zeros(1, dtype=torch.int32, device=engine.torch_device), to_device(engine, vals))
    return _inf_norm_csr(engine, h)


class _Operator:
    """H on the device: CSR or matrix-free hypercube."""

    def __init__(self, engine: Engine, spec: CtqwSpec | None = None, csr: DeviceCsr | None = None):
        self.engine = engine
        self.csr = csr
        self.hypercube = None
        if csr is None:
            g = spec.graph
            if g.kind == "hypercube" and g._generated:
                dim = int(g.params[0])
                marked = sorted(spec.marked)
                bits = None
                if marked:
                    import torch
                    bits = torch.empty(((1 << dim) + 31) // 32, dtype=torch.int32, device=engine.torch_device)
                    mk = torch.tensor(marked, dtype=torch.int64, device=engine.torch_device)
                    engine.call("qwb_marked_bitmap", 1 << dim, N.ptr(mk), len(marked), N.ptr(bits),
                                engine.stream())
                self.hypercube = (dim, float(spec.gamma), bits)
                self.n = 1 << dim
                self.inf_norm = _inf_norm_hypercube(engine, dim, float(spec.gamma), marked)
                return
            self.csr = device_hamiltonian(engine, spec)
        self.n = self.csr.n_rows
        self.inf_norm = _inf_norm_csr(engine, self.csr)
        self._work = None

    def work(self):
        if getattr(self, "_work", None) is None:
            self._work = empty_z(self.engine, 3 * self.n)
        return self._work

    def evolve(self, psi, t: float, tol: float) -> list[int]:
        """psi (device, in place) <- exp(-iHt) psi; returns terms per sub-step."""
        substeps = max(1, math.ceil(self.inf_norm * abs(t)))
        tau = t / substeps
        floor = tol * device_norm(self.engine, psi)
        terms = (C.c_int * substeps)()
        eng = self.engine
        from . import ctqw as _self   # read the (monkeypatchable) module constant
        max_terms = int(_self._MAX_SERIES_TERMS)
        if self.hypercube is not None:
            dim, gamma, bits = self.hypercube
            eng.call("qwb_taylor_evolve_hypercube", dim, gamma, N.ptr(bits), N.ptr(psi), N.ptr(self.work()),
                     substeps, tau, floor, max_terms, terms, eng.stream())
        else:
            h = self.csr
            eng.call("qwb_taylor_evolve_csr", h.n_rows, N.ptr(h.row_offsets), N.ptr(h.col), N.ptr(h.values),
                     N.ptr(psi), N.ptr(self.work()), substeps, tau, floor, max_terms, terms, eng.stream())
        return list(terms)


def evolve_state(engine: Engine, hamiltonian: CsrMatrix, psi: WalkState, t: float,
                 tol: float = DEFAULT_TOLERANCE) -> WalkState:
    """exp(-i H t) psi for a vertex-basis state (ctqw.py:123-171)."""
    engine._require_running()
    if not isinstance(psi.basis, VertexBasis):
        raise BasisMismatch("evolve_state expects a vertex-basis state")
    if psi.dim != hamiltonian.n_rows or hamiltonian.n_rows != hamiltonian.n_cols:
        raise DimensionMismatch(
            f"state dim {psi.dim} does not match Hamiltonian ({hamiltonian.n_rows}x{hamiltonian.n_cols})")
    if not (tol > 0):
        raise ValueError("tol must be positive")
    if t == 0:
        return WalkState(psi.basis, psi.amplitudes)
    op = _Operator(engine, csr=upload_csr(engine, hamiltonian))
    x = to_device(engine, psi.amplitudes)
    op.evolve(x, t, tol)
    arr, owner = to_host(x, pinned=True)
    return WalkState._adopt(psi.basis, arr, owner)


def simulate(engine: Engine, spec: CtqwSpec, sim_range, psi0: WalkState,
             tol: float = DEFAULT_TOLERANCE) -> list[WalkState]:
    """|psi(k delta_t)> for each k in the range, each evolved from the previous
    snapshot in one evolve (ctqw.py:174-202); H stays on the device."""
    engine._require_running()
    rng = SimRange.coerce(sim_range)
    if not isinstance(psi0.basis, VertexBasis) or psi0.dim != spec.graph.n:
        raise BasisMismatch("initial state must be in the vertex basis of the graph")
    x = to_device(engine, psi0.amplitudes)
    nrm = device_norm(engine, x)
    if abs(nrm - 1.0) > 1e-8:
        raise UnnormalizedInitialState(f"initial state norm {nrm} is not 1")
    if not (tol > 0):
        raise ValueError("tol must be positive")
    op = _Operator(engine, spec)
    ks = list(rng.indices())
    moves = sum(1 for a, b in zip([0] + ks, ks) if b != a)
    # snapshot downloads overlap the evolution towards the next snapshot
    pipe = SnapshotPipe(engine, x.numel(), moves)
    which = []         # per index in the range: capture number, or -1 for psi0 itself
    captured = 0
    cur_k = 0
    for k in ks:
        if k != cur_k:
            op.evolve(x, (k - cur_k) * spec.delta_t, tol)
            cur_k = k
            pipe.capture(lambda buf: buf.copy_(x), src=x if moves == 1 else None)
            captured += 1
        which.append(captured - 1)
    res = pipe.results()
    snaps = [WalkState._adopt(psi0.basis, arr, owner) for arr, owner in res]
    return [psi0 if w < 0 else snaps[w] for w in which]


def probability_distribution(states) -> list[np.ndarray]:
    """|psi|^2 per vertex (ctqw.py:205-212), on the GPU."""
    import torch
    eng = builder_engine()
    out = []
    for st in states:
        if not isinstance(st.basis, VertexBasis):
            raise BasisMismatch("expected vertex-basis states")
        x = to_device(eng, st.amplitudes)
        p = torch.empty(st.dim, dtype=torch.float64, device=eng.torch_device)
        eng.call("qwb_prob_abs2", st.dim, N.ptr(x), N.ptr(p), eng.stream())
        out.append(to_host(p))
    return out
