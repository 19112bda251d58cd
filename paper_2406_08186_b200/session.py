"""Paper-style session API: `Graph`, `Lattice`/`Grid`, `Cycle`, `Line`,
`Hypercube`, `Coined(...)`, `ContinuousTime(...)`.

The reference exposes this surface only in its TypeScript session wrapper
(`pkg/frontend/src/session.ts:60-170`, `graphs.ts:77-95`) and in the paper
text (`PAPER.md:113-172` ContinuousTime, `PAPER.md:219-263` Coined); both
delegate every computation to the functional core (`coined.simulate`,
`ctqw.simulate`, `probability_distribution`).  Here the same classes sit
directly on the B200 core — no CLI process hop, no JSON hand-off — and keep the
session semantics:

* a session holds a graph, the model parameters and (lazily) a `b200` engine;
* `ket(...)` builds computational-basis states (`coined.ket` / `ctqw.ket`),
  which combine with `+`, `-` and scalar `*` into superpositions;
* `simulate(range=..., state=...)` returns the list of `WalkState`s, range
  being an int m (= (0, m, 1)) or (start, stop, step) (`state.py:91-121`);
* `probability_distribution(states)` returns one float64 vector per state.

`set_marked` (named by the paper, absent from the reference core where marks
are fixed at spec construction) rebuilds the underlying spec, so
the next `simulate` uses the new oracle; the device operator is rebuilt on the
next call exactly as the reference rebuilds U on every `simulate`
(`coined.py:262`).
"""

from __future__ import annotations

import numpy as np

from . import coined as _coined
from . import ctqw as _ctqw
from .backend import CsrMatrix, Engine, init_engine
from .graphs import Graph as _GraphT
from .graphs import cycle as _cycle
from .graphs import graph_from_adjacency
from .graphs import grid as _grid
from .graphs import hypercube as _hypercube
from .graphs import line as _line
from .state import WalkState

__all__ = ["Graph", "Cycle", "Line", "Grid", "Lattice", "Hypercube", "Coined", "ContinuousTime"]


# ---------------------------------------------------------------------------
# graph constructors (graphs.ts:77-95 names; graphs.py:85-159 semantics)
# ---------------------------------------------------------------------------

def Graph(adjacency) -> _GraphT:
    """Graph from a square 0/1 adjacency (array-like, CsrMatrix or Graph)."""
    if isinstance(adjacency, _GraphT):
        return adjacency
    return graph_from_adjacency(adjacency)


def Cycle(n: int) -> _GraphT:
    return _cycle(n)


def Line(n: int) -> _GraphT:
    return _line(n)


def Grid(nx: int, ny: int | None = None, periodic: bool = True) -> _GraphT:
    """2-D lattice nx x ny (square if ny is omitted), periodic by default."""
    return _grid(nx, nx if ny is None else ny, periodic)


Lattice = Grid


def Hypercube(dim: int) -> _GraphT:
    return _hypercube(dim)


def _as_graph(graph) -> _GraphT:
    return graph if isinstance(graph, _GraphT) else Graph(graph)


def _marked_set(marked) -> frozenset:
    if marked is None:
        return frozenset()
    if isinstance(marked, (int, np.integer)):
        return frozenset({int(marked)})
    return frozenset(int(v) for v in marked)


class _Session:
    """Engine ownership shared by both walk models (one engine per session,
    created on first use; `close()` or garbage collection releases it)."""

    def __init__(self, graph, engine: Engine | None):
        self._graph = _as_graph(graph)
        self._engine = engine
        self._own_engine = engine is None

    @property
    def graph(self) -> _GraphT:
        return self._graph

    @property
    def engine(self) -> Engine:
        if self._engine is None or self._engine._stopped:
            self._engine = init_engine("b200")
            self._own_engine = True
        return self._engine

    def close(self) -> None:
        if self._own_engine and self._engine is not None and not self._engine._stopped:
            from .backend import stop_engine
            stop_engine(self._engine)
        self._engine = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


class ContinuousTime(_Session):
    """Continuous-time walk H = -gamma A - sum_{m in M} |m><m|, U(t) = e^{-iHt}
    (`PAPER.md:95-172`; TS `session.ts:81-106`; core `ctqw.py:60-212`).

    `time` is the snapshot interval delta_t: `simulate(range=21, state=psi0)`
    returns psi(k*time) for k = 0..20."""

    def __init__(self, graph, gamma: float, time: float, marked=None, *, engine: Engine | None = None,
                 tol: float = _ctqw.DEFAULT_TOLERANCE):
        super().__init__(graph, engine)
        self._tol = float(tol)
        self._spec = _ctqw.CtqwSpec(self._graph, float(gamma), float(time), _marked_set(marked))

    # parameters --------------------------------------------------------
    @property
    def spec(self) -> _ctqw.CtqwSpec:
        return self._spec

    def get_gamma(self) -> float:
        return self._spec.gamma

    def set_gamma(self, gamma: float) -> None:
        self._spec = _ctqw.CtqwSpec(self._graph, float(gamma), self._spec.delta_t, self._spec.marked)

    def get_time(self) -> float:
        return self._spec.delta_t

    def set_time(self, time: float) -> None:
        self._spec = _ctqw.CtqwSpec(self._graph, self._spec.gamma, float(time), self._spec.marked)

    def get_marked(self) -> list[int]:
        return sorted(self._spec.marked)

    def set_marked(self, marked=None) -> None:
        self._spec = _ctqw.CtqwSpec(self._graph, self._spec.gamma, self._spec.delta_t, _marked_set(marked))

    def get_hamiltonian(self) -> CsrMatrix:
        return _ctqw.build_hamiltonian(self._spec)

    # states ------------------------------------------------------------
    def ket(self, v: int) -> WalkState:
        return _ctqw.ket(self._spec, v)

    def simulate(self, range=None, state: WalkState | None = None, *, tol: float | None = None) -> list[WalkState]:
        if range is None or state is None:
            raise ValueError("simulate: both range and state are required")
        return _ctqw.simulate(self.engine, self._spec, range, state, self._tol if tol is None else tol)

    def probability_distribution(self, states) -> list[np.ndarray]:
        return _ctqw.probability_distribution(_listify(states))


class Coined(_Session):
    """Coined walk U = S C with the Grover coin and the flip-flop (any graph)
    or persistent (cycle, line, grid) shift; marked vertices get the -I coin
    block (`PAPER.md:174-263`; TS `session.ts:108-129`; core `coined.py:58-294`)."""

    def __init__(self, graph, shift: str = "flipflop", coin: str = "grover", marked=None,
                 marked_policy: str | None = None, *, engine: Engine | None = None):
        super().__init__(graph, engine)
        self._shift = shift
        self._coin = coin
        self._policy = marked_policy
        self._spec = self._make_spec(_marked_set(marked))

    def _make_spec(self, marked: frozenset) -> _coined.CoinedSpec:
        policy = self._policy or ("minus_identity" if marked else "none")
        return _coined.CoinedSpec(self._graph, self._shift, self._coin, marked, policy)

    # parameters --------------------------------------------------------
    @property
    def spec(self) -> _coined.CoinedSpec:
        return self._spec

    def get_shift(self) -> str:
        return self._shift

    def get_coin(self) -> str:
        return self._coin

    def get_marked(self) -> list[int]:
        return sorted(self._spec.marked)

    def set_marked(self, marked=None, marked_policy: str | None = None) -> None:
        if marked_policy is not None:
            self._policy = marked_policy
        self._spec = self._make_spec(_marked_set(marked))

    def get_evolution(self) -> CsrMatrix:
        """U = S C as a host CSR (coined.evolution_operator)."""
        return _coined.evolution_operator(self.engine, self._spec)

    # states ------------------------------------------------------------
    def ket(self, v: int, w: int) -> WalkState:
        return _coined.ket(self._spec, v, w)

    def uniform_state(self) -> WalkState:
        """1/sqrt(2|E|) on every arc (the usual spatial-search start)."""
        from .graphs import arc_basis
        b = arc_basis(self._graph)
        return WalkState(b, np.full(b.size, 1.0 / np.sqrt(b.size), dtype=np.complex128))

    def simulate(self, range=None, state: WalkState | None = None) -> list[WalkState]:
        if range is None or state is None:
            raise ValueError("simulate: both range and state are required")
        return _coined.simulate(self.engine, self._spec, range, state)

    def simulate_probabilities(self, range, state: WalkState) -> list[np.ndarray]:
        """probability_distribution(simulate(...)) reduced on the device."""
        return _coined.simulate_probabilities(self.engine, self._spec, range, state)

    def search(self, steps: int, state: WalkState | None = None, distribution_every: int = 0):
        """p(marked) after every step (fused into the lattice kernels)."""
        return _coined.search_trace(self.engine, self._spec, steps,
                                    self.uniform_state() if state is None else state, distribution_every)

    def probability_distribution(self, states) -> list[np.ndarray]:
        return _coined.probability_distribution(self._spec, _listify(states))


def _listify(states):
    return [states] if isinstance(states, WalkState) else list(states)
