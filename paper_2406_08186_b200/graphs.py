"""Graphs and the canonical arc basis (mirrors qwalk.graphs, graphs.py:28-235).

Named families (`cycle`, `line`, `grid`, `hypercube`) are built on the GPU
(`qwb_family_adjacency`, bit-exact with graphs.py:115-159) and lazily: a
`Graph` carries (kind, params) and materialises its host CSR adjacency only
when something asks for it.  The matrix-free lattice path never does, so an
8192 x 8192 torus costs no host memory.

`ArcBasis` keeps the reference's tail-major / head-minor order
(graphs.py:178-214) but replaces the per-arc Python dict (5 s and GBs of RSS
at 1024^2) by a binary search inside the tail's sorted neighbour row.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .backend import CsrMatrix, builder_engine, csr_from_triplets
from .errors import (
    IndexOutOfRange,
    NonSquare,
    NotAnArc,
    NotSymmetric,
    SelfLoopPresent,
    SizeTooSmall,
    VertexOutOfRange,
    WeightedAdjacency,
)

__all__ = [
    "Graph", "ArcBasis", "graph_from_adjacency", "graph_from_edges", "cycle", "line", "grid",
    "hypercube", "neighbors", "degree", "arc_basis", "arc_index", "arc_at",
]


class Graph:
    """Simple undirected graph with a validated CSR adjacency (graphs.py:45-65).

    kind is "generic", "cycle", "line", "grid" or "hypercube"; params holds
    the family parameters, e.g. (nx, ny, periodic).  Immutable.
    """

    __slots__ = ("n", "kind", "params", "_adjacency", "_nnz", "_device", "_generated")

    def __init__(self, n: int, adjacency: CsrMatrix | None = None, kind: str = "generic",
                 params: tuple = ()):
        object.__setattr__(self, "n", int(n))
        object.__setattr__(self, "kind", kind)
        object.__setattr__(self, "params", tuple(params))
        object.__setattr__(self, "_adjacency", adjacency)
        object.__setattr__(self, "_nnz", None if adjacency is None else adjacency.nnz)
        object.__setattr__(self, "_device", {})
        object.__setattr__(self, "_generated", adjacency is None)
        if adjacency is None and kind not in ("cycle", "line", "grid", "hypercube"):
            raise ValueError("a generic graph needs an adjacency matrix")

    def __setattr__(self, name, value):
        raise AttributeError("Graph is immutable")

    # --- adjacency -----------------------------------------------------------
    def device_adjacency(self, engine=None):
        """(row_offsets int64, col int64) torch tensors on the engine's GPU."""
        import torch
        eng = engine or builder_engine()
        key = eng.device
        hit = self._device.get(key)
        if hit is not None:
            return hit
        if not self._generated:
            a = self._adjacency
            offs = torch.from_numpy(a.row_offsets).to(eng.torch_device)
            col = torch.from_numpy(a.col_indices).to(eng.torch_device) if a.nnz else \
                torch.zeros(1, dtype=torch.int64, device=eng.torch_device)
        else:
            fam = N.FAMILY[self.kind]
            params = N.i64_array(self._family_params())
            offs = torch.empty(self.n + 1, dtype=torch.int64, device=eng.torch_device)
            nnz = C.c_int64(0)
            eng.call("qwb_family_adjacency", fam, params, N.ptr(offs), None, C.byref(nnz), eng.stream())
            col = torch.empty(max(1, nnz.value), dtype=torch.int64, device=eng.torch_device)
            eng.call("qwb_family_adjacency", fam, params, N.ptr(offs), N.ptr(col), None, eng.stream())
            object.__setattr__(self, "_nnz", int(nnz.value))
        self._device[key] = (offs, col)
        return offs, col

    def _family_params(self):
        if self.kind == "grid":
            nx, ny, periodic = self.params
            return (nx, ny, 1 if periodic else 0)
        return (self.params[0],)

    @property
    def adjacency(self) -> CsrMatrix:
        if self._adjacency is None:
            offs, col = self.device_adjacency()
            nnz = self.num_arcs
            a = CsrMatrix(self.n, self.n, offs.cpu().numpy(), col[:nnz].cpu().numpy(),
                          np.ones(nnz, dtype=np.complex128))
            object.__setattr__(self, "_adjacency", a)
        return self._adjacency

    @property
    def num_arcs(self) -> int:
        if self._nnz is None:
            self._nnz_closed_form()
        if self._nnz is None:
            self.device_adjacency()
        return int(self._nnz)

    def _nnz_closed_form(self):
        if not self._generated:
            return
        if self.kind == "grid":
            nx, ny, periodic = self.params
            if periodic and nx >= 3 and ny >= 3:
                object.__setattr__(self, "_nnz", 4 * nx * ny)
        elif self.kind == "cycle":
            object.__setattr__(self, "_nnz", 2 * self.params[0])
        elif self.kind == "line":
            object.__setattr__(self, "_nnz", 2 * (self.params[0] - 1))
        elif self.kind == "hypercube":
            object.__setattr__(self, "_nnz", self.params[0] * (1 << self.params[0]))

    @property
    def num_edges(self) -> int:
        return self.num_arcs // 2

    @property
    def is_torus(self) -> bool:
        """periodic grid with nx, ny >= 3: regular degree 4, matrix-free path."""
        return self._generated and self.kind == "grid" and bool(self.params[2]) and self.params[0] >= 3 and self.params[1] >= 3

    def __eq__(self, other):
        if not isinstance(other, Graph):
            return NotImplemented
        if self is other:
            return True
        if self.n != other.n or self.kind != other.kind or self.params != other.params:
            return False
        if self._generated and other._generated:
            return True
        a, b = self.adjacency, other.adjacency
        return np.array_equal(a.row_offsets, b.row_offsets) and np.array_equal(a.col_indices, b.col_indices)

    def __hash__(self):
        return hash((self.n, self.kind, self.params))

    def __repr__(self):
        return f"Graph(n={self.n}, kind={self.kind!r}, params={self.params})"


def _validate_pattern(a: CsrMatrix) -> None:
    """graphs.py:68-82 semantics."""
    if a.n_rows != a.n_cols:
        raise NonSquare(f"adjacency is {a.n_rows}x{a.n_cols}")
    a.validate()
    if a.nnz == 0:
        return
    if not np.all(a.values == 1.0):
        raise WeightedAdjacency("adjacency entries must all be exactly 1")
    rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_offsets))
    if np.any(rows == a.col_indices):
        raise SelfLoopPresent("adjacency diagonal must be zero")
    fwd = rows * a.n_cols + a.col_indices
    rev = a.col_indices * a.n_cols + rows
    if not np.array_equal(np.sort(fwd), np.sort(rev)):
        raise NotSymmetric("adjacency pattern must be symmetric")


def graph_from_adjacency(a, kind: str = "generic", params: tuple = ()) -> Graph:
    """Graph from a CSR or square array-like 0/1 adjacency (graphs.py:85-100)."""
    if isinstance(a, CsrMatrix):
        m = a
    else:
        arr = np.asarray(a)
        if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
            raise NonSquare(f"adjacency has shape {arr.shape}")
        r, c = np.nonzero(arr)
        m = csr_from_triplets(arr.shape[0], arr.shape[1], r, c, arr[r, c].astype(complex))
    _validate_pattern(m)
    return Graph(m.n_rows, m, kind, params)


def graph_from_edges(n: int, edges, kind: str = "generic", params: tuple = ()) -> Graph:
    """Graph on n vertices from (v, w) edges (graphs.py:103-112)."""
    e = np.asarray(list(edges), dtype=np.int64).reshape(-1, 2)
    rows = np.concatenate([e[:, 0], e[:, 1]])
    cols = np.concatenate([e[:, 1], e[:, 0]])
    a = csr_from_triplets(n, n, rows, cols, np.ones(rows.size, dtype=complex))
    _validate_pattern(a)
    return Graph(n, a, kind, params)


def cycle(n: int) -> Graph:
    """v ~ (v +- 1) mod n; n >= 3 (graphs.py:115-119)."""
    if n < 3:
        raise SizeTooSmall("cycle requires n >= 3")
    return Graph(n, None, "cycle", (int(n),))


def line(n: int) -> Graph:
    """Path graph; n >= 2 (graphs.py:122-126)."""
    if n < 2:
        raise SizeTooSmall("line requires n >= 2")
    return Graph(n, None, "line", (int(n),))


def grid(nx: int, ny: int, periodic: bool = True) -> Graph:
    """2-D lattice, vertex id x + nx*y, axis neighbours, wrapping if periodic
    (graphs.py:129-150)."""
    if nx < 2 or ny < 2:
        raise SizeTooSmall("grid requires nx, ny >= 2")
    return Graph(nx * ny, None, "grid", (int(nx), int(ny), bool(periodic)))


def hypercube(dim: int) -> Graph:
    """2**dim vertices, adjacent iff Hamming distance 1 (graphs.py:153-159)."""
    if dim < 1:
        raise SizeTooSmall("hypercube requires dim >= 1")
    return Graph(1 << dim, None, "hypercube", (int(dim),))


# ---------------------------------------------------------------------------
# closed forms for the regular families (graphs.py:115-159): a vertex's sorted
# neighbours and its arc-span start without materialising the adjacency (a
# host copy of the 8192^2 torus adjacency is 2 GB; ket() needs one index)
# ---------------------------------------------------------------------------

def _closed_form(g: Graph) -> bool:
    if not g._generated or g._adjacency is not None:
        return False
    if g.kind == "grid":
        return g.is_torus
    return g.kind in ("cycle", "line", "hypercube")


def _family_neighbors(g: Graph, v: int) -> list[int]:
    if g.kind == "grid":
        nx, ny, _ = g.params
        x, y = v % nx, v // nx
        cand = {((x + 1) % nx) + nx * y, ((x - 1) % nx) + nx * y, x + nx * ((y + 1) % ny), x + nx * ((y - 1) % ny)}
        return sorted(cand)
    if g.kind == "cycle":
        n = g.n
        return sorted({(v - 1) % n, (v + 1) % n})
    if g.kind == "line":
        return [u for u in (v - 1, v + 1) if 0 <= u < g.n]
    dim = g.params[0]   # hypercube: v xor 2^b, ascending
    return sorted(v ^ (1 << b) for b in range(dim))


def _family_row_offset(g: Graph, v: int) -> int:
    if g.kind == "grid":
        return 4 * v
    if g.kind == "cycle":
        return 2 * v
    if g.kind == "line":
        return 0 if v == 0 else 2 * v - 1
    return g.params[0] * v


def neighbors(g: Graph, v: int) -> np.ndarray:
    if not (0 <= v < g.n):
        raise VertexOutOfRange(f"vertex {v} not in 0..{g.n - 1}")
    if _closed_form(g):
        return np.asarray(_family_neighbors(g, int(v)), dtype=np.int64)
    a = g.adjacency
    return a.col_indices[a.row_offsets[v]: a.row_offsets[v + 1]].copy()


def degree(g: Graph, v: int) -> int:
    if not (0 <= v < g.n):
        raise VertexOutOfRange(f"vertex {v} not in 0..{g.n - 1}")
    if _closed_form(g):
        return len(_family_neighbors(g, int(v)))
    a = g.adjacency
    return int(a.row_offsets[v + 1] - a.row_offsets[v])


class ArcBasis:
    """Arcs (tail, head) sorted tail-major then head-minor (graphs.py:178-214)."""

    __slots__ = ("graph", "_arcs")

    def __init__(self, graph: Graph):
        self.graph = graph
        self._arcs = None

    @property
    def arcs(self) -> np.ndarray:
        if self._arcs is None:
            a = self.graph.adjacency
            tails = np.repeat(np.arange(self.graph.n, dtype=np.int64), np.diff(a.row_offsets))
            arcs = np.column_stack((tails, a.col_indices))
            arcs.setflags(write=False)
            self._arcs = arcs
        return self._arcs

    @property
    def size(self) -> int:
        return self.graph.num_arcs

    @property
    def tail_offsets(self) -> np.ndarray:
        return self.graph.adjacency.row_offsets

    def __eq__(self, other):
        if not isinstance(other, ArcBasis):
            return False
        return self is other or self.graph == other.graph

    def __hash__(self):
        return hash((self.graph.n, self.size))

    def __repr__(self):
        return f"ArcBasis(n={self.graph.n}, arcs={self.size})"


def arc_basis(g: Graph) -> ArcBasis:
    return ArcBasis(g)


def arc_index(b: ArcBasis, v: int, w: int) -> int:
    """Position of arc (v, w) (graphs.py:222-227)."""
    v, w = int(v), int(w)
    g = b.graph
    if not (0 <= v < g.n):
        raise NotAnArc(f"({v}, {w}) is not an arc of the graph")
    if _closed_form(g):
        nb = _family_neighbors(g, v)
        if w not in nb:
            raise NotAnArc(f"({v}, {w}) is not an arc of the graph")
        return _family_row_offset(g, v) + nb.index(w)
    a = g.adjacency
    lo, hi = int(a.row_offsets[v]), int(a.row_offsets[v + 1])
    j = lo + int(np.searchsorted(a.col_indices[lo:hi], w))
    if j >= hi or a.col_indices[j] != w:
        raise NotAnArc(f"({v}, {w}) is not an arc of the graph")
    return j


def arc_at(b: ArcBasis, idx: int) -> tuple[int, int]:
    if not (0 <= idx < b.size):
        raise IndexOutOfRange(f"arc index {idx} not in 0..{b.size - 1}")
    a = b.graph.adjacency
    v = int(np.searchsorted(a.row_offsets, idx, side="right") - 1)
    return v, int(a.col_indices[idx])
