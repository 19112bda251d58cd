"""CPU oracle for the B200 quantum-walk core — TEST INFRASTRUCTURE ONLY.

This module is a vectorised numpy restatement of the reference `qwalk` 0.1.0
algorithm for the hot path (operator builders, the CSR step loop, the Taylor
chain and the probability reducers).  It exists so that the GPU product can be
checked on identical inputs, and so that `bench.py --impl reference` can time
the reference algorithm on host cores.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` leg may import it.  The product package
(`paper_2406_08186_b200`) never imports or calls anything in `oracle/`.

Parity status: PINNED.  `tests/golden/make_golden.py` runs the real reference
(`/root/reference/pkg/src/qwalk`) and commits its outputs as `.npz` fixtures;
`tests/test_oracle.py` checks every function here against them bit for bit
(and, where `/root/reference` is mounted, against the live reference on the
reference's own random-graph seeds).

All arithmetic deliberately uses the same numpy primitives in the same order
as the reference, so results are bitwise identical, not merely close:
  * products  `values * x[cols]`                      (backend.py:400)
  * row sums  `np.add.reduceat`                       (backend.py:403)
  * |psi|^2   `np.abs(psi) ** 2` + `np.add.reduceat`  (coined.py:289-292)
  * scale/axpy/norm via complex scalars + np.linalg.norm (backend.py:433-464)

File:line citations refer to /root/reference/pkg/src/qwalk/.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# ---------------------------------------------------------------------------
# CSR container (mirrors backend.CsrMatrix fields, backend.py:105-153)
# ---------------------------------------------------------------------------


class Csr:
    __slots__ = ("n_rows", "n_cols", "row_offsets", "col_indices", "values")

    def __init__(self, n_rows, n_cols, row_offsets, col_indices, values):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.row_offsets = np.asarray(row_offsets, dtype=np.int64)
        self.col_indices = np.asarray(col_indices, dtype=np.int64)
        self.values = np.asarray(values, dtype=np.complex128)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols), dtype=np.complex128)
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_offsets))
        out[rows, self.col_indices] = self.values
        return out


def csr_from_triplets(n_rows, n_cols, rows, cols, values) -> Csr:
    """Stable key sort, merge duplicates by reduceat, bincount offsets.

    Restates backend.csr_from_triplets (backend.py:195-236).
    """
    r = np.asarray(rows, dtype=np.int64)
    c = np.asarray(cols, dtype=np.int64)
    v = np.asarray(values, dtype=np.complex128)
    if r.size == 0:
        return Csr(n_rows, n_cols, np.zeros(n_rows + 1, np.int64),
                   np.empty(0, np.int64), np.empty(0, np.complex128))
    key = r * n_cols + c
    order = np.argsort(key, kind="stable")
    ks = key[order]
    head = np.ones(ks.shape[0], dtype=bool)
    head[1:] = ks[1:] != ks[:-1]
    first = np.flatnonzero(head)
    uniq = ks[first]
    summed = np.add.reduceat(v[order], first)
    out_rows = uniq // n_cols
    counts = np.bincount(out_rows, minlength=n_rows)
    offsets = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return Csr(n_rows, n_cols, offsets, uniq % n_cols, summed)


# ---------------------------------------------------------------------------
# graph families (graphs.py:103-159) -> (row_offsets, col_indices), int64
# ---------------------------------------------------------------------------


def _adjacency_from_candidates(cand: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """cand: (n, k) int64 neighbour candidates, -1 = absent.  Sorted, deduplicated
    rows (the reference dedups through a Python set, graphs.py:138-150)."""
    n, k = cand.shape
    s = np.sort(cand, axis=1)
    keep = s >= 0
    if k > 1:
        keep[:, 1:] &= s[:, 1:] != s[:, :-1]
    counts = keep.sum(axis=1)
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=offs[1:])
    return offs, s[keep].astype(np.int64)


def grid_adjacency(nx: int, ny: int, periodic: bool = True):
    """Torus / open grid, vertex id x + nx*y (graphs.py:129-150)."""
    n = nx * ny
    v = np.arange(n, dtype=np.int64)
    x, y = v % nx, v // nx
    cand = np.full((n, 4), -1, dtype=np.int64)
    if periodic:
        cand[:, 0] = (x - 1) % nx + nx * y
        cand[:, 1] = (x + 1) % nx + nx * y
        cand[:, 2] = x + nx * ((y - 1) % ny)
        cand[:, 3] = x + nx * ((y + 1) % ny)
    else:
        cand[:, 0] = np.where(x > 0, v - 1, -1)
        cand[:, 1] = np.where(x < nx - 1, v + 1, -1)
        cand[:, 2] = np.where(y > 0, v - nx, -1)
        cand[:, 3] = np.where(y < ny - 1, v + nx, -1)
    return _adjacency_from_candidates(cand)


def cycle_adjacency(n: int):
    """v ~ (v +- 1) mod n (graphs.py:115-119)."""
    v = np.arange(n, dtype=np.int64)
    return _adjacency_from_candidates(np.stack([(v - 1) % n, (v + 1) % n], axis=1))


def line_adjacency(n: int):
    """Path graph (graphs.py:122-126)."""
    v = np.arange(n, dtype=np.int64)
    return _adjacency_from_candidates(
        np.stack([np.where(v > 0, v - 1, -1), np.where(v < n - 1, v + 1, -1)], axis=1))


def hypercube_adjacency(dim: int):
    """v ~ v xor 2^b (graphs.py:153-159)."""
    n = 1 << dim
    v = np.arange(n, dtype=np.int64)
    cand = np.stack([v ^ (1 << b) for b in range(dim)], axis=1)
    return _adjacency_from_candidates(cand)


def edges_adjacency(n: int, edges):
    """graph_from_edges (graphs.py:103-112): both directions, merged by triplets."""
    e = np.asarray(list(edges), dtype=np.int64).reshape(-1, 2)
    rows = np.concatenate([e[:, 0], e[:, 1]])
    cols = np.concatenate([e[:, 1], e[:, 0]])
    a = csr_from_triplets(n, n, rows, cols, np.ones(rows.size, dtype=complex))
    return a.row_offsets, a.col_indices


# ---------------------------------------------------------------------------
# arc basis (graphs.py:178-235)
# ---------------------------------------------------------------------------


def arc_tails(offs: np.ndarray) -> np.ndarray:
    return np.repeat(np.arange(offs.shape[0] - 1, dtype=np.int64), np.diff(offs))


def arcs(offs, cols) -> np.ndarray:
    """(2|E|, 2) tail-major/head-minor list (graphs.py:189-190)."""
    return np.column_stack((arc_tails(offs), cols))


def arc_positions(offs, cols, tails, heads) -> np.ndarray:
    """Index of arcs (tail, head); replaces the per-arc dict lookup of
    graphs.arc_index (graphs.py:192-194, 222-227) by a sorted-key search."""
    n = offs.shape[0] - 1
    keys = arc_tails(offs) * n + cols
    q = np.asarray(tails, np.int64) * n + np.asarray(heads, np.int64)
    pos = np.searchsorted(keys, q)
    if np.any(pos >= keys.shape[0]) or np.any(keys[np.minimum(pos, keys.shape[0] - 1)] != q):
        raise KeyError("not an arc")
    return pos


def reverse_arcs(offs, cols) -> np.ndarray:
    """targets of the flip-flop shift: index of (w, v) for arc (v, w) (coined.py:222-227)."""
    return arc_positions(offs, cols, cols, arc_tails(offs))


def persistent_targets(kind: str, params: tuple, offs, cols) -> np.ndarray:
    """Direction-preserving shift targets (coined.py:104-146)."""
    tails, heads = arc_tails(offs), cols
    n = offs.shape[0] - 1
    if kind == "cycle":
        d = (heads - tails) % n
        return arc_positions(offs, cols, heads, (heads + d) % n)
    if kind == "line":
        d = heads - tails
        nxt = heads + d
        ok = (nxt >= 0) & (nxt < n)
        return arc_positions(offs, cols, heads, np.where(ok, nxt, tails))
    nx, ny, _periodic = params
    vx, vy = tails % nx, tails // nx
    wx, wy = heads % nx, heads // nx
    dx, dy = (wx - vx) % nx, (wy - vy) % ny
    horiz = dy == 0
    sx = np.where(dx == 1, 1, -1)
    sy = np.where(dy == 1, 1, -1)
    tx = np.where(horiz, (wx + sx) % nx, wx)
    ty = np.where(horiz, wy, (wy + sy) % ny)
    return arc_positions(offs, cols, heads, tx + nx * ty)


# ---------------------------------------------------------------------------
# coined operator builder (coined.py:164-238)
# ---------------------------------------------------------------------------


def grover_coin_triplets(offs):
    """Block (2/d) J - I per vertex on its arc span, exact zeros dropped
    (coined.py:164-185).  Returns (rows, cols, vals) in the reference's order."""
    deg = np.diff(offs)
    d_arc = np.repeat(deg, deg)                 # degree of each row's tail
    start_arc = np.repeat(offs[:-1], deg)       # span start of each row
    rows = np.repeat(np.arange(d_arc.shape[0], dtype=np.int64), d_arc)
    # column j-th of row i: span_start + j
    row_start = np.repeat(start_arc, d_arc)
    within = np.arange(rows.shape[0], dtype=np.int64) - np.repeat(
        np.concatenate(([0], np.cumsum(d_arc)[:-1])), d_arc)
    cols = row_start + within
    dd = np.repeat(d_arc, d_arc).astype(np.float64)
    vals = 2.0 / dd - np.where(rows == cols, 1.0, 0.0)
    keep = vals != 0.0
    return rows[keep], cols[keep], vals[keep].astype(np.complex128)


def coin_csr(offs, marked=()) -> Csr:
    """Grover coin with the -I oracle folded in (coined.py:164-219)."""
    n_arcs = int(offs[-1])
    rows, cols, vals = grover_coin_triplets(offs)
    coin = csr_from_triplets(n_arcs, n_arcs, rows, cols, vals)
    marked = sorted(set(int(v) for v in marked))
    if not marked:
        return coin
    in_span = np.zeros(n_arcs, dtype=bool)
    for v in marked:
        in_span[offs[v]:offs[v + 1]] = True
    crow = arc_tails(coin.row_offsets)
    keep = ~in_span[crow]
    diag = np.concatenate([np.arange(offs[v], offs[v + 1], dtype=np.int64) for v in marked])
    r = np.concatenate([crow[keep], diag])
    c = np.concatenate([coin.col_indices[keep], diag])
    v_ = np.concatenate([coin.values[keep], np.full(diag.shape[0], -1.0 + 0j)])
    return csr_from_triplets(n_arcs, n_arcs, r, c, v_)


def evolution_operator(offs, cols, shift="flipflop", marked=(), kind="generic",
                       params=()) -> Csr:
    """U = S C: row k of C becomes row targets[k] (coined.py:230-238)."""
    coin = coin_csr(offs, marked)
    if shift == "flipflop":
        targets = reverse_arcs(offs, cols)
    else:
        targets = persistent_targets(kind, params, offs, cols)
    rows = np.repeat(targets, np.diff(coin.row_offsets))
    n_arcs = int(offs[-1])
    return csr_from_triplets(n_arcs, n_arcs, rows, coin.col_indices, coin.values)


# ---------------------------------------------------------------------------
# step loop (backend.py:394-430, coined.py:250-272)
# ---------------------------------------------------------------------------


def csr_rows(m: Csr, v: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """Rows [lo, hi) of m @ v: gather, multiply, reduceat (backend.py:394-404)."""
    start, stop = int(m.row_offsets[lo]), int(m.row_offsets[hi])
    out = np.zeros(hi - lo, dtype=np.complex128)
    if start == stop:
        return out
    prod = m.values[start:stop] * v[m.col_indices[start:stop]]
    lens = np.diff(m.row_offsets[lo:hi + 1])
    nz = lens > 0
    out[nz] = np.add.reduceat(prod, m.row_offsets[lo:hi][nz] - start)
    return out


def row_blocks(n_rows: int, parts: int):
    b = np.linspace(0, n_rows, parts + 1).astype(int)
    return [(int(x), int(y)) for x, y in zip(b[:-1], b[1:]) if y > x]


class Matvec:
    """Serial or row-block threaded CSR matvec (backend.py:407-430).  Both give
    bitwise-identical results: every row is reduced by one worker."""

    def __init__(self, threads: int = 1):
        self.threads = max(1, int(threads))
        self.pool = ThreadPoolExecutor(self.threads) if self.threads > 1 else None

    def __call__(self, m: Csr, v: np.ndarray) -> np.ndarray:
        if self.pool is None:
            return csr_rows(m, v, 0, m.n_rows)
        blocks = row_blocks(m.n_rows, self.threads)
        return np.concatenate(list(self.pool.map(lambda b: csr_rows(m, v, *b), blocks)))

    def close(self):
        if self.pool is not None:
            self.pool.shutdown(wait=True)
            self.pool = None


def coined_simulate(u: Csr, psi0: np.ndarray, indices, matvec=None) -> list[np.ndarray]:
    """Snapshots U^k psi0 advanced from the previous snapshot (coined.py:263-272)."""
    mv = matvec or Matvec(1)
    out, cur, k0 = [], np.asarray(psi0, np.complex128), 0
    for k in indices:
        for _ in range(k - k0):
            cur = mv(u, cur)
        k0 = k
        out.append(cur.copy())
    return out


def coined_probability(offs, psi: np.ndarray) -> np.ndarray:
    """p[v] = sum over v's arcs of |psi|^2 (coined.py:275-294)."""
    lens = np.diff(offs)
    nz = lens > 0
    mags = np.abs(psi) ** 2
    p = np.zeros(offs.shape[0] - 1)
    if mags.size:
        p[nz] = np.add.reduceat(mags, offs[:-1][nz])
    return p


# ---------------------------------------------------------------------------
# continuous-time walk (ctqw.py:84-212)
# ---------------------------------------------------------------------------

DEFAULT_TOLERANCE = 1e-12     # ctqw.py:54
MAX_SERIES_TERMS = 1000       # ctqw.py:57


class SeriesNotConverged(RuntimeError):
    pass


def hamiltonian(offs, cols, gamma: float, marked=()) -> Csr:
    """H = -gamma A - sum_M |v><v|, diagonal inserted in sorted position (ctqw.py:84-98)."""
    n = offs.shape[0] - 1
    marked = sorted(set(int(v) for v in marked))
    rows = np.concatenate([arc_tails(offs), np.asarray(marked, np.int64)])
    c = np.concatenate([cols, np.asarray(marked, np.int64)])
    vals = np.concatenate([np.full(cols.shape[0], -gamma, dtype=np.complex128),
                           np.full(len(marked), -1.0, dtype=np.complex128)])
    return csr_from_triplets(n, n, rows, c, vals)


def inf_norm(m: Csr) -> float:
    """max_i sum_j |H_ij| via reduceat (ctqw.py:112-120)."""
    if m.nnz == 0:
        return 0.0
    mags = np.abs(m.values)
    lens = np.diff(m.row_offsets)
    sums = np.zeros(m.n_rows)
    nz = lens > 0
    sums[nz] = np.add.reduceat(mags, m.row_offsets[:-1][nz])
    return float(sums.max())


def evolve_state(h: Csr, psi: np.ndarray, t: float, tol: float = DEFAULT_TOLERANCE,
                 matvec=None, max_terms: int = MAX_SERIES_TERMS, stats=None) -> np.ndarray:
    """Sub-stepped truncated Taylor action of exp(-iHt) (ctqw.py:123-171)."""
    mv = matvec or Matvec(1)
    psi = np.asarray(psi, np.complex128)
    if t == 0:
        return psi.copy()
    substeps = max(1, math.ceil(inf_norm(h) * abs(t)))
    tau = t / substeps
    floor = tol * float(np.linalg.norm(psi))
    cur = psi
    for _ in range(substeps):
        acc = cur.copy()
        term = cur.copy()
        for k in range(1, max_terms + 1):
            hterm = mv(h, term)
            term = complex(-1j * tau / k) * hterm
            acc = acc + complex(1.0) * term
            if float(np.linalg.norm(term)) <= floor:
                if stats is not None:
                    stats.append(k)
                break
        else:
            raise SeriesNotConverged(f"series did not reach tol={tol} within {max_terms} terms")
        cur = acc
    return cur


def ctqw_simulate(h: Csr, psi0: np.ndarray, indices, delta_t: float,
                  tol: float = DEFAULT_TOLERANCE, matvec=None) -> list[np.ndarray]:
    """Each snapshot evolved from the previous one in one call (ctqw.py:174-202)."""
    out, cur, k0 = [], np.asarray(psi0, np.complex128), 0
    for k in indices:
        if k != k0:
            cur = evolve_state(h, cur, (k - k0) * delta_t, tol, matvec)
            k0 = k
        out.append(cur.copy())
    return out


def ctqw_probability(psi: np.ndarray) -> np.ndarray:
    """|psi|^2 (ctqw.py:205-212)."""
    return np.abs(psi) ** 2


def default_threads() -> int:
    return os.cpu_count() or 1
