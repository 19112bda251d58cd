"""Multi-GPU walks: a periodic lattice split into y-slabs (coined walk), and a
hypercube split into 2^S vertex shards (continuous-time walk).

No reference counterpart (the reference's only parallelism is the in-process
row-block pool, backend.py:426-430; multi-GPU is future work).

Plumbing: one process per GPU (torchrun), `torch.distributed` only to agree on
the NCCL unique id; the per-step halo exchange runs inside libqwb200
(`qwb_slab_run`: NCCL send/recv of two nx-long rows on a comm stream,
overlapped with the interior rows).  Results are bitwise equal to the
single-GPU run because every arc is computed with the same formula and the
position classes use global coordinates.

The hypercube CTQW shards vertex v to rank v >> (dim - S):
every Taylor term exchanges the local term slice with the S partner ranks
r ^ 2^j (NCCL grouped send/recv inside `qwb_taylor_evolve_hypercube_sharded`)
and all-gathers one float64 for the stop test; NVLink-bound by construction
(S x 16 B x 2^(dim-S) per rank per term against ~64 B x 2^(dim-S) of HBM).

Any other graph (SURVEY §8(e) "generic-graph CSR"): the rows of U (= arcs,
reference order) are split into contiguous, nnz-balanced ranges; each rank
keeps its rows with columns renumbered into an extended vector [own entries |
halo], and per step receives exactly the halo entries its rows read from each
peer (precomputed send/recv index lists, one NCCL group), then runs the CSR
SpMV kernel on its rows: the single-GPU arithmetic, so bitwise equal.

The plans (`slab_partition`, `neighbours`, `hypercube_shard`,
`hypercube_partners`, `csr_partition`) are plain Python so they are tested on
CPU with the gloo backend (tests/test_distributed_cpu.py).
"""

from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

from . import _native as N
from .backend import Engine, empty_z
from .errors import DimensionMismatch


def slab_partition(ny: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced y-slabs [(y0, rows)], every slab >= 2 rows."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if ny < 2 * world:
        raise DimensionMismatch(f"ny={ny} too small for {world} slabs of >= 2 rows")
    base, extra = divmod(ny, world)
    out, y = [], 0
    for r in range(world):
        rows = base + (1 if r < extra else 0)
        out.append((y, rows))
        y += rows
    return out


def neighbours(rank: int, world: int) -> tuple[int, int]:
    """(rank below, rank above) on the periodic y ring."""
    return (rank - 1) % world, (rank + 1) % world


def owned_arc_range(nx: int, y0: int, rows: int) -> tuple[int, int]:
    """Arcs of rows [y0, y0+rows) in the reference order: contiguous, 4 per vertex."""
    return 4 * nx * y0, 4 * nx * (y0 + rows)


def _nccl_path() -> str | None:
    try:
        import nvidia.nccl
        for base in list(getattr(nvidia.nccl, "__path__", [])):
            p = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p
    except Exception:
        pass
    return None


def hypercube_shard(dim: int, world: int, rank: int) -> tuple[int, int]:
    """Vertex range [lo, hi) of `rank` when hypercube(dim) is split over
    `world` = 2^S ranks: the vertices whose top S bits equal rank."""
    S = _log2_world(world)
    if dim - S < 10:
        raise DimensionMismatch(f"hypercube({dim}) over {world} ranks leaves shards < 2^10 vertices")
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} not in 0..{world - 1}")
    n = 1 << (dim - S)
    return rank * n, (rank + 1) * n


def hypercube_partners(rank: int, world: int) -> list[int]:
    """Ranks holding the neighbours across each rank bit j: rank ^ 2^j."""
    return [rank ^ (1 << j) for j in range(_log2_world(world))]


def _log2_world(world: int) -> int:
    if world < 1 or world & (world - 1):
        raise ValueError(f"world size {world} is not a power of two")
    return world.bit_length() - 1


class CsrShard:
    """One rank's part of a row-partitioned CSR operator (host arrays).

    rows [r0, r1) of the global matrix; `row_offsets` rebased to 0, `col`
    renumbered: own column c -> c - r0, halo column -> n_local + its position
    in `halo` (sorted by owner rank, then column).  `recv_counts[q]` halo
    entries come from rank q; `send_idx[q]` are the local indices rank q
    reads from this rank (in rank q's halo order)."""

    __slots__ = ("rank", "r0", "r1", "row_offsets", "col", "values", "halo", "recv_counts", "send_idx")

    def __init__(self, **kw):
        for k, v in kw.items():
            setattr(self, k, v)

    @property
    def n_local(self) -> int:
        return self.r1 - self.r0

    @property
    def peers(self) -> list[int]:
        """ranks exchanged with (either direction), ascending"""
        return sorted({q for q, c in enumerate(self.recv_counts) if c} |
                      {q for q, ix in enumerate(self.send_idx) if len(ix)})


def csr_row_ranges(row_offsets: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous row ranges with about nnz / world entries each (every range
    non-empty when there are at least `world` rows)."""
    n = int(row_offsets.shape[0] - 1)
    if world < 1:
        raise ValueError("world must be >= 1")
    if n < world:
        raise DimensionMismatch(f"{n} rows cannot be split over {world} ranks")
    nnz = int(row_offsets[-1])
    cuts = [0]
    for r in range(1, world):
        c = int(np.searchsorted(row_offsets, nnz * r / world, side="left"))
        c = min(max(c, cuts[-1] + 1), n - (world - r))
        cuts.append(c)
    cuts.append(n)
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


def csr_partition(row_offsets, col_indices, values, world: int) -> list[CsrShard]:
    """Split a CSR matrix (square, global columns) row-wise over `world` ranks
    with the halo lists of every rank."""
    row_offsets = np.asarray(row_offsets, dtype=np.int64)
    col_indices = np.asarray(col_indices, dtype=np.int64)
    ranges = csr_row_ranges(row_offsets, world)
    starts = np.array([r0 for r0, _ in ranges], dtype=np.int64)
    owner_of = lambda cols: np.searchsorted(starts, cols, side="right") - 1   # noqa: E731
    shards = []
    for rank, (r0, r1) in enumerate(ranges):
        lo, hi = int(row_offsets[r0]), int(row_offsets[r1])
        cols = col_indices[lo:hi]
        own = (cols >= r0) & (cols < r1)
        ext = np.unique(cols[~own])                      # sorted global halo columns
        owners = owner_of(ext)
        order = np.lexsort((ext, owners))                # by owner rank, then column
        halo, owners = ext[order], owners[order]
        pos = np.empty(0, dtype=np.int64) if halo.size == 0 else None
        local = np.empty(cols.shape[0], dtype=np.int64)
        local[own] = cols[own] - r0
        if halo.size:
            # halo position of every remote column
            sorter = np.argsort(halo)
            pos = sorter[np.searchsorted(halo, cols[~own], sorter=sorter)]
            local[~own] = (r1 - r0) + pos
        recv_counts = np.bincount(owners, minlength=world).astype(np.int64)
        shards.append(CsrShard(rank=rank, r0=r0, r1=r1,
                               row_offsets=row_offsets[r0:r1 + 1] - lo, col=local,
                               values=np.asarray(values)[lo:hi], halo=halo, recv_counts=recv_counts,
                               send_idx=[None] * world))
    # what each rank sends: the entries the others' halos list, in their order
    for sh in shards:
        offs = np.concatenate([[0], np.cumsum(sh.recv_counts)])
        for q in range(world):
            want = sh.halo[offs[q]:offs[q + 1]]
            shards[q].send_idx[sh.rank] = (want - shards[q].r0).astype(np.int64)
    for sh in shards:
        sh.send_idx = [np.zeros(0, np.int64) if ix is None else ix for ix in sh.send_idx]
    return shards


class _DeviceCsrShard:
    """A CsrShard on the device: local CSR (int32 renumbered columns), the
    ping-pong extended vectors and the exchange lists."""

    def __init__(self, engine: Engine, sh: CsrShard):
        import torch
        from .backend import DeviceCsr, to_device
        self.engine, self.sh = engine, sh
        n_ext = sh.n_local + len(sh.halo)
        dev = engine.torch_device
        self.csr = DeviceCsr(sh.n_local, n_ext, to_device(engine, sh.row_offsets),
                             torch.from_numpy(sh.col.astype(np.int32)).to(dev),
                             to_device(engine, np.ascontiguousarray(sh.values, dtype=np.complex128)))
        self.x = empty_z(engine, max(1, n_ext))
        self.y = empty_z(engine, max(1, n_ext))
        self.peers = sh.peers
        send = [sh.send_idx[q] for q in self.peers]
        self.send_off = np.concatenate([[0], np.cumsum([len(i) for i in send])]).astype(np.int64)
        rc = [int(sh.recv_counts[q]) for q in self.peers]
        self.recv_off = np.concatenate([[0], np.cumsum(rc)]).astype(np.int64)
        flat = np.concatenate(send) if send else np.zeros(0, np.int64)
        self.send_idx = torch.from_numpy(flat.astype(np.int64)).to(dev) if flat.size else None
        self.send_buf = empty_z(engine, max(1, int(self.send_off[-1])))

    def step_local(self):
        """y[:n_local] = local rows of U applied to x (halo already in place)."""
        from .backend import spmv_device
        spmv_device(self.engine, self.csr, self.x, self.y)
        self.x, self.y = self.y, self.x


class ShardedCsrWalk:
    """This rank's rows of a coined walk on any graph (U built on the device,
    partitioned by `csr_partition`), NCCL halo exchange per step.  For
    lattices use SlabLattice (matrix-free).  Call collectively."""

    def __init__(self, engine: Engine, spec, rank: int = 0, world: int = 1, group=None,
                 comm: bool | None = None):
        from . import coined as CO
        self.engine, self.rank, self.world = engine, int(rank), int(world)
        self.comm = self.world > 1 if comm is None else bool(comm)
        u = CO.device_operator(engine, spec.graph, spec.shift, spec.active_marked).to_host()
        self.shards = csr_partition(u.row_offsets, u.col_indices, u.values, self.world)
        self.local = _DeviceCsrShard(engine, self.shards[self.rank])
        self.r0, self.r1 = self.local.sh.r0, self.local.sh.r1
        if self.comm:
            _init_comm(engine, self.rank, self.world, group)

    def load(self, owned_arcs) -> None:
        """owned_arcs: device tensor of this rank's arcs [r0, r1) (reference order)."""
        self.local.x[: self.local.sh.n_local].copy_(owned_arcs)

    def advance(self, steps: int) -> None:
        L = self.local
        peers = (C.c_int * max(1, len(L.peers)))(*L.peers)
        for _ in range(int(steps)):
            if self.comm:
                self.engine.call("qwb_csr_halo_exchange", L.sh.n_local, N.ptr(L.x), N.ptr(L.send_idx),
                                 L.send_off.ctypes.data_as(N._p_i64), L.recv_off.ctypes.data_as(N._p_i64),
                                 peers, len(L.peers), N.ptr(L.send_buf), self.engine.stream())
            L.step_local()

    def store(self, owned_arcs) -> None:
        owned_arcs.copy_(self.local.x[: self.local.sh.n_local])

    def close(self) -> None:
        if self.comm:
            self.engine.call("qwb_comm_destroy")


def emulate_csr_shards(engine: Engine, spec, world: int, psi: np.ndarray, steps: int) -> np.ndarray:
    """The generic-graph row partition for `world` ranks on ONE device: the
    halo lists are applied with device gathers in place of the NCCL group,
    each shard stepped by the CSR kernel on its renumbered rows.  Returns the
    full arc state.  Test hook for the multi-GPU generic-graph path."""
    import torch
    from . import coined as CO
    u = CO.device_operator(engine, spec.graph, spec.shift, spec.active_marked).to_host()
    shards = csr_partition(u.row_offsets, u.col_indices, u.values, world)
    dev = [_DeviceCsrShard(engine, sh) for sh in shards]
    full = torch.from_numpy(np.ascontiguousarray(psi, dtype=np.complex128)).to(engine.torch_device)
    for d in dev:
        d.x[: d.sh.n_local].copy_(full[d.sh.r0:d.sh.r1])
    idx = [[torch.from_numpy(d.sh.send_idx[q]).to(engine.torch_device) for q in range(world)] for d in dev]
    for _ in range(int(steps)):
        for i, d in enumerate(dev):           # halo of shard i, ordered by owner rank
            parts = [dev[q].x[idx[q][i]] for q in range(world) if d.sh.recv_counts[q]]
            if parts:
                d.x[d.sh.n_local: d.sh.n_local + len(d.sh.halo)].copy_(torch.cat(parts))
        for d in dev:
            d.step_local()
    return torch.cat([d.x[: d.sh.n_local] for d in dev]).cpu().numpy()


def _init_comm(engine: Engine, rank: int, world: int, group=None) -> None:
    """NCCL communicator inside libqwb200 (torch.distributed only carries the id)."""
    import torch.distributed as dist
    lib = N.load()
    path = _nccl_path()
    if path and not os.environ.get("QWB_NCCL_LIB"):
        os.environ["QWB_NCCL_LIB"] = path
    uid = C.create_string_buffer(128)
    if rank == 0:
        N.check(lib.qwb_comm_unique_id(uid))
    obj = [uid.raw if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = C.create_string_buffer(obj[0], 128)
    engine.call("qwb_comm_init", uid, world, rank)
    if os.environ.get("QWB_LOG_COMM"):
        import sys
        print(f"qwb: NCCL communicator initialised: rank {rank} nranks {world} device {engine.device}",
              file=sys.stderr, flush=True)


def _hypercube_setup(engine: Engine, dim: int, gamma: float, marked):
    import torch
    from . import ctqw as CT
    marked = sorted(int(v) for v in marked)
    n = 1 << dim
    for v in marked:
        if not (0 <= v < n):
            from .errors import MarkedVertexOutOfRange
            raise MarkedVertexOutOfRange(f"marked vertex {v} not in 0..{n - 1}")
    bits = None
    if marked:
        bits = torch.empty((n + 31) // 32, dtype=torch.int32, device=engine.torch_device)
        mk = torch.tensor(marked, dtype=torch.int64, device=engine.torch_device)
        engine.call("qwb_marked_bitmap", n, N.ptr(mk), len(marked), N.ptr(bits), engine.stream())
    inf_norm = CT._inf_norm_hypercube(engine, dim, float(gamma), marked)
    return bits, inf_norm


class ShardedHypercubeWalk:
    """This rank's shard of a continuous-time walk on hypercube(dim),
    H = -gamma A - sum_M |v><v| (ctqw.py:84-98).  Call collectively."""

    def __init__(self, engine: Engine, dim: int, gamma: float, marked=(), rank: int = 0, world: int = 1,
                 group=None, comm: bool | None = None):
        self.engine = engine
        self.dim, self.gamma = int(dim), float(gamma)
        self.rank, self.world = int(rank), int(world)
        self.comm = self.world > 1 if comm is None else bool(comm)
        self.S = _log2_world(self.world)
        self.lo, self.hi = hypercube_shard(self.dim, self.world, self.rank)
        self.n_local = self.hi - self.lo
        self.group = group
        if self.world > 1 and not self.comm:
            # the single-GPU kernel needs the whole 2^dim state; a shard holds
            # 2^(dim-S) entries (emulate_hypercube_shards runs shards locally)
            raise ValueError("ShardedHypercubeWalk with world > 1 needs comm=True")
        self.bits, self.inf_norm = _hypercube_setup(engine, self.dim, self.gamma, marked)
        self.work = empty_z(engine, (3 + self.S) * self.n_local)
        if self.comm:
            _init_comm(engine, self.rank, self.world, group)

    def global_norm(self, psi_local) -> float:
        from .backend import device_norm
        local = device_norm(self.engine, psi_local) ** 2
        if self.world == 1:
            return math.sqrt(local)
        import torch.distributed as dist
        parts = [None] * self.world
        dist.all_gather_object(parts, local, group=self.group)
        return math.sqrt(sum(parts))

    def evolve(self, psi_local, t: float, tol: float = 1e-12) -> list[int]:
        """psi_local (device, in place) <- this rank's slice of exp(-iHt) psi;
        returns the term count of each sub-step (the same on every rank)."""
        from . import ctqw as CT
        if t == 0:
            return []
        substeps = max(1, math.ceil(self.inf_norm * abs(t)))
        tau = t / substeps
        floor = tol * self.global_norm(psi_local)
        terms = (C.c_int * substeps)()
        eng = self.engine
        if not self.comm:
            eng.call("qwb_taylor_evolve_hypercube", self.dim, self.gamma, N.ptr(self.bits), N.ptr(psi_local),
                     N.ptr(self.work), substeps, tau, floor, int(CT._MAX_SERIES_TERMS), terms, eng.stream())
        else:
            eng.call("qwb_taylor_evolve_hypercube_sharded", self.dim, self.S, self.gamma, N.ptr(self.bits),
                     N.ptr(psi_local), N.ptr(self.work), substeps, tau, floor, int(CT._MAX_SERIES_TERMS),
                     terms, eng.stream())
        return list(terms)

    def close(self) -> None:
        if self.comm:
            self.engine.call("qwb_comm_destroy")


def emulate_hypercube_shards(engine: Engine, dim: int, gamma: float, marked, world: int, psi: np.ndarray,
                             t: float, tol: float = 1e-12):
    """Run the hypercube shard decomposition for `world` shards on ONE device
    (partner slices read in place of the NCCL exchange); returns (full state,
    terms per sub-step).  Test hook for the multi-GPU CTQW path."""
    import torch
    from . import ctqw as CT
    S = _log2_world(world)
    bits, inf_norm = _hypercube_setup(engine, dim, gamma, marked)
    full = torch.from_numpy(np.ascontiguousarray(psi, dtype=np.complex128)).to(engine.torch_device)
    nl = (1 << dim) >> S
    shards = [full[r * nl:(r + 1) * nl].clone() for r in range(world)]
    works = [empty_z(engine, 3 * nl) for _ in range(world)]
    substeps = max(1, math.ceil(inf_norm * abs(t)))
    tau = t / substeps
    floor = tol * float(np.linalg.norm(psi))
    terms = (C.c_int * substeps)()
    ps = (C.c_void_p * world)(*[N.ptr(x) for x in shards])
    ws = (C.c_void_p * world)(*[N.ptr(x) for x in works])
    engine.call("qwb_taylor_evolve_hypercube_shards_local", dim, S, float(gamma), N.ptr(bits), ps, ws, substeps,
                tau, floor, int(CT._MAX_SERIES_TERMS), terms, engine.stream())
    return torch.cat(shards).cpu().numpy(), list(terms)


class SlabLattice:
    """This rank's slab of a periodic nx x ny lattice walk (flip-flop or
    persistent shift, optional marked vertices).  Call collectively."""

    def __init__(self, engine: Engine, nx: int, ny: int, shift: str = "flipflop", marked=(),
                 rank: int = 0, world: int = 1, group=None, comm: bool | None = None):
        import torch
        self.engine = engine
        self.nx, self.ny = int(nx), int(ny)
        self.rank, self.world = int(rank), int(world)
        # comm: run through the NCCL exchange (default when world > 1; with
        # world == 1 the single slab exchanges with itself = the torus wrap)
        self.comm = self.world > 1 if comm is None else bool(comm)
        self.y0, self.rows = slab_partition(self.ny, self.world)[self.rank]
        self.below, self.above = neighbours(self.rank, self.world)
        self.shift = N.SHIFT[shift]
        self.bits = None
        self.marked = sorted(int(v) for v in marked)
        self.marked_arr = N.i64_array(self.marked)
        if marked:
            n = self.nx * self.ny
            self.bits = torch.empty((n + 31) // 32, dtype=torch.int32, device=engine.torch_device)
            mk = torch.tensor(self.marked, dtype=torch.int64, device=engine.torch_device)
            engine.call("qwb_marked_bitmap", n, N.ptr(mk), len(marked), N.ptr(self.bits), engine.stream())
        # fused path: G = 4T ghost state rows each side, G steps per temporally
        # blocked launch (the same G on every rank: from the smallest slab)
        self.ghost = slab_ghost_rows(self.nx, self.ny, self.world, len(self.marked))
        size = 4 * self.nx * (self.rows + 2 * (self.ghost or 1))
        self.a = empty_z(engine, size)
        self.b = empty_z(engine, size)
        self.a.zero_()
        self.b.zero_()
        if self.comm:
            _init_comm(engine, self.rank, self.world, group)

    def load(self, owned_arcs) -> None:
        """owned_arcs: device tensor of this slab's arcs (reference order)."""
        if self.ghost:
            self.engine.call("qwb_slab_to_planes_g", self.nx, self.ny, self.y0, self.rows, self.ghost,
                             N.ptr(owned_arcs), N.ptr(self.a), self.engine.stream())
        else:
            self.engine.call("qwb_slab_to_planes", self.nx, self.ny, self.y0, self.rows, N.ptr(owned_arcs),
                             N.ptr(self.a), self.engine.stream())

    def advance(self, steps: int) -> None:
        if steps <= 0:
            return
        eng = self.engine
        if not self.comm:
            raise RuntimeError("use the single-GPU lattice path for world == 1 (or comm=True)")
        flag = C.c_int(0)
        if self.ghost:
            eng.call("qwb_slab_run_fused", self.nx, self.ny, self.y0, self.rows, self.ghost, self.shift,
                     N.ptr(self.bits), self.marked_arr, len(self.marked), N.ptr(self.a), N.ptr(self.b), int(steps),
                     self.below, self.above, C.byref(flag), eng.stream())
        else:
            eng.call("qwb_slab_run", self.nx, self.ny, self.y0, self.rows, self.shift, N.ptr(self.bits),
                     N.ptr(self.a), N.ptr(self.b), int(steps), self.below, self.above, C.byref(flag),
                     eng.stream())
        if flag.value:
            self.a, self.b = self.b, self.a

    def store(self, owned_arcs) -> None:
        if self.ghost:
            self.engine.call("qwb_slab_from_planes_g", self.nx, self.ny, self.y0, self.rows, self.ghost,
                             N.ptr(self.a), N.ptr(owned_arcs), self.engine.stream())
        else:
            self.engine.call("qwb_slab_from_planes", self.nx, self.ny, self.y0, self.rows, N.ptr(self.a),
                             N.ptr(owned_arcs), self.engine.stream())

    def probability(self, p) -> None:
        if self.ghost:
            self.engine.call("qwb_slab_probability_g", self.nx, self.ny, self.y0, self.rows, self.ghost,
                             N.ptr(self.a), N.ptr(p), self.engine.stream())
        else:
            self.engine.call("qwb_slab_probability", self.nx, self.ny, self.y0, self.rows, N.ptr(self.a),
                             N.ptr(p), self.engine.stream())

    def close(self) -> None:
        if self.comm:
            self.engine.call("qwb_comm_destroy")


def slab_depth() -> int:
    """T, the coined steps per temporally blocked slab launch (kSlabDepth)."""
    t = C.c_int(0)
    N.check(N.load().qwb_slab_depth(C.byref(t)))
    return int(t.value)


def slab_ghost_rows(nx: int, ny: int, world: int, n_marked: int) -> int:
    """Ghost rows G of the fused (temporally blocked) slab path, 0 when it is
    not available (tiny lattices, slabs thinner than G rows, or
    QWB_SLAB_FUSED=0).  Identical on every rank."""
    if os.environ.get("QWB_SLAB_FUSED", "1") == "0":
        return 0
    min_rows = min(r for _, r in slab_partition(ny, world))
    g = C.c_int(0)
    N.check(N.load().qwb_slab_ghost_rows(nx, ny, min_rows, n_marked, C.byref(g)))
    return int(g.value)


def emulate_slabs_fused(engine: Engine, nx: int, ny: int, world: int, psi_arcs: np.ndarray, steps: int,
                        shift: str = "flipflop", marked=()):
    """The fused slab decomposition (G ghost state rows, G steps per
    exchange as G / T temporally blocked launches, single pull steps for the remainder) for
    `world` slabs on ONE device, exchanging ghost rows with device copies
    exactly as qwb_slab_run_fused's NCCL group does.  Returns the full arc
    state.  Test hook for the multi-GPU path."""
    import torch
    parts = slab_partition(ny, world)
    sh = N.SHIFT[shift]
    marked = sorted(int(v) for v in marked)
    G = slab_ghost_rows(nx, ny, world, len(marked))
    if G == 0:
        raise ValueError("the fused slab path is not available for this lattice")
    bits = None
    if marked:
        n = nx * ny
        bits = torch.empty((n + 31) // 32, dtype=torch.int32, device=engine.torch_device)
        mk = torch.tensor(marked, dtype=torch.int64, device=engine.torch_device)
        engine.call("qwb_marked_bitmap", n, N.ptr(mk), len(marked), N.ptr(bits), engine.stream())
    marr = N.i64_array(marked)
    full = torch.from_numpy(np.ascontiguousarray(psi_arcs)).to(engine.torch_device)
    cur, nxt = [], []
    for (y0, rows) in parts:
        a = empty_z(engine, 4 * nx * (rows + 2 * G)).zero_()
        b = empty_z(engine, 4 * nx * (rows + 2 * G)).zero_()
        lo, hi = owned_arc_range(nx, y0, rows)
        engine.call("qwb_slab_to_planes_g", nx, ny, y0, rows, G, N.ptr(full[lo:hi]), N.ptr(a), engine.stream())
        cur.append(a)
        nxt.append(b)
    nl = N.i64_array([r for (_, r) in parts])
    T = slab_depth()   # G = m T

    def launch(nsteps, ext):
        nonlocal cur, nxt
        for i, (y0, rows) in enumerate(parts):
            engine.call("qwb_slab_advance_local", nx, ny, y0, rows, G, sh, N.ptr(bits), marr, len(marked),
                        N.ptr(cur[i]), N.ptr(nxt[i]), nsteps, ext, engine.stream())
        cur, nxt = nxt, cur

    # qwb_slab_run_fused's schedule: per exchange of g = jT rows, j launches
    # over the owned rows extended by (j-1)T, ..., 0 rows; then single steps
    k = 0
    while k < steps:
        g = min(G, (steps - k) // T * T) or 1
        ptrs = (C.c_void_p * world)(*[N.ptr(t) for t in cur])
        engine.call("qwb_slab_ghost_exchange_local", nx, G, g, nl, ptrs, world, engine.stream())
        if g == 1:
            launch(1, 0)
        else:
            for ext in range(g - T, -1, -T):
                launch(T, ext)
        k += g
    out = torch.empty_like(full)
    for i, (y0, rows) in enumerate(parts):
        lo, hi = owned_arc_range(nx, y0, rows)
        engine.call("qwb_slab_from_planes_g", nx, ny, y0, rows, G, N.ptr(cur[i]), N.ptr(out[lo:hi]), engine.stream())
    return out.cpu().numpy()


def emulate_slabs(engine: Engine, nx: int, ny: int, world: int, psi_arcs: np.ndarray, steps: int,
                  shift: str = "flipflop", marked=()):
    """Run the slab decomposition for `world` slabs on ONE device (slab kernel
    + the same two-row exchange as qwb_slab_run, done with device copies) and
    return the full arc state.  Test hook for the multi-GPU path."""
    import torch
    parts = slab_partition(ny, world)
    sh = N.SHIFT[shift]
    bits = None
    if marked:
        n = nx * ny
        bits = torch.empty((n + 31) // 32, dtype=torch.int32, device=engine.torch_device)
        mk = torch.tensor(sorted(marked), dtype=torch.int64, device=engine.torch_device)
        engine.call("qwb_marked_bitmap", n, N.ptr(mk), len(marked), N.ptr(bits), engine.stream())
    full = torch.from_numpy(np.ascontiguousarray(psi_arcs)).to(engine.torch_device)
    cur, nxt = [], []
    for (y0, rows) in parts:
        a = empty_z(engine, 4 * nx * (rows + 2)).zero_()
        b = empty_z(engine, 4 * nx * (rows + 2)).zero_()
        lo, hi = owned_arc_range(nx, y0, rows)
        engine.call("qwb_slab_to_planes", nx, ny, y0, rows, N.ptr(full[lo:hi]), N.ptr(a), engine.stream())
        cur.append(a)
        nxt.append(b)
    nl = N.i64_array([r for (_, r) in parts])
    for _ in range(steps):
        for i, (y0, rows) in enumerate(parts):
            engine.call("qwb_slab_step", nx, ny, y0, rows, sh, N.ptr(bits), N.ptr(cur[i]), N.ptr(nxt[i]), 0,
                        engine.stream())
        ptrs = (C.c_void_p * world)(*[N.ptr(t) for t in nxt])
        engine.call("qwb_slab_exchange_local", nx, sh, nl, ptrs, world, engine.stream())
        cur, nxt = nxt, cur
    out = torch.empty_like(full)
    for i, (y0, rows) in enumerate(parts):
        lo, hi = owned_arc_range(nx, y0, rows)
        engine.call("qwb_slab_from_planes", nx, ny, y0, rows, N.ptr(cur[i]), N.ptr(out[lo:hi]), engine.stream())
    return out.cpu().numpy()
