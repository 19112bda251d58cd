"""Multi-GPU decomposition checked on CPU.

1. The numpy model of the plane-layout step (tests/planes_model.py) equals the
   reference CSR step bitwise (so the model is a valid stand-in for the kernel).
2. The slab plan (paper_2406_08186_b200.distributed.slab_partition /
   neighbours) + the per-step two-row exchange reproduces the unsharded walk
   bitwise, with real processes exchanging rows over torch.distributed gloo
   (world sizes 2 and 3).  The GPU path runs the same plan with NCCL.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import planes_model as PM
from oracle import qwalk_oracle as O
from paper_2406_08186_b200 import distributed as DI


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _psi(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=n) + 1j * rng.normal(size=n)
    return v / np.linalg.norm(v)


@pytest.mark.parametrize("nx,ny,shift,marked", [(5, 5, "flipflop", ()), (7, 4, "persistent", (9,)),
                                                 (16, 12, "flipflop", (0, 37, 191)), (3, 3, "persistent", ())])
def test_planes_model_equals_reference_step(nx, ny, shift, marked):
    offs, cols = O.grid_adjacency(nx, ny)
    u = O.evolution_operator(offs, cols, shift, marked, "grid", (nx, ny, True))
    psi = _psi(4 * nx * ny, nx * ny)
    ref = O.coined_simulate(u, psi, [9])[0]
    got = PM.run_full(nx, ny, psi, 9, shift, marked)
    assert np.array_equal(got, ref)


def test_partition_plan():
    for ny, w in ((8, 2), (9, 2), (2048, 8), (10, 3), (6, 3)):
        parts = DI.slab_partition(ny, w)
        assert sum(r for _, r in parts) == ny
        assert all(r >= 2 for _, r in parts)
        assert [y for y, _ in parts] == list(np.cumsum([0] + [r for _, r in parts])[:-1])
        assert max(r for _, r in parts) - min(r for _, r in parts) <= 1
    assert DI.neighbours(0, 4) == (3, 1)
    assert DI.neighbours(3, 4) == (2, 0)
    with pytest.raises(Exception):
        DI.slab_partition(5, 3)
    assert DI.owned_arc_range(10, 2, 3) == (80, 200)


def test_slabs_single_process_equal_full():
    nx, ny = 6, 9
    psi = _psi(4 * nx * ny, 1)
    for shift in ("flipflop", "persistent"):
        full = PM.run_full(nx, ny, psi, 7, shift, (13,))
        for w in (2, 3, 4):
            parts = DI.slab_partition(ny, w)
            slabs = []
            for (y0, rows) in parts:
                lo, hi = DI.owned_arc_range(nx, y0, rows)
                slabs.append(PM.arcs_to_planes(nx, ny, psi[lo:hi], y0, rows, extra=1))
            for _ in range(7):
                slabs = [PM.step_slab(nx, ny, y0, rows, s, shift, (13,)) for s, (y0, rows) in zip(slabs, parts)]
                PM.exchange_local(slabs, shift)
            got = np.concatenate([PM.planes_to_arcs(nx, ny, s, y0, rows, extra=1)
                                  for s, (y0, rows) in zip(slabs, parts)])
            assert np.array_equal(got, full), (shift, w)


def _worker(rank, world, port, nx, ny, steps, shift, marked, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    psi = _psi(4 * nx * ny, 3)
    y0, rows = DI.slab_partition(ny, world)[rank]
    below, above = DI.neighbours(rank, world)
    pd, pu = PM.edge_planes(shift)
    lo, hi = DI.owned_arc_range(nx, y0, rows)
    planes = PM.arcs_to_planes(nx, ny, psi[lo:hi], y0, rows, extra=1)
    for _ in range(steps):
        planes = PM.step_slab(nx, ny, y0, rows, planes, shift, marked)
        # same pairing as comm.cu's NCCL group: send down / recv from up / send up / recv from down
        send_down = torch.from_numpy(planes[pd, 0, :].copy())
        send_up = torch.from_numpy(planes[pu, rows + 1, :].copy())
        recv_up = torch.empty_like(send_down)
        recv_down = torch.empty_like(send_up)
        ops = [dist.P2POp(dist.isend, send_down, below), dist.P2POp(dist.irecv, recv_up, above),
               dist.P2POp(dist.isend, send_up, above), dist.P2POp(dist.irecv, recv_down, below)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        planes[pd, rows, :] = recv_up.numpy()
        planes[pu, 1, :] = recv_down.numpy()
    local = PM.planes_to_arcs(nx, ny, planes, y0, rows, extra=1)
    np.save(os.path.join(out_dir, f"slab{rank}.npy"), local)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,shift", [(2, "flipflop"), (3, "persistent"), (2, "persistent")])
def test_gloo_multiprocess_halo_exchange(tmp_path, world, shift):
    import torch.multiprocessing as mp
    nx, ny, steps, marked = 8, 10, 6, (17, 44)
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, nx, ny, steps, shift, marked, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    got = np.concatenate([np.load(tmp_path / f"slab{r}.npy") for r in range(world)])
    offs, cols = O.grid_adjacency(nx, ny)
    u = O.evolution_operator(offs, cols, shift, marked, "grid", (nx, ny, True))
    ref = O.coined_simulate(u, _psi(4 * nx * ny, 3), [steps])[0]
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------------------
# hypercube CTQW shards: vertex v -> rank v >> (dim - S);
# per Taylor term each rank exchanges its term slice with partners r ^ 2^j
# and the stop test uses the all-gathered norm.  The model below runs that
# plan in real processes over gloo with the oracle's row arithmetic
# (oracle.csr_rows restates numpy's gather-multiply-reduceat), and must equal
# the oracle's single-process evolve bitwise.
# ---------------------------------------------------------------------------

def test_hypercube_plan():
    assert DI.hypercube_shard(12, 4, 2) == (2048, 3072)
    assert DI.hypercube_partners(5, 8) == [4, 7, 1]
    assert DI.hypercube_partners(0, 1) == []
    with pytest.raises(Exception):
        DI.hypercube_shard(12, 3, 0)          # not a power of two
    with pytest.raises(Exception):
        DI.hypercube_shard(11, 4, 0)          # shards < 2^10 vertices
    # every neighbour of a shard's vertex is local or in exactly one partner shard
    dim, world = 12, 4
    for r in range(world):
        lo, hi = DI.hypercube_shard(dim, world, r)
        owners = {((v ^ (1 << b)) >> (dim - 2)) for v in range(lo, hi, 97) for b in range(dim)}
        assert owners == {r, *DI.hypercube_partners(r, world)}


def _hc_worker(rank, world, port, dim, gamma, marked, t, out_dir):
    import math

    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    offs, cols = O.hypercube_adjacency(dim)
    h = O.hamiltonian(offs, cols, gamma, marked)
    n = 1 << dim
    psi = _psi(n, dim)
    lo, hi = DI.hypercube_shard(dim, world, rank)
    partners = DI.hypercube_partners(rank, world)
    cur = psi[lo:hi].copy()
    substeps = max(1, math.ceil(O.inf_norm(h) * abs(t)))
    tau = t / substeps
    floor = 1e-12 * float(np.linalg.norm(psi))
    view = np.zeros(n, dtype=np.complex128)
    terms = []
    for _ in range(substeps):
        acc, term = cur.copy(), cur.copy()
        for k in range(1, 1000):
            # exchange the term slice with every partner (one grouped round)
            send = torch.from_numpy(term.view(np.float64).copy())
            recvs = [torch.empty_like(send) for _ in partners]
            ops = []
            for p, rv in zip(partners, recvs):
                ops += [dist.P2POp(dist.isend, send, p), dist.P2POp(dist.irecv, rv, p)]
            for r in (dist.batch_isend_irecv(ops) if ops else []):
                r.wait()
            view[lo:hi] = term
            for p, rv in zip(partners, recvs):
                plo, phi = DI.hypercube_shard(dim, world, p)
                view[plo:phi] = rv.numpy().view(np.complex128)
            hterm = O.csr_rows(h, view, lo, hi)
            term = complex(-1j * tau / k) * hterm
            acc = acc + complex(1.0) * term
            parts = [None] * world
            dist.all_gather_object(parts, float(np.vdot(term, term).real))
            if math.sqrt(sum(parts)) <= floor:
                terms.append(k)
                break
        cur = acc
    np.save(os.path.join(out_dir, f"shard{rank}.npy"), cur)
    np.save(os.path.join(out_dir, f"terms{rank}.npy"), np.array(terms))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,marked", [(2, (3, 1500)), (4, (0,))])
def test_gloo_multiprocess_hypercube_shards(tmp_path, world, marked):
    import torch.multiprocessing as mp
    dim, gamma, t = 12, 1.0 / 12, 0.8
    port = _free_port()
    mp.start_processes(_hc_worker, args=(world, port, dim, gamma, marked, t, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    got = np.concatenate([np.load(tmp_path / f"shard{r}.npy") for r in range(world)])
    terms = [list(np.load(tmp_path / f"terms{r}.npy")) for r in range(world)]
    assert all(tr == terms[0] for tr in terms)
    offs, cols = O.hypercube_adjacency(dim)
    stats = []
    ref = O.evolve_state(O.hamiltonian(offs, cols, gamma, marked), _psi(1 << dim, dim), t, stats=stats)
    assert terms[0] == stats
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------------------
# generic-graph CSR rows: contiguous nnz-balanced row ranges,
# columns renumbered into [own | halo], per-step exchange of exactly the halo
# entries (precomputed lists), then the local rows -- over gloo, vs the oracle
# ---------------------------------------------------------------------------

def _generic_u(n=120, seed=3):
    rng = np.random.default_rng(seed)
    edges = sorted({(min(a, b), max(a, b)) for a, b in rng.integers(0, n, size=(400, 2)) if a != b})
    offs, cols = O.edges_adjacency(n, edges)
    return O.evolution_operator(offs, cols, "flipflop", (5, 77))


def test_csr_partition_plan():
    u = _generic_u()
    for world in (1, 2, 3, 7):
        shards = DI.csr_partition(u.row_offsets, u.col_indices, u.values, world)
        assert shards[0].r0 == 0 and shards[-1].r1 == u.n_rows
        assert all(a.r1 == b.r0 for a, b in zip(shards, shards[1:]))
        nnz = [int(s.row_offsets[-1]) for s in shards]
        assert max(nnz) - min(nnz) <= 2 * int(np.diff(u.row_offsets).max()) + u.nnz // world // 4 + 4
        x = _psi(u.n_rows, world)
        ref = O.csr_rows(u, x, 0, u.n_rows)
        got = []
        for sh in shards:
            xe = np.concatenate([x[sh.r0:sh.r1], x[sh.halo]])
            got.append(O.csr_rows(O.Csr(sh.n_local, xe.size, sh.row_offsets, sh.col, sh.values), xe, 0, sh.n_local))
            assert sh.rank not in sh.peers
        assert np.array_equal(np.concatenate(got), ref)


def _csr_worker(rank, world, port, steps, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    u = _generic_u()
    sh = DI.csr_partition(u.row_offsets, u.col_indices, u.values, world)[rank]
    x = _psi(u.n_rows, 11)[sh.r0:sh.r1].copy()
    m = O.Csr(sh.n_local, sh.n_local + len(sh.halo), sh.row_offsets, sh.col, sh.values)
    offs = np.concatenate([[0], np.cumsum(sh.recv_counts)])
    for _ in range(steps):
        ops, recvs = [], {}
        for q in sh.peers:       # same pairing as qwb_csr_halo_exchange's NCCL group
            if len(sh.send_idx[q]):
                ops.append(dist.P2POp(dist.isend, torch.from_numpy(x[sh.send_idx[q]].view(np.float64).copy()), q))
            if sh.recv_counts[q]:
                recvs[q] = torch.empty(2 * int(sh.recv_counts[q]), dtype=torch.float64)
                ops.append(dist.P2POp(dist.irecv, recvs[q], q))
        for r in (dist.batch_isend_irecv(ops) if ops else []):
            r.wait()
        xe = np.concatenate([x, np.zeros(len(sh.halo), complex)])
        for q, t in recvs.items():
            xe[sh.n_local + offs[q]: sh.n_local + offs[q + 1]] = t.numpy().view(np.complex128)
        x = O.csr_rows(m, xe, 0, sh.n_local)
    np.save(os.path.join(out_dir, f"csr{rank}.npy"), x)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_multiprocess_csr_halo(tmp_path, world):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_csr_worker, args=(world, port, 9, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    got = np.concatenate([np.load(tmp_path / f"csr{r}.npy") for r in range(world)])
    u = _generic_u()
    ref = O.coined_simulate(u, _psi(u.n_rows, 11), [9])[0]
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------------------
# fused lattice slabs (qwb_slab_run_fused): G ghost state rows each side, G
# steps per exchange (single steps for the remainder), over gloo, vs the oracle
# ---------------------------------------------------------------------------

def _ghost_worker(rank, world, port, nx, ny, G, steps, shift, marked, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    psi = _psi(4 * nx * ny, 21)
    y0, rows = DI.slab_partition(ny, world)[rank]
    below, above = DI.neighbours(rank, world)
    lo, hi = DI.owned_arc_range(nx, y0, rows)
    win = PM.ghost_window(nx, ny, psi[lo:hi], y0, rows, G)
    k = 0
    while k < steps:
        g = G if k + G <= steps else 1
        down, up = PM.ghost_sends(win, rows, G, g)
        from_above = torch.empty(down.shape, dtype=torch.complex128)
        from_below = torch.empty(up.shape, dtype=torch.complex128)
        # comm.cu's pairing: send down / recv from above / send up / recv from below
        ops = [dist.P2POp(dist.isend, torch.from_numpy(down), below), dist.P2POp(dist.irecv, from_above, above),
               dist.P2POp(dist.isend, torch.from_numpy(up), above), dist.P2POp(dist.irecv, from_below, below)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        win = PM.ghost_receive(win, rows, G, g, from_above.numpy(), from_below.numpy())
        win = PM.ghost_steps(nx, ny, y0, rows, G, win, g, shift, marked)
        k += g
    np.save(os.path.join(out_dir, f"ghost{rank}.npy"), PM.planes_to_arcs(nx, ny, win, y0, rows, extra=G))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,G,shift", [(2, 4, "flipflop"), (2, 8, "flipflop"), (3, 3, "persistent"), (2, 2, "flipflop")])
def test_gloo_multiprocess_ghost_slabs(tmp_path, world, G, shift):
    import torch.multiprocessing as mp
    nx, ny, steps, marked = 8, 18, 11, (17, 100)
    port = _free_port()
    mp.start_processes(_ghost_worker, args=(world, port, nx, ny, G, steps, shift, marked, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    got = np.concatenate([np.load(tmp_path / f"ghost{r}.npy") for r in range(world)])
    offs, cols = O.grid_adjacency(nx, ny)
    u = O.evolution_operator(offs, cols, shift, marked, "grid", (nx, ny, True))
    assert np.array_equal(got, O.coined_simulate(u, _psi(4 * nx * ny, 21), [steps])[0])
