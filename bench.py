#!/usr/bin/env python
"""Benchmark: coined Grover walk on a 2-D torus, arc-amplitude updates/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1], "2D Lattice ... (4M vertices, 16M arcs),
1000 steps"; the vertex/arc counts are those of 2048 x 2048):
grid(2048, 2048) torus, flip-flop shift, Grover coin, dense random psi0
(seed 0).  One bench step = 1000 coined-walk steps.  On N > 1 GPUs (torchrun)
the lattice is 2048 x (2048 N), split into y-slabs with an NCCL halo exchange
every step (weak scaling); the whole-job value is the sum over ranks, timed
as the max over ranks.

JSON line keys beyond the base contract:
  roofline      dominant kernel (the temporally blocked lattice kernel: T
                coined steps per launch): algorithmic 32 B per arc-step x the
                arc-steps of one launch, CUDA-event time per launch over the
                timed region, against the measured HBM copy peak
                (MEASURED_PEAKS.json); compulsory (once-per-launch) bytes beside
  cpu_baseline  the reference algorithm (oracle/ numpy port of backend._csr_rows
                with the reference's row-block thread pool) on this host
  e2e           the public API call coined.simulate(engine, spec, (1000,1001,1),
                psi0) with host (pinned) psi0 in and the host result out
  also          secondary measurements: 4096^2 (C3 size, the north-star 70 %
                gate) and the device CSR SpMV path (K1) at 2048^2
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "arc-amplitude updates/sec per coined-walk step (2D lattice); % of HBM roofline"
UNIT = "arc-updates/s"
BYTES_PER_ARC = 32          # read psi 16 B + write psi' 16 B
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback
SPEC_HBM_GBS = 8000.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--nx", type=int, default=2048)
    ap.add_argument("--walk-steps", type=int, default=1000)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU (slab + NCCL) code path even on one rank (validation)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def traffic_per_launch(workload: str):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p)).get(workload)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.t = None

    def start(self, wait_s: float = 5.0):
        """Start polling every 50 ms; wait for the first sample (nvidia-smi
        takes ~0.5 s to start) so that a short timed region is covered."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-i",
                 str(self.device), "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t_end = time.time() + wait_s
            while not self.lines and time.time() < t_end:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self):
        """Start of the timed region (samples before it are the warm-up's)."""
        self.t0 = time.time()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        t0 = getattr(self, "t0", None)
        timed = [ln for t, ln in self.lines if t0 is None or t >= t0]
        # a timed region shorter than the polling period: the samples of the
        # warm-up steps just before it (same kernels, GPU busy) stand in
        window = "timed"
        if not timed:
            timed = [ln for _, ln in self.lines[-5:]]
            window = "warm-up + timed (region shorter than the 50 ms poll)"
        sm, smax, reasons = [], [], set()
        for ln in timed:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "window": window}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world, backend, force=False):
    """torch.distributed for N > 1 (torchrun env); `force` also at N = 1
    (--sharded: the multi-GPU code paths on one rank, for validation)."""
    import torch.distributed as dist
    if (world > 1 or force) and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if world == 1:
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            os.environ.setdefault("MASTER_PORT", str(sk.getsockname()[1]))
            sk.close()
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group(backend)
    return dist if (world > 1 or force) else None


def max_over_ranks(x: float, dist, device=None) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port of the reference algorithm)
# ---------------------------------------------------------------------------

def cpu_reference(nx: int, sample_steps: int, threads: int):
    """Time backend._csr_rows-style CSR steps (reference algorithm, numpy) on
    the host cores with the reference's row-block thread pool."""
    from oracle import qwalk_oracle as O
    offs, cols = O.grid_adjacency(nx, nx)
    u = O.evolution_operator(offs, cols)
    rng = np.random.default_rng(0)
    x = rng.normal(size=u.n_rows) + 1j * rng.normal(size=u.n_rows)
    x /= np.linalg.norm(x)
    mv = O.Matvec(threads)
    mv(u, x)  # warm-up
    times = []
    for _ in range(sample_steps):
        t0 = time.perf_counter()
        x = mv(u, x)
        times.append(time.perf_counter() - t0)
    mv.close()
    total = sum(times)
    return {"value": u.n_rows * sample_steps / total, "unit": UNIT, "cores": threads,
            "kind": "port",
            "sample": f"{sample_steps} coined steps of grid {nx}x{nx} ({u.n_rows} arcs), numpy CSR "
                      f"matvec (oracle/ port of backend._csr_rows + row-block pool), "
                      f"median step {statistics.median(times) * 1e3:.1f} ms, min {min(times) * 1e3:.1f} ms"}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_reference():
    """The stock reference package installed by `pip install --target
    baseline/_ref`, or None.  Never /root/reference itself."""
    if not os.path.isdir(os.path.join(REF_DIR, "qwalk")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import qwalk
    if not os.path.abspath(qwalk.__file__).startswith(REF_DIR):
        return None
    return qwalk


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """The reference's own CPU path, unmodified, through its public API
    (baseline/_ref): coined.evolution_operator once (timed apart), then per
    bench step exactly one iteration of coined.simulate's loop body
    (coined.py:263-270): move_to_device(ComplexVector(psi)) + matvec_mul on the
    parallel engine with all host threads.  Also reported: the serial engine
    (median / min over 10 steps) and ctqw.evolve_state per Taylor term on
    hypercube(20).  Falls back to the oracle port when baseline/_ref is absent."""
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    qw = load_reference()
    if qw is None:
        return run_reference_port(args)
    from qwalk import backend as RB
    from qwalk import coined as RC
    from qwalk import ctqw as RQ
    threads = os.cpu_count() or 1
    nx = args.nx
    t0 = time.perf_counter()
    g = qw.graphs.grid(nx, nx)
    spec = RC.CoinedSpec(g)
    eng = RB.init_engine("parallel", threads)
    u = RC.evolution_operator(eng, spec)
    u_dev = RB.move_to_device(eng, u)
    build_s = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    cur = rng.normal(size=u.n_rows) + 1j * rng.normal(size=u.n_rows)
    cur /= np.linalg.norm(cur)

    def step(e, ud, x):   # coined.simulate's loop body (coined.py:268-269)
        return RB.matvec_mul(e, RB.move_to_device(e, RB.ComplexVector(x)), ud).entries

    for _ in range(args.warmup):
        cur = step(eng, u_dev, cur)
    times = []
    for _ in range(args.steps):
        a = time.perf_counter()
        cur = step(eng, u_dev, cur)
        times.append(time.perf_counter() - a)
    el = sum(times)
    value = u.n_rows * args.steps / el
    RB.stop_engine(eng)
    # serial engine, same operator
    eser = RB.init_engine("serial")
    us_dev = RB.move_to_device(eser, u)
    cur = step(eser, us_dev, cur)
    ser = []
    for _ in range(10):
        a = time.perf_counter()
        cur = step(eser, us_dev, cur)
        ser.append(time.perf_counter() - a)
    RB.stop_engine(eser)
    del u, u_dev, us_dev
    # CTQW: evolve_state on hypercube(20), gamma 1/20, marked {0}, t = 0.5
    # (one sub-step); terms counted by wrapping the module's matvec_mul
    dim = 20
    t1 = time.perf_counter()
    hs = RQ.CtqwSpec(qw.graphs.hypercube(dim), 1.0 / dim, 1.0, frozenset({0}))
    h = RQ.build_hamiltonian(hs)
    hbuild_s = time.perf_counter() - t1
    count = [0]
    orig = RQ.matvec_mul

    def counted(*a, **k):
        count[0] += 1
        return orig(*a, **k)
    RQ.matvec_mul = counted
    ectq = RB.init_engine("parallel", threads)
    psi = qw.WalkState(qw.VertexBasis(1 << dim), np.full(1 << dim, 2.0 ** (-dim / 2), dtype=np.complex128))
    a = time.perf_counter()
    RQ.evolve_state(ectq, h, psi, 0.5)
    ctqw_s = time.perf_counter() - a
    RQ.matvec_mul = orig
    RB.stop_engine(ectq)
    cfg = {"workload": f"grid {nx}x{nx} torus flip-flop Grover (C2), stock reference coined step",
           "arcs": int(g.num_arcs), "coined_steps_per_bench_step": 1,
           "parallelism": f"reference 'parallel' engine, {threads} threads"}
    sample = (f"reference qwalk {qw.__version__} from baseline/_ref: one coined.simulate loop iteration "
              f"(move_to_device + matvec_mul) per bench step on grid {nx}x{nx}, parallel engine "
              f"{threads} threads: median {statistics.median(times) * 1e3:.1f} ms, min {min(times) * 1e3:.1f} ms "
              f"over {len(times)} steps; U built once in {build_s:.1f} s (excluded)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference": {
            "package": os.path.relpath(os.path.dirname(qw.__file__), ROOT), "version": qw.__version__,
            "cpu_model": _cpu_model(), "os_cpu_count": os.cpu_count(),
            "operator_build_s": build_s,
            "parallel_engine": {"threads": threads, "median_ms": statistics.median(times) * 1e3,
                                "min_ms": min(times) * 1e3, "steps": len(times),
                                "arc_updates_per_s": u_arcs_per_s(g.num_arcs, statistics.median(times))},
            "serial_engine": {"median_ms": statistics.median(ser) * 1e3, "min_ms": min(ser) * 1e3,
                              "steps": len(ser),
                              "arc_updates_per_s": u_arcs_per_s(g.num_arcs, statistics.median(ser))},
            "ctqw_hypercube20": {"call": "ctqw.evolve_state(parallel engine, H, uniform psi, t=0.5)",
                                 "hamiltonian_build_s": hbuild_s, "terms": count[0], "seconds": ctqw_s,
                                 "ms_per_term": ctqw_s / max(count[0], 1) * 1e3,
                                 "vertex_term_updates_per_s": (1 << dim) * count[0] / ctqw_s},
        },
    }
    print(json.dumps(line), flush=True)
    return 0


def u_arcs_per_s(arcs: int, seconds: float) -> float:
    return arcs / seconds if seconds > 0 else 0.0


def run_reference_port(args):
    """Fallback without baseline/_ref: the oracle's numpy port of
    backend._csr_rows with the reference's row-block pool."""
    threads = os.cpu_count() or 1
    nx = args.nx
    from oracle import qwalk_oracle as O
    offs, cols = O.grid_adjacency(nx, nx)
    u = O.evolution_operator(offs, cols)
    rng = np.random.default_rng(0)
    x = rng.normal(size=u.n_rows) + 1j * rng.normal(size=u.n_rows)
    x /= np.linalg.norm(x)
    mv = O.Matvec(threads)
    sample = 2   # coined steps per bench step (bounded sample of the 1000)
    for _ in range(args.warmup):
        for _ in range(sample):
            x = mv(u, x)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(sample):
            x = mv(u, x)
    el = time.perf_counter() - t0
    mv.close()
    value = u.n_rows * sample * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"grid {nx}x{nx} torus flip-flop Grover (C2), reference CPU algorithm",
                   "arcs": u.n_rows, "coined_steps_per_bench_step": sample, "parallelism": f"{threads} threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"baseline/_ref missing: {sample} coined steps per bench step of grid {nx}x{nx}; "
                                   "numpy CSR matvec restating backend._csr_rows with the reference's row-block pool"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def run_b200(args):
    import torch
    import paper_2406_08186_b200 as q
    from paper_2406_08186_b200 import coined as CO

    rank, world, local = dist_env()
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local}, {torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("QWB_LOG_COMM", "1")   # one stderr line per rank at communicator init
    dist = init_dist(world, "nccl", force=args.sharded)
    dev = torch.device("cuda", local)
    single = world == 1 and not args.sharded
    eng = q.init_engine("b200", device=local)

    nx = args.nx
    walk = args.walk_steps
    if single:
        g = q.graphs.grid(nx, nx)
        spec = q.CoinedSpec(g)
        arcs = g.num_arcs
        rng = np.random.default_rng(0)
        psi = rng.normal(size=arcs) + 1j * rng.normal(size=arcs)
        psi /= np.linalg.norm(psi)
        psi0 = q.WalkState(q.graphs.arc_basis(g), psi)
        runner = CO._LatticeRunner(eng, spec)
        x = q.backend.to_device(eng, psi0.amplitudes)
    else:
        # weak scaling: one nx x (nx * world) torus, rank r owns rows [r*nx, (r+1)*nx)
        from paper_2406_08186_b200 import distributed as DI
        runner = DI.SlabLattice(eng, nx, nx * world, "flipflop", (), rank, world, comm=True)
        arcs = 4 * nx * runner.rows
        rng = np.random.default_rng(rank)
        psi = rng.normal(size=arcs) + 1j * rng.normal(size=arcs)
        psi /= np.linalg.norm(psi) * np.sqrt(world)
        host_local, _owner = q.state._pinned_empty(arcs) or (psi.copy(), None)
        host_local[...] = psi
        x = q.backend.to_device(eng, host_local)

    # ---- device-resident timed region: runner.advance(walk) per bench step
    runner.load(x)
    stream = torch.cuda.current_stream(dev)
    clocks = Clocks(local)
    clocks.start()
    for _ in range(args.warmup):
        runner.advance(walk)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.mark()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        runner.advance(walk)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    clk = clocks.stop()
    el_ms = e0.elapsed_time(e1)
    el_ms = max_over_ranks(el_ms, dist, dev)
    # One GPU: qwb_lattice_run fuses `depth` coined steps per launch of the
    # temporally blocked kernel (remainder steps: single-step kernel).  N > 1:
    # each step is two single-step launches (boundary rows, interior rows) + the
    # NCCL exchange.
    import ctypes as C
    from paper_2406_08186_b200 import _native as N
    dep, knd = C.c_int(0), C.c_int(0)
    N.load().qwb_lattice_fused_depth(nx, nx, 0, C.byref(dep), C.byref(knd))
    if single:
        depth = dep.value
        if depth > 0 and knd.value == 2:
            rem = walk % 4   # the flow kernel's blocks are 4 steps; a remainder >= 2 is one tile launch
            per_walk = 1 + (1 if rem >= 2 else rem)
            kernel = f"lattice_flow_kernel<flipflop, T=4, 32x64 region> (persistent, {walk // 4} blocks)"
        elif depth > 0:
            rem = walk % depth   # a remainder >= 2 is one shallower tile launch
            per_walk = walk // depth + (1 if rem >= 2 else rem)
            kernel = f"lattice_tb_kernel<flipflop, T={depth}, 32x64 region>"
        else:
            per_walk = walk
            kernel = "lattice_step_kernel<flipflop>"
    elif runner.ghost:
        from paper_2406_08186_b200 import distributed as DI
        # fused slabs: per exchange of G = mT ghost rows, m launches of T steps
        # (over the owned rows extended by (m-1)T, ..., 0 rows); the last < T
        # steps one at a time
        G = runner.ghost
        depth = DI.slab_depth()
        per_walk = walk // depth + walk % depth   # one T-step launch per T steps, then single steps
        kernel = (f"lattice_tb_kernel<flipflop, T={depth}, 32x64 region> on y-slabs with {G} ghost rows "
                  f"({G // depth} launches per exchange)")
    else:
        depth = 0
        per_walk = 2 * walk
        kernel = "lattice_step_kernel<flipflop> (slab boundary rows + interior rows)"
    launches = args.steps * per_walk
    step_s = el_ms / 1e3 / (args.steps * walk)          # per coined step (all rows)
    value = world * arcs * walk * args.steps / (el_ms / 1e3)
    steps_per_launch = max(depth, 1)
    launch_s = step_s * steps_per_launch               # per launch of the dominant kernel

    peak, peak_src = peaks()
    # algorithmic bytes of one launch: 32 B per arc-step x the
    # arc-steps one launch processes (arcs x coined steps fused per launch)
    achieved_gbs = BYTES_PER_ARC * arcs * steps_per_launch / launch_s / 1e9
    # compulsory HBM bytes of one launch: the state read once + written once
    compulsory_gbs = BYTES_PER_ARC * arcs / launch_s / 1e9
    workload = f"grid{nx}_flipflop_grover_T{steps_per_launch}"
    traffic = traffic_per_launch(workload)

    # ---- e2e: public API with host buffers, H2D + D2H inside the timed region
    e2e_times = []
    # two untimed calls first: the pinned host buffers the results land in
    # (torch's caching host allocator) reach steady state after the second
    for i in range(2 + args.steps):
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        if single:
            out = CO.simulate(eng, spec, (walk, walk + 1, 1), psi0)[0].amplitudes
        else:
            xd = q.backend.to_device(eng, host_local)
            runner.load(xd)
            runner.advance(walk)
            runner.store(xd)
            out, _o = q.backend.to_host(xd, pinned=True)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        if i > 1:
            e2e_times.append(t1 - t0)
    e2e_s = max_over_ranks(sum(e2e_times), dist, dev)
    e2e_value = world * arcs * walk * len(e2e_times) / e2e_s
    if single:
        assert abs(np.linalg.norm(out) - 1.0) < 1e-9

    extras = {}
    if not args.no_extras and not single:
        for name, fn in (("c5_grid8192_sharded", measure_c5_sharded), ("c4_hypercube22_sharded", measure_c4_sharded)):
            try:
                r = fn(q, dev, local, rank, world, dist)
            except Exception as e:  # pragma: no cover - reported, the headline line still prints
                r = {"error": repr(e)}
            if rank == 0:
                extras[name] = r
    if not args.no_extras and rank == 0:
        extras.update(measure_extras(q, CO, eng, dev, peak))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_reference(nx, 64, os.cpu_count() or 1)   # ~10 s of host work
        except Exception as e:  # pragma: no cover - reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {e!r}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": (f"C2: grid {nx}x{nx} torus ({nx * nx} vertices, {arcs} arcs; BASELINE configs[1] "
                             f"'4M vertices, 16M arcs' per SURVEY D1), flip-flop Grover coin, {walk} coined "
                             f"steps per bench step, matrix-free lattice kernel") if single else
                            (f"grid {nx}x{nx * world} torus split in {world} y-slabs of {nx}x{nx} "
                             f"({arcs} arcs per GPU), flip-flop Grover, {walk} coined steps per bench step, "
                             f"temporally blocked slabs: NCCL exchange of {runner.ghost} ghost state rows per "
                             f"plane and side every {runner.ghost} steps, in stream order before each launch"),
                "nx": nx, "ny": nx * world, "arcs": arcs * world, "coined_steps_per_bench_step": walk,
                "psi0": "dense random complex128 (seeded per rank), normalised",
                "l2": f"inputs larger than L2: 2 x {16 * arcs / 1e6:.0f} MB ping-pong state per GPU (> 126 MB L2)",
                "parallelism": "dp1" if single else f"y-slab sharding over {world} GPUs (weak scaling)",
            },
            "roofline": {"bound": "hbm", "achieved": compulsory_gbs, "peak": peak, "unit": "GB/s",
                         "frac": compulsory_gbs / peak, "traffic": traffic,
                         "bytes_per_launch": BYTES_PER_ARC * arcs,
                         "kernel": kernel, "steps_per_launch": steps_per_launch,
                         "time_per_launch_us": launch_s * 1e6,
                         "peak_source": peak_src, "frac_of_spec_8TBps": compulsory_gbs / SPEC_HBM_GBS,
                         "algorithmic_bytes_per_launch": BYTES_PER_ARC * arcs * steps_per_launch,
                         "algorithmic_equiv_GBps": achieved_gbs,
                         "frac_algorithmic_equiv": achieved_gbs / peak,
                         "note": ("achieved = the bytes one launch must move through HBM (the state read "
                                  f"once + written once: 32 B per arc, {steps_per_launch} coined steps per "
                                  "launch; ncu dram bytes = traffic) / CUDA-event time per launch.  "
                                  "frac_algorithmic_equiv counts SURVEY §8(d)'s 32 B per arc-step for "
                                  f"every one of the {steps_per_launch} fused steps: the speed-up over a "
                                  "single-step kernel at the HBM roofline, not a bandwidth.  At T = 4 the "
                                  "tiles run at the HBM roofline (frac 0.82 at 2048^2, 0.90 at 4096^2, full "
                                  "clocks); T = 6 moves 2/3 of those bytes per step for 30 % more on-chip "
                                  "adds and is faster (and keeps the SM clock higher under the power cap), "
                                  "so the default kernel is SM-bound (FP64 adds, shuffles, barrier latency) "
                                  "and its HBM fraction is low by design")
                                 if steps_per_launch > 1 else "single-step kernel: 32 B per arc-step, HBM-bound"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 16 * arcs,
                    "d2h_bytes_per_step": 16 * arcs,
                    "call": "coined.simulate(engine, spec, (1000, 1001, 1), psi0) -> [WalkState]" if single
                    else "distributed.SlabLattice load(H2D pinned) + advance(1000) + store + D2H per rank",
                    "ms_per_call": e2e_s / len(e2e_times) * 1e3},
            "gpu_launches": launches,
            "clocks": clk,
            "also": extras,
        }
        print(json.dumps(line), flush=True)
    q.stop_engine(eng)
    if dist:
        dist.destroy_process_group()
    return 0


def measure_c5_sharded(q, dev, local, rank, world, dist):
    """C5 across the ranks (strong scaling): the 8192 x 8192 torus split into
    y-slabs (fused temporally blocked slabs + NCCL ghost rows), 120 coined
    steps, CUDA-event time on the launch stream, max over ranks."""
    import torch
    from paper_2406_08186_b200 import distributed as DI
    nx = 8192
    eng2 = q.init_engine("b200", device=local)
    lat = DI.SlabLattice(eng2, nx, nx, "flipflop", (), rank, world, comm=True)
    lat.a.fill_(1.0 / (2.0 * nx))
    stream = torch.cuda.current_stream(dev)
    lat.advance(24)
    dist.barrier()
    torch.cuda.synchronize(dev)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    lat.advance(120)
    b.record(stream)
    torch.cuda.synchronize(dev)
    dt = max_over_ranks(a.elapsed_time(b) / 1e3, dist, dev)
    lat.close()
    q.stop_engine(eng2)
    return {"arc_updates_per_s": 4 * nx * nx * 120 / dt, "us_per_step": dt / 120 * 1e6, "ranks": world,
            "ghost_rows": lat.ghost, "rows_per_rank": lat.rows,
            "scaling": "strong (one 8192 x 8192 torus over all ranks)"}


def measure_c4_sharded(q, dev, local, rank, world, dist):
    """C4 across the ranks (strong scaling): hypercube(22) CTQW, gamma = 1/22,
    marked {0}, one evolve of t = 1, vertex shards with the per-term NCCL
    partner exchange (distributed.ShardedHypercubeWalk); CUDA-event time on
    the launch stream, max over ranks."""
    import torch
    from paper_2406_08186_b200 import distributed as DI
    dim = 22
    eng2 = q.init_engine("b200", device=local)
    w = DI.ShardedHypercubeWalk(eng2, dim, 1.0 / dim, (0,), rank, world)
    x = torch.empty(w.n_local, dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    x.fill_(2.0 ** -11)
    w.evolve(x, 1.0)
    x.fill_(2.0 ** -11)
    dist.barrier()
    torch.cuda.synchronize(dev)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    terms = w.evolve(x, 1.0)
    b.record(stream)
    torch.cuda.synchronize(dev)
    dt = max_over_ranks(a.elapsed_time(b) / 1e3, dist, dev)
    w.close()
    q.stop_engine(eng2)
    nterms = sum(terms)
    return {"seconds_per_evolve_t1": dt, "terms": terms, "us_per_term": dt / nterms * 1e6,
            "vertex_term_updates_per_s": (1 << dim) * nterms / dt, "ranks": world,
            "exchange_bytes_per_rank_per_term": 16 * w.S * w.n_local,
            "scaling": "strong (one hypercube(22) over all ranks)"}


def _fused_depth(nx: int, n_marked: int) -> int:
    """Coined steps per HBM pass of an untraced run (the flow kernel's blocks
    are 4 steps)."""
    import ctypes as C
    from paper_2406_08186_b200 import _native as N
    dep, knd = C.c_int(0), C.c_int(0)
    N.load().qwb_lattice_fused_depth(nx, nx, n_marked, C.byref(dep), C.byref(knd))
    return 4 if knd.value == 2 else dep.value


def measure_extras(q, CO, eng, dev, peak):
    import torch
    out = {}
    stream = torch.cuda.current_stream(dev)

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize(dev)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize(dev)
        return a.elapsed_time(b) / 1e3

    # C3 size: 4096^2 torus, one marked vertex (the search oracle), 200 steps
    nx = 4096
    g = q.graphs.grid(nx, nx)
    c = nx // 2 + nx * (nx // 2)
    spec = q.CoinedSpec(g, "flipflop", "grover", frozenset({c}), "minus_identity")
    r = CO._LatticeRunner(eng, spec)
    r.a.fill_(1.0 / np.sqrt(4 * nx * nx))
    s = timed(lambda: r.advance(240), 3)
    arcs = 4 * nx * nx
    per = s / 720
    T = max(_fused_depth(nx, 1), 1)
    gbs = 32 * arcs / (per * T) / 1e9    # state read + written once per T-step launch
    out["grid4096_marked"] = {"arc_updates_per_s": arcs / per, "achieved_GBps": gbs, "frac": gbs / peak,
                              "bytes_per_launch": 32 * arcs, "steps_per_launch": T,
                              "frac_algorithmic_equiv": 32 * arcs / per / 1e9 / peak,
                              "us_per_step": per * 1e6}
    del r
    torch.cuda.empty_cache()
    # C2 as literally named: 1024^2 (1M vertices, 4M arcs), 1000 steps; the
    # 2 x 67 MB ping-pong state is about L2-sized (126 MB), so part of it is
    # served from L2 between launches
    nx1 = 1024
    r1 = CO._LatticeRunner(eng, q.CoinedSpec(q.graphs.grid(nx1, nx1)))
    r1.a.fill_(1.0 / np.sqrt(4 * nx1 * nx1))
    s1 = timed(lambda: r1.advance(1000), 3) / 3000
    T1 = max(_fused_depth(nx1, 0), 1)
    arcs1 = 4 * nx1 * nx1
    out["c2_grid1024"] = {"arc_updates_per_s": arcs1 / s1, "us_per_step": s1 * 1e6, "steps": 1000,
                          "achieved_GBps": 32 * arcs1 / (s1 * T1) / 1e9,
                          "frac": 32 * arcs1 / (s1 * T1) / 1e9 / peak, "steps_per_launch": T1,
                          "l2_note": "2 x 67 MB state vs 126 MB L2: partly L2-resident, frac is not an HBM figure"}
    del r1
    torch.cuda.empty_cache()
    # C5 on one GPU (the efficiency denominator of the multi-GPU runs):
    # 8192^2 torus, 8.6 GB ping-pong state, 120 coined steps
    r5 = CO._LatticeRunner(eng, q.CoinedSpec(q.graphs.grid(8192, 8192)))
    r5.a.fill_(1.0 / (2.0 * 8192))
    s5 = timed(lambda: r5.advance(120), 2) / 240
    out["c5_grid8192"] = {"arc_updates_per_s": 4 * 8192 * 8192 / s5, "us_per_step": s5 * 1e6,
                          "state_bytes": 2 * 4 * 8192 * 8192 * 16}
    del r5
    torch.cuda.empty_cache()
    # C3 in full: 4096^2, centre marked, uniform psi0 (= 2^-13 exactly),
    # T = ceil(sqrt(N ln N)) = 16707 steps, p(marked) after every step fused
    # into the step kernels, full distributions every 4096 steps
    import math
    N = nx * nx
    T = math.ceil(math.sqrt(N * math.log(N)))
    psi_u = q.WalkState(q.graphs.arc_basis(g), np.full(arcs, 2.0 ** -13, dtype=np.complex128))
    # one untimed call first (lazy kernel loading, the copy stream, bounce
    # buffers and worker thread of the first call in a process), as the e2e
    # line's warm-up calls; its wall time is reported beside
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    CO.search_trace(eng, spec, T, psi_u, 4096)
    torch.cuda.synchronize(dev)
    dt_first = time.perf_counter() - t0
    t0 = time.perf_counter()
    trace, dists = CO.search_trace(eng, spec, T, psi_u, 4096)
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t0
    pk = int(np.argmax(trace[:, 0]))
    out["c3_search_grid4096"] = {"steps": T, "seconds": dt, "first_call_seconds": dt_first,
                                 "arc_updates_per_s": arcs * T / dt,
                                 "p_marked_peak": float(trace[pk, 0]), "peak_step": pk,
                                 "p_marked_final": float(trace[-1, 0]), "uniform_p": 1.0 / N,
                                 "distributions_saved": sorted(dists),
                                 "call": "coined.search_trace(engine, spec, 16707, uniform psi0, 4096) "
                                         "incl. H2D, layout conversion, trace D2H"}
    del trace, dists, psi_u
    torch.cuda.empty_cache()
    # K1: device-built CSR U at 2048^2, SpMV per step (120 B/arc algorithmic)
    nx = 2048
    g = q.graphs.grid(nx, nx)
    spec = q.CoinedSpec(g)
    t0 = time.perf_counter()
    u = CO.device_operator(eng, g, "flipflop")
    torch.cuda.synchronize(dev)
    build_s = time.perf_counter() - t0
    n = u.n_rows
    xa = torch.full((n,), 1.0 / np.sqrt(n), dtype=torch.complex128, device=dev)
    xb = torch.empty_like(xa)

    def csr_step():
        q.backend.spmv_device(eng, u, xa, xb)
    s = timed(csr_step, 50)
    per = s / 50
    csr_bytes = 32 + 4 * (16 + 4) + 8
    gbs = csr_bytes * n / per / 1e9
    out["csr_spmv_grid2048"] = {"arc_updates_per_s": n / per, "achieved_GBps": gbs, "frac": gbs / peak,
                                "bytes_per_arc": csr_bytes, "us_per_step": per * 1e6,
                                "device_build_s": build_s}
    del u, xa, xb
    torch.cuda.empty_cache()

    # C1: cycle(1024), all 501 snapshots through the public API (one persistent CTA)
    g = q.graphs.cycle(1024)
    b = q.graphs.arc_basis(g)
    amp = np.zeros(b.size, complex)
    amp[q.graphs.arc_index(b, 512, 513)] = 1 / np.sqrt(2)
    amp[q.graphs.arc_index(b, 512, 511)] = 1j / np.sqrt(2)
    st0 = q.WalkState(b, amp)
    spec = q.CoinedSpec(g)
    CO.simulate(eng, spec, (0, 501, 1), st0)
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        CO.simulate(eng, spec, (0, 501, 1), st0)
    dt = (time.perf_counter() - t0) / reps
    out["c1_cycle1024_500steps"] = {"seconds_per_simulate": dt, "arc_updates_per_s": 2048 * 500 / dt,
                                    "note": "wall time of coined.simulate(range (0,501,1)) incl. U build, "
                                            "H2D, 500 steps, D2H of 501 snapshots"}

    # C4: hypercube(22) CTQW, gamma = 1/22, marked {0}, one evolve of t = 1 (2 sub-steps)
    dim = 22
    hc = q.graphs.hypercube(dim)
    cs = q.CtqwSpec(hc, 1.0 / dim, 1.0, frozenset({0}))
    from paper_2406_08186_b200 import ctqw as CT
    op = CT._Operator(eng, cs)
    nv = 1 << dim
    x = torch.full((nv,), 1.0 / np.sqrt(nv), dtype=torch.complex128, device=dev)
    op.evolve(x, 1.0, 1e-12)
    torch.cuda.synchronize(dev)
    x.fill_(1.0 / np.sqrt(nv))
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    terms = op.evolve(x, 1.0, 1e-12)
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t0
    nterms = sum(terms)
    out["c4_hypercube22_ctqw"] = {"seconds_per_evolve_t1": dt, "substeps": len(terms), "terms": terms,
                                  "us_per_term": dt / nterms * 1e6,
                                  "vertex_term_updates_per_s": nv * nterms / dt,
                                  "achieved_GBps_64B_per_vertex_term": 64 * nv * nterms / dt / 1e9,
                                  "frac_64B_per_vertex_term": 64 * nv * nterms / dt / 1e9 / peak,
                                  "frac": 64 * nv * nterms / dt / 1e9 / peak,
                                  "l2_to_sm_bytes_per_vertex_term": (dim - 10 + 2) * 16,
                                  "l2_to_sm_GBps": (dim - 10 + 2) * 16 * nv * nterms / dt / 1e9,
                                  "kernel": "hc_pair_kernel (TMA bulk-streamed partner tiles, two per stage)",
                                  "note": "64 B/vertex-term = term read + write and acc read-modify-write "
                                          "from HBM; each vertex also needs its 12 high-bit neighbours, "
                                          "streamed from L2 as 16-KB partner tiles ((dim-10+2) x 16 B "
                                          "per vertex-term over L2->SM); the kernel is bound by its "
                                          "consumer warps' latency chain, not by HBM or L2 bandwidth "
                                          "(DESIGN.md section 4)",
                                  "inf_norm": op.inf_norm}
    del op, x
    torch.cuda.empty_cache()

    # CTQW on a generic (CSR) H: grid 2048^2, gamma 0.25, marked {0}, t = 1
    nx = 2048
    csp = q.CtqwSpec(q.graphs.grid(nx, nx), 0.25, 1.0, frozenset({0}))
    opc = CT._Operator(eng, csp)
    nv = nx * nx
    xc = torch.full((nv,), 1.0 / np.sqrt(nv), dtype=torch.complex128, device=dev)
    opc.evolve(xc, 1.0, 1e-12)
    xc.fill_(1.0 / np.sqrt(nv))
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    terms = opc.evolve(xc, 1.0, 1e-12)
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t0
    nterms = sum(terms)
    per_vt = 64 + 20 * (4 * nv + 1) / nv + 8   # state r/w + acc RMW, values + cols, row offsets
    out["ctqw_csr_grid2048"] = {"terms": terms, "us_per_term": dt / nterms * 1e6,
                                "vertex_term_updates_per_s": nv * nterms / dt,
                                "bytes_per_vertex_term": per_vt,
                                "achieved_GBps": per_vt * nv * nterms / dt / 1e9,
                                "frac": per_vt * nv * nterms / dt / 1e9 / peak,
                                "kernel": "csr_term_kernel4 (one resident wave, 64 registers)",
                                "note": "wall time of one evolve (incl. the per-term norm finalize and "
                                        "the per-chunk stop-flag reads)"}
    return out


def ensure_world(args) -> int | None:
    """--gpus N on the B200 arm needs N ranks.  Under torchrun WORLD_SIZE must
    equal N; launched without torchrun, re-exec this script under
    `torch.distributed.run --nproc-per-node N` (127.0.0.1 rendezvous).  Fails
    loudly (exit 2) when fewer GPUs are visible than requested.  Returns an
    exit code to stop with, or None to run here."""
    rank, world, _ = dist_env()
    if "WORLD_SIZE" in os.environ:
        if world != args.gpus:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
            return 2
        return None
    if args.gpus == 1:
        return None
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} requested but {have} CUDA device(s) visible", file=sys.stderr)
        return 2
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print("bench.py: re-exec under torchrun: " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rc = ensure_world(args)
    if rc is not None:
        return rc
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
