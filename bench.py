#!/usr/bin/env python
"""Benchmark of the B200 state-vector core (BASELINE.json metric).

Workload ("sweep", the default): BASELINE config 2 -- a Haar-random 2x2
unitary applied to every qubit in turn of a normalised Gaussian complex128
state with 2^m amplitudes per GPU (m = 30: 16 GiB), fresh unitaries each
step.  On N GPUs the state has n = m + log2(N) qubits (weak scaling, the
top log2(N) qubits global, as in config 4), so each step also runs log2(N)
global-qubit gates through the exchange path.

Unit: one gate applied to 2^30 amplitudes (an n=30 gate-update).  `value`
is whole-job gate-updates/s in that unit (at N=1 exactly config 2's
gate-updates/s); hbm_gbs is the algorithmic traffic (32 B per amplitude per
gate, read + write) over the device time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--local-qubits M] [--no-fuse] [--workload sweep|qaoa]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gate-updates/s and achieved HBM GB/s (n=30 c128); weak-scaled n=33-36 on 1-8 GPUs"
UNIT = "gate-updates/s (n=30-equivalent: 1 unit = one 2x2 gate on 2^30 c128 amplitudes)"
FP64_PEAK_TOPS = 62 * 148 * 1.965e9 / 1e12  # measured on B200 (tools/exp/fp64.cu)
LAUNCH_KINDS = {1: "k_gate1q", 2: "k_controlled", 3: "k_cut_phase", 4: "k_tile",
                5: "k_exchange_peer", 6: "k_tree", 7: "k_fact", 8: "k_fact_gen", 9: "k_perm"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 10; the QAOA swarm: 50, BASELINE config 5)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--local-qubits", type=int, default=None,
                    help="amplitudes per GPU = 2^M (default: 30 for the config-2 sweep at "
                         "N=1, 33 for the weak-scaled config-4 layer at N>1)")
    ap.add_argument("--no-fuse", action="store_true")
    ap.add_argument("--numerics", default="factored", choices=["factored", "exact"],
                    help="factored: QS_FUSE_FACTORED (Euler-factored 1q gates, within 1e-12 "
                         "of the reference); exact: QS_FUSE_EXACT (bit-identical)")
    ap.add_argument("--workload", default=None,
                    choices=["sweep", "qaoa", "cfg1", "cfg3", "cfg4", "noise"],
                    help="default: sweep (config 2) at N=1, cfg4 (config 4, weak-scaled) at N>1")
    ap.add_argument("--ref-local-qubits", type=int, default=23,
                    help="reference arm at N>1: amplitudes per thread-rank (host RAM bound)")
    ap.add_argument("--no-config4-point", action="store_true",
                    help="N=1 sweep: skip the config-4 n=33 point of the weak-scaling curve")
    ap.add_argument("--seed", type=int, default=20260809)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--pool-chunks", type=int, default=1,
                    help="qaoa: the GPU's share of the pool as this many batched sub-pools, so "
                         "the host builds chunk k+1's program while chunk k runs (each chunk "
                         "has its own stream: per-launch times overlap, so the pass roofline "
                         "is only meaningful with 1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"])
    ap.add_argument("--no-per-target", action="store_true")
    ap.add_argument("--no-exact-compare", action="store_true")
    ap.add_argument("--remap", action="store_true",
                    help="gates on global qubits swap the qubit into a local position "
                         "(half the NVLink traffic) instead of the pair exchange")
    args = ap.parse_args()
    if args.workload is None:
        args.workload = "sweep" if args.gpus == 1 else "cfg4"
    if args.steps is None:
        args.steps = 50 if args.workload == "qaoa" else 10
    if args.local_qubits is None:
        args.local_qubits = 33 if (args.gpus > 1 and args.workload == "cfg4") else 30
    return args


def fuse_mode(args):
    if args.no_fuse:
        return False
    return "factored" if args.numerics == "factored" else True


# ---- clocks -------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh).get(kernel)
    except (OSError, ValueError):
        return None


# ---- distributed plumbing -------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world):
    if world == 1:
        return None
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group(backend="gloo")
    return dist


def max_over_ranks(dist, x: float) -> float:
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ---- CPU baseline (oracle port, host threads) ----------------------------------------
def cpu_sweep_sample(m: int, gates: int, seed: int) -> dict:
    """Time the reference algorithm (oracle restatement, all host threads) on
    a bounded sample: `gates` single-gate applications on a 2^m state."""
    from oracle import cpu_baseline as cb

    rng = np.random.default_rng(seed)
    psi = np.full(1 << m, 2.0 ** (-m / 2.0), dtype=np.complex128)
    targets = [int(x) for x in np.linspace(0, m - 1, gates).round()]
    us = [haar(rng) for _ in targets]
    cb.apply_1q_threaded(psi, 0, np.eye(2, dtype=np.complex128))  # warm (page faults)
    t0 = time.perf_counter()
    for q, u in zip(targets, us):
        cb.apply_1q_threaded(psi, q, u)
    dt = time.perf_counter() - t0
    units = len(targets) * (2.0 ** m) / 2.0 ** 30
    return {"value": units / dt, "unit": UNIT, "cores": cb.threads(), "kind": "port",
            "sample": f"{len(targets)} single-gate applications (targets {targets}) on a "
                      f"2^{m} complex128 state, oracle/cpu_baseline.py (numpy, "
                      f"{cb.threads()} threads), {dt:.2f} s"}


def cpu_controlled_sample(m: int, pair, phi_u, seed: int) -> dict:
    """Config 3's CPU baseline: the reference's controlled-gate kernel
    (statevector.py:180-195, oracle/cpu_baseline.py threaded port) for the
    first seeded pair's CNOT, CPhase and controlled Haar on a 2^m state."""
    from oracle import cpu_baseline as cb

    c, t = pair
    phi, u = phi_u
    psi = np.full(1 << m, 2.0 ** (-m / 2.0), dtype=np.complex128)
    mats = [np.array([[0, 1], [1, 0]], dtype=np.complex128),
            np.diag([1.0, np.exp(1j * phi)]).astype(np.complex128), u]
    cb.apply_1q_threaded(psi, 0, np.eye(2, dtype=np.complex128))  # warm (page faults)
    t0 = time.perf_counter()
    for mat in mats:
        cb.apply_controlled_threaded(psi, c, t, mat)
    dt = time.perf_counter() - t0
    units = len(mats) * (2.0 ** m) / 2.0 ** 30
    return {"value": units / dt, "unit": UNIT, "cores": cb.threads(), "kind": "port",
            "sample": f"CNOT, CPhase and controlled Haar on pair (c={c}, t={t}) of a 2^{m} "
                      f"complex128 state, oracle/cpu_baseline.py (numpy, {cb.threads()} "
                      f"threads), {dt:.2f} s"}


def cpu_layer_sample(m: int, cx, seed: int) -> dict:
    """Config 4's CPU baseline at one GPU (every qubit local): two Haar gates
    of the layer and its first CX(q, n-1-q), reference kernels, threaded port."""
    from oracle import cpu_baseline as cb

    rng = np.random.default_rng(seed)
    psi = np.full(1 << m, 2.0 ** (-m / 2.0), dtype=np.complex128)
    X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
    cb.apply_1q_threaded(psi, 0, np.eye(2, dtype=np.complex128))  # warm (page faults)
    t0 = time.perf_counter()
    cb.apply_1q_threaded(psi, 0, haar(rng))
    cb.apply_1q_threaded(psi, m - 1, haar(rng))
    cb.apply_controlled_threaded(psi, cx[0], cx[1], X)
    dt = time.perf_counter() - t0
    units = 3 * (2.0 ** m) / 2.0 ** 30
    return {"value": units / dt, "unit": UNIT, "cores": cb.threads(), "kind": "port",
            "sample": f"Haar on qubits 0 and {m - 1} + CX{tuple(cx)} of a 2^{m} complex128 "
                      f"state, oracle/cpu_baseline.py (numpy, {cb.threads()} threads), {dt:.2f} s"}


def haar(rng):
    from paper_2001_10554_b200.workloads import haar_2x2

    return haar_2x2(rng)


def host_gaussian_state(m: int, seed: int) -> np.ndarray:
    """Normalised i.i.d. N(0,1) re/im state of 2^m amplitudes (the recipe of
    tests/oracles.py:99-101), filled in parallel chunks from spawned seeds."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import cpu_baseline as cb

    psi = np.empty(1 << m, dtype=np.complex128)
    view = psi.view(np.float64)
    chunk = 1 << 24
    seeds = np.random.SeedSequence(seed).spawn(max(1, view.size // chunk))

    def fill(k):
        g = np.random.default_rng(seeds[k])
        g.standard_normal(out=view[k * chunk:(k + 1) * chunk])

    with ThreadPoolExecutor(cb.threads()) as ex:
        list(ex.map(fill, range(len(seeds))))
    norm = 0.0
    for k in range(0, psi.size, chunk):
        a = psi[k:k + chunk]
        norm += float(np.vdot(a, a).real)
    psi *= 1.0 / np.sqrt(norm)
    return psi


def run_reference(args):
    """--impl reference: the reference's own CPU algorithm of the path (the
    oracle's numpy restatement, all host threads; the Python reference cannot
    travel to the GPU box) on OUR arm's workload, each step a bounded sample.
    N=1: the config-2 sweep on a normalised Gaussian 2^m state, 3 consecutive
    gates of the sweep per step (targets in sweep order, fresh Haar each).
    N>1 (torchrun): rank 0 alone runs the reference's distributed path --
    local gates plus the Fig. 3 pair exchange (oracle/distribution.py,
    restating distribution.py:121-230) -- on N thread-ranks at a reduced
    2^ref_local_qubits amplitudes per rank, one config-4 layer per step."""
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    from oracle import cpu_baseline as cb

    if world > 1:
        return run_reference_dist(args, world)
    m = args.local_qubits
    rng = np.random.default_rng(args.seed + 1)
    psi = host_gaussian_state(m, args.seed)
    per_step = 3
    q = 0

    def step():
        nonlocal q
        for _ in range(per_step):
            cb.apply_1q_threaded(psi, q, haar(rng))
            q = (q + 1) % m

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    units = args.steps * per_step * (2.0 ** m) / 2.0 ** 30
    value = units / dt
    sample = (f"{per_step} consecutive gates of the config-2 sweep per step (targets in sweep "
              f"order, fresh Haar 2x2 each) on a normalised Gaussian 2^{m} c128 state, "
              f"oracle/cpu_baseline.py (numpy, {cb.threads()} threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128 (f64 pairs)", "data": "synthetic",
        "config": {"workload": f"config 2 sweep: Haar 2x2 on each of the {m} qubits in turn, "
                               f"fresh unitaries per step, normalised Gaussian state, "
                               f"2^{m} c128 amplitudes per GPU (n={m}, 0 global qubits)",
                   "qubits": m, "local_qubits": m, "sample": sample, "same_workload": True,
                   "parallelism": f"{cb.threads()} host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cb.threads(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_reference_dist(args, world):
    """Rank 0 of a torchrun: the reference's distributed config-4 layer on
    `world` thread-ranks (oracle restatement), host RAM-bounded size."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import distribution as odist
    from oracle import statevector as osv

    m = args.ref_local_qubits
    p = world.bit_length() - 1
    n = m + p
    psi = host_gaussian_state(n, args.seed)
    parts = [psi[r << m:(r + 1) << m] for r in range(world)]
    rng = np.random.default_rng(args.seed + 1)
    pool = ThreadPoolExecutor(world)
    cx = [(q, n - 1 - q) for q in range(n // 2)]
    X = np.array([[0, 1], [1, 0]], dtype=np.complex128)

    def layer():
        for q in range(n):
            u = haar(rng)
            if q < m:  # every rank its local pairs, concurrently
                list(pool.map(lambda part: osv.apply_1q(part, q, u), parts))
            else:
                odist.apply_one_qubit_gate(parts, n, q, u)
        for c, t in cx:
            if c < m and t < m:
                list(pool.map(lambda part: osv.apply_controlled(part, c, t, X), parts))
            else:
                odist.apply_controlled_gate(parts, n, c, t, X)

    for _ in range(args.warmup):
        layer()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        layer()
    dt = time.perf_counter() - t0
    gates = n + len(cx)
    value = args.steps * gates * (2.0 ** n) / 2.0 ** 30 / dt
    sample = (f"config-4 layers at n={n} = {m} local + {p} global qubits on {world} thread-ranks "
              f"(2^{m} c128 per rank; the GPU arm holds 2^{args.local_qubits}), oracle "
              "restatement of the reference's local kernels and Fig. 3 pair exchange")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128 (f64 pairs)", "data": "synthetic",
        "config": {"workload": f"config 4 layer (weak-scaled): Haar 2x2 on all n qubits, then "
                               f"CX(q, n-1-q) for q < n/2; {world} ranks",
                   "qubits": n, "local_qubits": m, "sample": sample, "same_workload": False,
                   "parallelism": f"{world} thread-ranks"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": world, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---- our arm ----------------------------------------------------------------------------
def physical_devices(dist, local: int) -> int:
    """Distinct (host, device) pairs the ranks ran on (emulated ranks share one)."""
    if dist is None:
        return 1
    import socket

    mine = (socket.gethostname(), int(local))
    allv = [None] * dist.get_world_size()
    dist.all_gather_object(allv, mine)
    return len(set(allv))


def run_ours(args):
    world, rank, local = dist_env()
    emulated = bool(os.environ.get("QSB_ALL_RANKS_ON_DEVICE0"))
    if emulated and world > 1 and args.exchange == "nccl":
        raise SystemExit("bench.py: NCCL refuses two ranks on one GPU (ncclCommInitRank: invalid "
                         "usage); the emulated run uses --exchange peer")
    if emulated:
        local = 0  # functional multi-rank run on one GPU (exchange kernels never wait on each other)
    dist = init_dist(world)
    import paper_2001_10554_b200 as qs
    from paper_2001_10554_b200 import _native, runtime
    from paper_2001_10554_b200 import distribution as qdist
    from paper_2001_10554_b200 import transport as qtp
    from paper_2001_10554_b200.workloads import device_gaussian

    if qs.device_count() < 1:
        raise SystemExit("bench.py: no CUDA device -- the B200 core has no CPU fallback")
    if world & (world - 1):
        raise SystemExit("bench.py: --gpus must be a power of two")
    devices = physical_devices(dist, local)
    m = args.local_qubits
    p = world.bit_length() - 1
    n = m + p
    transport = qtp.TorchTransport(exchange_mode=args.exchange) if world > 1 else None
    if args.workload == "qaoa":
        return run_qaoa(args, dist, transport, world, rank, local)
    if args.workload == "cfg1":
        return run_cfg1(args, dist, world, rank, local)
    if args.workload == "noise":
        return run_noise(args, dist, transport, world, rank, local)
    ctx = runtime.make_context(transport, n, 1, device=local, fuse=fuse_mode(args),
                               remap=args.remap)
    ctx.norm_check_interval = 0
    st = ctx.state
    comm = ctx.comm
    group_norm = (lambda x: qdist.group_reduce_sum(x, ctx.topology, comm)) if world > 1 else None
    device_gaussian(st, args.seed, group_norm)
    rng = np.random.default_rng(args.seed + 1)
    total_steps = args.warmup + args.steps
    sweeps = [[haar(rng) for _ in range(n)] for _ in range(total_steps)]

    from paper_2001_10554_b200.circuit import GateSpec

    cx_pairs = [(q, n - 1 - q) for q in range(n // 2)] if args.workload == "cfg4" else []
    cfg3 = args.workload == "cfg3"
    if cfg3:
        # config 3: 64 seeded (control, target) pairs, control != target, each
        # getting CNOT, CPhase(phi ~ U[0,2pi)) and a controlled Haar 2x2
        prng = np.random.default_rng(args.seed + 3)
        pairs = []
        while len(pairs) < 64:
            c, t = (int(x) for x in prng.integers(0, n, size=2))
            if c != t:
                pairs.append((c, t))
        sweeps = [[(prng.uniform(0, 2 * np.pi), haar(prng)) for _ in pairs]
                  for _ in range(total_steps)]

    def step(us, c=None):
        c = ctx if c is None else c
        if cfg3:
            for (cq, tq), (phi, u) in zip(pairs, us):
                runtime.apply_gate(c, GateSpec("cx", (cq, tq)))
                runtime.apply_gate(c, GateSpec("cphase", (cq, tq), float(phi)))
                runtime.apply_gate(c, GateSpec("cu", (cq, tq), matrix=u))
            c.flush()
            return
        # config 2: Haar gate on every qubit; config 4 adds CX(q, n-1-q), q < n/2
        # (pairs cross the local/global boundary: routed like the reference)
        for k in range(n):
            runtime.apply_gate(c, GateSpec("custom", (k,), matrix=us[k]))
        for cq, tq in cx_pairs:
            runtime.apply_gate(c, GateSpec("cx", (cq, tq)))
        c.flush()

    for s in range(args.warmup):
        step(sweeps[s])
    st.synchronize()
    barrier(dist)
    clocks = ClockSampler(local)
    clocks.start()
    st.launch_log(True)
    st.event_record(0)
    t0 = time.perf_counter()
    for s in range(args.steps):
        step(sweeps[args.warmup + s])
    st.event_record(1)
    st.synchronize()
    wall = time.perf_counter() - t0
    ms_dev = st.event_elapsed_ms(0, 1)
    st.launch_log(False)
    launch_ms, launch_kind = st.read_launch_log()
    clock = clocks.stop()
    barrier(dist)
    ms_total = max_over_ranks(dist, ms_dev)
    gates_per_step = 3 * 64 if cfg3 else n + len(cx_pairs)
    units_per_step = gates_per_step * (2.0 ** n) / 2.0 ** 30
    value = units_per_step * args.steps / (ms_total / 1e3)
    # algorithmic: every 1q gate r+w of the slice, a CX the control=1 half,
    # a CPhase (diag(1,z)) the control=1, target=1 quarter
    if cfg3:
        bytes_per_step_per_gpu = (16.0 + 8.0 + 16.0) * (2 ** m) * 64
    else:
        bytes_per_step_per_gpu = 32.0 * (2 ** m) * n + 16.0 * (2 ** m) * len(cx_pairs)
    hbm_gbs = bytes_per_step_per_gpu * world * args.steps / (ms_total / 1e3) / 1e9

    # dominant kernel and its roofline
    peak, peak_src = measured_peak()
    kinds, share = {}, {}
    for k, t in zip(launch_kind, launch_ms):
        kinds.setdefault(int(k), []).append(float(t))
    dom = max(kinds, key=lambda k: sum(kinds[k])) if kinds else 4
    dom_ms = float(np.mean(kinds[dom])) if kinds else float("nan")
    for k, v in kinds.items():
        share[LAUNCH_KINDS.get(k, str(k))] = {"launches": len(v), "ms": float(np.sum(v)),
                                             "share": float(np.sum(v) / ms_dev)}
    # Roofline of the dominant kernel on its own algorithmic bytes: one fused
    # pass reads and writes each amplitude of the slice once, 32*2^m B, the
    # least any pass can move (SURVEY 8(d)'s per-gate figure is the same 32 B
    # per amplitude); frac = that / avg launch time / measured copy peak.
    # fusion_gain = gate-updates one launch applies (the unfused simulator
    # moves 32*2^m B per gate-update, so the algorithmic-per-gate rate is
    # fusion_gain x the pass rate).
    launches_per_step = len(kinds.get(dom, [])) / max(args.steps, 1)
    units_per_launch = gates_per_step / max(launches_per_step, 1e-9)
    pass_bytes = 32.0 * (2 ** m)
    physical = pass_bytes / (dom_ms / 1e3) / 1e9
    tr = ncu_traffic(LAUNCH_KINDS.get(dom, ""))
    traffic = None
    if tr and tr.get("bytes_per_amplitude"):
        traffic = tr["bytes_per_amplitude"] * (2 ** m)

    # global-qubit gates: NVLink bytes per exchange launch (per direction per
    # GPU: the partner's half read + our half written back by the partner =
    # 2^m * 16 B each way, the reference's Fig. 3 volume) over its time
    nvlink = None
    exch = kinds.get(5, [])
    if world > 1 and exch:
        per_dir = 16.0 * (2 ** m)
        ms_ex = float(np.mean(exch))
        gbs = per_dir / (ms_ex / 1e3) / 1e9
        nvlink = {"exchange_mode": ("remap (peer swap of half the slice)" if args.remap
                                    else args.exchange),
                  "launches_per_step": len(exch) / args.steps, "avg_launch_ms": ms_ex,
                  "bytes_per_direction_per_launch": per_dir if not args.remap else per_dir / 2,
                  "gbs_per_direction": gbs if not args.remap else gbs / 2,
                  "peak_nominal": 900.0, "peak_measured_peer_copy": 770.0,
                  "frac_of_nominal": (gbs if not args.remap else gbs / 2) / 900.0,
                  "emulated_on_one_gpu": emulated,
                  "note": ("ranks emulated on one GPU: the partner's slice is local HBM, not "
                           "NVLink" if emulated else
                           "CUDA events around each k_exchange_peer launch; "
                           "B200_PROFILING.md peer copy 770 GB/s per direction")}

    # e2e through the public API with host buffers (upload + sweep + download)
    e2e_resident = run_e2e_resident(args, ctx, st, sweeps, step, n, dist, gates_per_step)
    if m <= 31:
        e2e = run_e2e(args, ctx, st, sweeps, step, m, n, dist, gates_per_step)
    else:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
               "note": f"skipped: a 2^{m}-amplitude pinned host copy does not fit beside the "
                       "state on this host"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and m <= 30:
        if cfg3:
            cpu = cpu_controlled_sample(m, pairs[0], sweeps[0][0], args.seed)
        elif cx_pairs:
            cpu = cpu_layer_sample(m, cx_pairs[0], args.seed)
        else:
            cpu = cpu_sweep_sample(m, 3, args.seed)

    # config 2's per-target table: each target as a single unfused gate kernel
    per_target = (per_target_table(st, m, args.seed)
                  if not args.no_per_target and args.workload == "sweep" else None)
    passes_per_step = len(launch_ms) / max(args.steps, 1)
    actual_gbs = 32.0 * (2 ** m) * passes_per_step * args.steps / (ms_dev / 1e3) / 1e9
    # numpy-exact pair update: 20 FP64 ops per pair (a CX touches half the pairs);
    # factored: a 4-FMA shear per pair (2 per amplitude; lean passes pad every
    # register round to 4 shears) plus two product diagonals (~13 per amplitude)
    factored = fuse_mode(args) == "factored"
    if factored and cfg3:
        # the three controlled gates of a pair fuse into one controlled matrix
        fp64_per_amp = 5.0 * 64
        fp64_note = ("factored: CNOT, CPhase and controlled-Haar of a pair fused into one "
                     "controlled gate; 10 FP64 instructions per amplitude of the control=1 half")
    elif factored:
        # CNOT passes are permutations (k_perm): no arithmetic
        fp64_per_amp = (2.0 * 4 * sum(-(-r // 4) for r in (12, 9, 9)) if n == 30 else 2.0 * n) \
            + 26.0
        fp64_note = ("factored: 2 FP64 instructions per amplitude per shear (register rounds "
                     "padded to 4 shears), two product diagonals ~13 each; the pass is not "
                     "FP64-bound; CNOT passes are permutations")
    else:
        fp64_per_amp = (5.0 + 1.0 + 5.0) * 64 if cfg3 else 10.0 * (n + 0.5 * len(cx_pairs))
        fp64_note = ("10 FP64 instructions per amplitude per gate (numpy-exact complex "
                     "arithmetic)")
    fp64_ops = fp64_per_amp * (2 ** m) * args.steps
    fp64_rate = fp64_ops / (ms_dev / 1e3) / 1e12
    # the bit-exact numerics on the same workload, for comparison, and the
    # factored numerics' error against it on one step from the same state
    exact_cmp = numerics_error = None
    if factored and not args.no_exact_compare:
        ctx.queue.fuse = True
        step(sweeps[0])
        st.synchronize()
        st.event_record(0)
        for s in range(min(args.steps, 5)):
            step(sweeps[args.warmup + s])
        st.event_record(1)
        st.synchronize()
        ms_exact = max_over_ranks(dist, st.event_elapsed_ms(0, 1)) / min(args.steps, 5)
        ctx.queue.fuse = "factored"
        exact_cmp = {"value": units_per_step / (ms_exact / 1e3), "ms_per_step": ms_exact,
                     "numerics": "exact (QS_FUSE_EXACT: bit-identical to the reference's numpy "
                                 "arithmetic)"}
        if world == 1:
            numerics_error = factored_vs_exact(args, ctx, sweeps, step, n)
    config4_point = None
    if args.workload == "sweep" and world == 1 and not args.no_config4_point:
        del ctx, st
        config4_point = run_config4_point(args, 33, 3)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": devices, "ranks": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128 (f64 pairs)", "data": "synthetic",
            "config": {
                "workload": (f"config 2 sweep: Haar 2x2 on each of the {n} qubits in turn, "
                             if args.workload == "sweep" else
                             "config 3: CNOT, CPhase(phi) and controlled Haar 2x2 on each of "
                             "64 seeded (control, target) pairs, "
                             if cfg3 else
                             f"config 4 layer: Haar 2x2 on each of the {n} qubits, then "
                             f"CX(q, n-1-q) for q < {n // 2}, ")
                            + f"fresh unitaries per step, normalised Gaussian state, "
                            f"2^{m} c128 amplitudes per GPU (n={n}, {p} global qubits)",
                "qubits": n, "local_qubits": m, "gates_per_step": gates_per_step,
                "fused": not args.no_fuse,
                "numerics": ("factored (QS_FUSE_FACTORED: the controlled gates of a pair fused "
                             "into one controlled matrix; within 1e-12 of the reference, "
                             "tests/test_gpu_factored.py)" if factored and cfg3 else
                             "factored (QS_FUSE_FACTORED: Euler-factored 1q gates as 4-FMA "
                             "shears + merged diagonals; within 1e-12 of the reference, "
                             "tests/test_gpu_factored.py, tests/test_gpu_headline.py)"
                             if factored else
                             "exact (bit-identical to the reference's numpy arithmetic)"),
                "parallelism": (f"state sharded over {world} ranks on {devices} GPU(s)"
                                + (" (emulated: every rank on GPU 0)" if emulated else "")),
                "exchange": (None if world == 1 else
                             "qubit remapping (peer swap of half the slice)" if args.remap
                             else args.exchange),
                "l2": (f"inputs larger than L2 ({16 * 2 ** m / 2 ** 30:g} GiB state per GPU "
                       "vs 126 MB L2)" if 16 * 2 ** m > 126e6 else
                       f"state fits in L2 ({16 * 2 ** m / 2 ** 20:g} MiB): not a roofline run")},
            "hbm_gbs": hbm_gbs,
            "hbm_gbs_note": "algorithmic: 32 B/amplitude for every gate (what an unfused "
                            "gate-by-gate simulator moves); fusion moves less, see hbm_gbs_actual",
            "hbm_gbs_actual": actual_gbs,
            "hbm_actual_frac_of_measured": actual_gbs / peak,
            "passes_per_step": passes_per_step,
            "fp64": {"tera_ops_per_s": fp64_rate, "peak": FP64_PEAK_TOPS,
                     "frac": fp64_rate / FP64_PEAK_TOPS,
                     "note": fp64_note + "; peak = measured DFMA/DMUL/DADD issue rate "
                             "62 lanes/clk/SM x 148 SMs x 1.965 GHz (tools/exp/fp64.cu)"},
            "exact_numerics": exact_cmp,
            "numerics_error": numerics_error,
            "per_target_unfused": per_target,
            "roofline": {"kernel": LAUNCH_KINDS.get(dom, str(dom)), "bound": "hbm",
                         "achieved": physical, "peak": peak, "unit": "GB/s",
                         "frac": physical / peak, "traffic": traffic,
                         "bytes_per_launch": pass_bytes, "avg_launch_ms": dom_ms,
                         "fusion_gain": units_per_launch,
                         "algorithmic_per_gate_gbs": physical * units_per_launch,
                         "peak_source": peak_src,
                         "note": "achieved = 32*2^m B (one read + write of the slice, the "
                                 "pass's algorithmic bytes) / avg launch time (CUDA events on "
                                 "the library stream); traffic = ncu dram bytes per launch; "
                                 "fusion_gain = gate-updates per launch"},
            "nvlink": nvlink,
            "kernel_share": share,
            "gpu_launches": int(len(launch_ms)),
            "wall_s": wall,
            "clocks": clock,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_resident": e2e_resident,
            "config4_n33_single_gpu": config4_point,
        }
        print(json.dumps(line))
    barrier(dist)
    return 0


def factored_vs_exact(args, ctx, sweeps, step, n):
    """numerics_error: one timed-workload step in the factored numerics against
    the exact (bit-identical) path from the same state, on the device
    (qs_state_diff): max|d|, ||d||_2/||psi||_2, max|d|/max|psi|."""
    from paper_2001_10554_b200 import _native, runtime
    from paper_2001_10554_b200.workloads import device_gaussian

    other = runtime.make_context(None, n, 1, device=ctx.device, fuse=True)
    other.norm_check_interval = 0
    device_gaussian(ctx.state, args.seed + 5)
    device_gaussian(other.state, args.seed + 5)
    step(sweeps[-1], ctx)
    step(sweeps[-1], other)
    d = ctx.state.diff(other.state)
    del other
    return {"max_abs": d["max_abs"], "rel_l2": d["rel_l2"], "rel_max": d["rel_max"],
            "bound": 1e-12,
            "note": "one step of the timed workload in the factored numerics vs the exact "
                    "(bit-identical) path from the same normalised Gaussian state, full "
                    f"2^{n} state compared on the device; tests/test_gpu_headline.py pins "
                    "both against the CPU oracle at n=30"}


def run_config4_point(args, m, layers):
    """The N=1 point of config 4's weak-scaling curve (n=33, 128 GiB state,
    no global qubit): Haar on all 33 qubits + CX(q, 32-q), q < 16, per layer."""
    from paper_2001_10554_b200 import runtime
    from paper_2001_10554_b200.circuit import GateSpec
    from paper_2001_10554_b200.workloads import device_gaussian

    try:
        ctx = runtime.make_context(None, m, 1, fuse=fuse_mode(args))
    except MemoryError as exc:
        return {"skipped": f"n={m} state does not fit: {exc}"}
    ctx.norm_check_interval = 0
    st = ctx.state
    device_gaussian(st, args.seed)
    rng = np.random.default_rng(args.seed + 9)
    cx = [(q, m - 1 - q) for q in range(m // 2)]

    def layer():
        for k in range(m):
            runtime.apply_gate(ctx, GateSpec("custom", (k,), matrix=haar(rng)))
        for c, t in cx:
            runtime.apply_gate(ctx, GateSpec("cx", (c, t)))
        ctx.flush()

    layer()
    st.synchronize()
    st.event_record(0)
    for _ in range(layers):
        layer()
    st.event_record(1)
    st.synchronize()
    ms = st.event_elapsed_ms(0, 1) / layers
    gates = m + len(cx)
    del ctx, st
    return {"qubits": m, "ms_per_layer": ms, "layers": layers,
            "value": gates * (2.0 ** m) / 2.0 ** 30 / (ms / 1e3), "unit": UNIT,
            "numerics": args.numerics,
            "note": "config 4 at N=1 (n=33, every qubit local): the base of the weak-scaling "
                    "curve that --gpus N runs at 2^33 amplitudes per GPU"}


def run_e2e_resident(args, ctx, st, sweeps, step, n, dist, gates_per_step):
    """The same metric through the public API with the state resident in HBM
    (as a user of the drop-in keeps it): every step sends its 30 unitaries
    from host memory (runtime.apply_gate) and reads the step's metric back
    (runtime.measure_norm_squared -> host float).  Wall clock per step."""
    from paper_2001_10554_b200 import runtime

    k = max(3, args.steps)
    st.synchronize()
    barrier(dist)
    t0 = time.perf_counter()
    norms = []
    for s in range(k):
        step(sweeps[s % len(sweeps)])
        norms.append(float(runtime.measure_norm_squared(ctx)))
    dt = max_over_ranks(dist, time.perf_counter() - t0)
    units = gates_per_step * (2.0 ** n) / 2.0 ** 30
    return {"value": units * k / dt, "unit": UNIT, "h2d_bytes_per_step": 64 * gates_per_step,
            "d2h_bytes_per_step": 8, "steps": k, "norm_sq_last": norms[-1],
            "note": "state resident in HBM between steps (the drop-in's StatePartition); per "
                    "step the unitaries go host->device through runtime.apply_gate and the "
                    "step's norm^2 comes back through runtime.measure_norm_squared"}


def per_target_table(st, m, seed):
    """Config 2's per-target numbers: one Haar gate on target q as a single
    streaming kernel (k_gate1q), median of 3, algorithmic 32 B/amplitude."""
    from paper_2001_10554_b200 import _native as N

    rng = np.random.default_rng(seed + 7)
    peak, _ = measured_peak()
    rows = []
    for q in range(m):
        u = haar(rng).view(np.float64).ravel()
        g = [N.QsGate(0, q, -1, 0, 0, 0)]
        times = []
        for _ in range(3):
            st.event_record(2)
            st.apply_program(g, u, fuse=False)
            st.event_record(3)
            times.append(st.event_elapsed_ms(2, 3))
        ms = float(np.median(times))
        gbs = 32.0 * (2 ** m) / (ms / 1e3) / 1e9
        rows.append({"q": q, "ms": round(ms, 4), "gbs": round(gbs, 1),
                     "frac_of_measured": round(gbs / peak, 4), "frac_of_8tbs": round(gbs / 8000, 4)})
    return {"kernel": "k_gate1q", "rows": rows,
            "min_frac_of_measured": min(r["frac_of_measured"] for r in rows),
            "min_frac_of_8tbs": min(r["frac_of_8tbs"] for r in rows)}


def run_e2e(args, ctx, st, sweeps, step, m, n, dist, gates_per_step):
    """Same metric through the public API with pinned host buffers: every step
    uploads the state (StatePartition.amplitudes = host), runs the gates
    (runtime.apply_gate) and reads the result back (read_amplitudes)."""
    import torch

    from paper_2001_10554_b200 import statevector as sv

    k = max(1, args.e2e_steps)
    host_in = torch.empty(2 << m, dtype=torch.float64, pin_memory=True).numpy().view(np.complex128)
    host_out = torch.empty(2 << m, dtype=torch.float64, pin_memory=True).numpy().view(np.complex128)
    sv.read_amplitudes(ctx.partition, host_in)
    barrier(dist)
    t0 = time.perf_counter()
    ctx.partition.amplitudes = host_in                      # step 0 input
    for s in range(k):
        step(sweeps[s % len(sweeps)])
        if s + 1 < k:
            # step s result out while step s+1 input comes in (full duplex)
            sv.exchange_amplitudes(ctx.partition, host_in, host_out)
        else:
            sv.read_amplitudes(ctx.partition, host_out)
    dt = time.perf_counter() - t0
    dt = max_over_ranks(dist, dt)
    units = gates_per_step * (2.0 ** n) / 2.0 ** 30
    return {"value": units * k / dt, "unit": UNIT, "h2d_bytes_per_step": 16 * (2 ** m),
            "d2h_bytes_per_step": 16 * (2 ** m), "steps": k,
            "note": "per GPU bytes; wall clock around every step's input upload, gates and "
                    "result download through the public API (amplitudes setter / "
                    "exchange_amplitudes, runtime.apply_gate, read_amplitudes); a step's "
                    "download and the next step's upload share one full-duplex transfer"}


QAOA_N, QAOA_P, QAOA_POOL = 20, 4, 512


def pso_step(pos, vel, best_pos, best_val, gbest, values, rng, lo=0.0, hi=np.pi):
    """Standard PSO move (reference optimize.py:79-117 restated for the pool
    driver): fold in values, then v <- w v + phi_p r_p (best - x) + phi_g r_g (g - x)."""
    better = values > best_val
    best_val = np.where(better, values, best_val)
    best_pos = np.where(better[:, None], pos, best_pos)
    k = int(np.argmax(best_val))
    gbest = best_pos[k].copy()
    r = rng.random((pos.shape[0], 2))
    vel = 0.66 * vel + 1.6 * r[:, :1] * (best_pos - pos) + 0.62 * r[:, 1:] * (gbest - pos)
    pos = lo + np.mod(pos + vel - lo, hi - lo)
    return pos, vel, best_pos, best_val, gbest


def qaoa_tables(positions, depth):
    """Per-state slot tables: qaoa_bindings (circuit.py) for every row, as
    columns (gamma_k = x[k-1], beta_k = 2 * x[p+k-1]; same IEEE products)."""
    pos = np.asarray(positions, dtype=np.float64)
    tables = {}
    for k in range(1, depth + 1):
        tables[f"gamma{k}"] = pos[:, k - 1].copy()
        tables[f"beta{k}"] = 2.0 * pos[:, depth + k - 1]
    return tables


def exact_maxcut(graph, n):
    idx = np.arange(1 << n, dtype=np.uint64)
    cuts = np.zeros(idx.shape, dtype=np.float64)
    for u, v in graph.edges:
        cuts += ((idx >> np.uint64(u)) ^ (idx >> np.uint64(v))) & np.uint64(1)
    return float(cuts.max())


def cpu_qaoa_sample(graph, positions, depth, threads):
    """Reference algorithm (oracle port) on the host: `threads` QAOA circuits
    evaluated concurrently, one per host thread (numpy releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import circuit as ocirc
    from oracle import statevector as osv

    n = graph.num_vertices
    edges = list(graph.edges)

    def one(pos):
        prog = [{"kind": "h", "qubits": (q,)} for q in range(n)]
        for k in range(depth):
            prog.append({"kind": "diagcost", "param": pos[k], "edges": edges})
            prog += [{"kind": "rx", "qubits": (q,), "param": 2.0 * pos[depth + k]}
                     for q in range(n)]
        return osv.maxcut_expectation(ocirc.run(n, prog), edges)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        vals = list(ex.map(one, positions[:threads]))
    dt = time.perf_counter() - t0
    return len(vals) / dt, dt, vals


def run_qaoa(args, dist, comm, world, rank, local):
    """BASELINE config 5 as the reference's `qpool qaoa-pso --vertices 20
    --depth 4 --particles 512 --budget 512*K` runs it (cli.py:249-262,
    optimize.py:172-216): the keyed 3-regular graph
    random_3regular_graph(20, pool_stream.split(0)), the keyed swarm
    init_swarm(512, 8, stream=pool_stream.split(1)), and per swarm step all 512
    particles evaluated as one pool program (reset + 104 gates + <C>), the
    values shared pool-wide, then step_swarm.  The pool is split across GPUs
    in contiguous blocks (no state exchange).  Parameter tables go
    host->device and <C> device->host inside every step (the step is end to
    end)."""
    from paper_2001_10554_b200 import optimize as qopt
    from paper_2001_10554_b200 import runtime
    from paper_2001_10554_b200.circuit import build_qaoa_circuit
    from paper_2001_10554_b200.noise import SCOPE_POOL, RandomStream

    n, depth, S = QAOA_N, QAOA_P, QAOA_POOL
    first, count = runtime.split_pool(S, rank, world)
    pool_stream = RandomStream(args.seed, SCOPE_POOL, 0)
    graph = qopt.random_3regular_graph(n, pool_stream.split(0))
    circ = build_qaoa_circuit(graph, depth)
    exact = qopt.exact_maxcut(graph)
    swarm = qopt.init_swarm(S, 2 * depth, stream=pool_stream.split(1))
    ctxs = qopt.pool_contexts(n, count, args.pool_chunks, args.seed, device=local,
                              fuse=fuse_mode(args))
    for c in ctxs:
        c.norm_check_interval = 0
    edges = np.asarray(graph.edges, dtype=np.int32)
    host_ms = []

    def share(mine):
        if dist is None:
            return mine
        import torch

        buf = torch.zeros(S, dtype=torch.float64)
        buf[first:first + count] = torch.from_numpy(mine)
        dist.all_reduce(buf)  # disjoint blocks: the sum is the concatenation
        return buf.numpy()

    def step():
        pos = np.stack([swarm.particles[k].position for k in range(first, first + count)])
        mine = qopt.evaluate_swarm(ctxs, circ, pos, depth, edges) / exact
        values = share(np.asarray(mine, dtype=np.float64))
        t = time.perf_counter()
        qopt.step_swarm(swarm, values)
        host_ms.append(1e3 * (time.perf_counter() - t))
        return values

    for _ in range(args.warmup):
        step()
    for c in ctxs:
        c.state.synchronize()
    barrier(dist)
    host_ms.clear()
    clocks = ClockSampler(local)
    clocks.start()
    for c in ctxs:
        c.state.launch_log(True)
    folds0 = {id(c): c.pool.state.uniform_folds for c in ctxs}
    t0 = time.perf_counter()
    for _ in range(args.steps):
        values = step()
    for c in ctxs:
        c.state.synchronize()
    wall = time.perf_counter() - t0
    logs = []
    for c in ctxs:
        c.state.launch_log(False)
        logs.append(c.state.read_launch_log())
    launch_ms = np.concatenate([l[0] for l in logs])
    launch_kind = np.concatenate([l[1] for l in logs])
    clock = clocks.stop()
    wall = max_over_ranks(dist, wall)
    gates_per_circuit = len(circ.gates)
    circuits = S * args.steps
    units = circuits * gates_per_circuit * (2.0 ** n) / 2.0 ** 30
    value = units / wall
    kinds = {}
    for k, t in zip(launch_kind, launch_ms):
        kinds.setdefault(int(k), []).append(float(t))
    dev_ms = sum(sum(v) for v in kinds.values())
    peak, peak_src = measured_peak()
    gates_per_step = count * len(circ.gates)
    pass_kinds = [k for k in kinds if LAUNCH_KINDS.get(k, "") in PASS_KINDS]
    # bytes the pass launches move: a read + write of the chunk's states (32 B per
    # amplitude); a pass that generates its uniform input in registers
    # (k_fact_gen) only writes; in the exact mode the uniform state is filled
    # (16 B per amplitude) inside the first pass's launch scope
    pass_bytes_total = 0.0
    folds = 0
    for c, (_, lk) in zip(ctxs, logs):
        amps_c = c.num_states * 2.0 ** n
        for k in lk:
            name = LAUNCH_KINDS.get(int(k), "")
            if name in PASS_KINDS:
                pass_bytes_total += (16.0 if name == "k_fact_gen" else 32.0) * amps_c
        filled = c.pool.state.uniform_folds - folds0[id(c)] - int(np.sum(np.asarray(lk) == 8))
        pass_bytes_total += 16.0 * amps_c * max(0, filled)
        folds += c.pool.state.uniform_folds - folds0[id(c)]
    passes_per_step = sum(len(kinds[k]) for k in pass_kinds) / args.steps
    pass_ms = sum(sum(kinds[k]) for k in pass_kinds) / args.steps
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import cpu_baseline as cb

        pos = np.stack([p.position for p in swarm.particles])
        cps, dt, _ = cpu_qaoa_sample(graph, pos, depth, cb.threads())
        cpu = {"value": cps * gates_per_circuit * (2.0 ** n) / 2.0 ** 30, "unit": UNIT,
               "cores": cb.threads(), "kind": "port",
               "sample": f"{cb.threads()} QAOA circuits (n={n}, p={depth}, {gates_per_circuit} "
                         f"gates + <C>) on {cb.threads()} host threads, oracle port, {dt:.2f} s",
               "circuits_per_s": cps}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c128 (f64 pairs)", "data": "synthetic",
            "config": {"workload": f"config 5: qaoa-pso --vertices {n} --depth {depth} "
                                   f"--particles {S} --seed {args.seed}: keyed random 3-regular "
                                   "graph (pool_stream.split(0)), keyed swarm "
                                   "(pool_stream.split(1)), one swarm step = the 512 "
                                   "circuits as pool programs (one per sub-pool chunk, the "
                                   "reset + Hadamard layer folded into a uniform start) + <C> "
                                   "+ step_swarm",
                       "pool": S, "per_gpu": count, "swarm_steps": args.steps,
                       "gates_per_circuit": gates_per_circuit, "fused": not args.no_fuse,
                       "numerics": args.numerics,
                       "l2": f"pool of {count} x 2^{n} c128 = {count * 16 * 2 ** n / 2 ** 30:.0f} "
                             "GiB per GPU, larger than L2"},
            "circuits_per_s": circuits / wall,
            "global_best_ratio": float(swarm.global_best_value),
            "host_pso_ms_per_step": float(np.mean(host_ms)) if host_ms else None,
            "pass_ms_per_step": pass_ms, "passes_per_step": passes_per_step,
            "roofline": pool_roofline(kinds, 32.0 * (2 ** n) * count / len(ctxs),
                                      count * (2 ** n) / len(ctxs),
                                      gates_per_step / count, peak, peak_src, "qaoa",
                                      args.steps * len(ctxs), total_bytes=pass_bytes_total),
            "pool_chunks": len(ctxs),
            "uniform_start_folds_per_step": folds / args.steps,
            "kernel_share": {LAUNCH_KINDS.get(k, str(k)): {"launches": len(v),
                                                           "share": float(np.sum(v) / dev_ms)}
                             for k, v in kinds.items()},
            "gpu_launches": int(len(launch_ms)),
            "clocks": clock,
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT,
                    "h2d_bytes_per_step": int(count * (2 * depth * 8 * n + 2 * 31 * 16 * depth)),
                    "d2h_bytes_per_step": int(8 * count),
                    "note": "the step itself is end to end: parameter tables up, <C> down"},
        }
        print(json.dumps(line))
    barrier(dist)
    return 0



def run_cfg1(args, dist, world, rank, local):
    """BASELINE config 1 (n=20, 10 layers of H/RX/RZ + brick CNOTs, 295 gates,
    |0...0>), the reference's CPU-runnable case, through the public API: a
    step is one runtime.simulate_circuit call -- context, the fused program,
    and the download of the full 2^20-amplitude state, as the reference
    returns it (runtime.py:291-302).  Every rank runs its own replica."""
    from paper_2001_10554_b200 import runtime
    from paper_2001_10554_b200.circuit import Circuit
    from paper_2001_10554_b200.workloads import config1_gates

    n = 20
    circ = Circuit(n, tuple(config1_gates(n, 10, args.seed)))
    psi = None
    for _ in range(args.warmup):
        psi = runtime.simulate_circuit(circ, device=local)
    barrier(dist)
    clocks = ClockSampler(local)
    clocks.start()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        psi = runtime.simulate_circuit(circ, device=local)
    wall = time.perf_counter() - t0
    clock = clocks.stop()
    wall = max_over_ranks(dist, wall)
    gates = len(circ.gates)
    units = world * args.steps * gates * (2.0 ** n) / 2.0 ** 30
    # kernels one call launches (a context made the way simulate_circuit makes it)
    cctx = runtime.make_context(None, n, 1, 0, device=local)
    cctx.state.launch_log(True)
    runtime.run_circuit(cctx, circ)
    cctx.flush()
    cctx.state.synchronize()
    cctx.state.launch_log(False)
    launches = len(cctx.state.read_launch_log()[0])
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import circuit as ocirc

        prog = [{"kind": g.kind, "qubits": g.qubits, "param": g.param} for g in circ.gates]
        t1 = time.perf_counter()
        ref = ocirc.run(n, prog)
        dt = time.perf_counter() - t1
        cpu = {"value": gates * (2.0 ** n) / 2.0 ** 30 / dt, "unit": UNIT, "cores": 1,
               "kind": "port",
               "sample": f"one config-1 circuit ({gates} gates, n={n}) through the oracle's "
                         f"gate-by-gate restatement of run_circuit (numpy, 1 thread), {dt:.2f} s",
               "max_abs_diff_vs_ours": float(np.max(np.abs(ref - psi))),
               "bit_identical_to_ours": bool(np.array_equal(ref.view(np.uint64),
                                                            np.asarray(psi).view(np.uint64)))}
    if rank == 0:
        value = units / wall
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128 (f64 pairs)", "data": "synthetic",
            "config": {"workload": f"config 1: n={n}, 10 layers of H/RX(theta)/RZ(theta) per qubit "
                                   f"+ brick CNOTs ({gates} gates) from |0...0>, one "
                                   "runtime.simulate_circuit call per step (exact numerics, "
                                   "full state downloaded)",
                       "gates_per_step": gates, "replicas": world,
                       "l2": "state (16 MiB) fits in L2: an API-latency workload, not a "
                             "roofline run"},
            "circuits_per_s": world * args.steps / wall,
            "roofline": None,
            "gpu_launches": int(launches * args.steps),
            "clocks": clock,
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 16 * (2 ** n),
                    "note": "the step is the public API call itself: gate list in, the "
                            "full state out"},
        }
        print(json.dumps(line))
    barrier(dist)
    return 0

PASS_KINDS = ("k_tile", "k_fact", "k_fact_gen")


def pool_roofline(kinds, pass_bytes, amps, gates_per_state, peak, peak_src, tag, steps,
                  total_bytes=None):
    """Roofline of a pool step's fused passes (every k_fact / k_tile launch):
    achieved = one read + write of this GPU's pool per pass (32 B per
    amplitude) x passes / their summed launch time; traffic = ncu dram bytes
    per amplitude of the same workload's capture (profiles/ncu_traffic.json,
    key kernel@tag) x amplitudes; fusion_gain = gate-updates per state per pass."""
    passes = {LAUNCH_KINDS.get(k, str(k)): v for k, v in kinds.items()
              if LAUNCH_KINDS.get(k, "") in PASS_KINDS}
    n = sum(len(v) for v in passes.values())
    ms = sum(sum(v) for v in passes.values())
    dom = max(passes, key=lambda k: sum(passes[k])) if passes else None
    moved = pass_bytes * n if total_bytes is None else total_bytes
    achieved = moved / (ms / 1e3) / 1e9 if ms else None
    tr = ncu_traffic(f"{dom}@{tag}") if dom else None
    traffic = tr["bytes_per_amplitude"] * amps if tr and tr.get("bytes_per_amplitude") else None
    return {"kernel": "+".join(sorted(passes)), "bound": "hbm", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak if achieved else None, "traffic": traffic,
            "bytes_per_launch": pass_bytes, "avg_launch_ms": ms / n if n else None,
            "launches": n, "fusion_gain": gates_per_state * steps / (n or 1),
            "per_kernel_ms": {k: float(np.mean(v)) for k, v in passes.items()},
            "peak_source": peak_src,
            "note": "achieved = 32 B per amplitude of this GPU's pool per pass (one read + "
                    "write) x pass launches / their summed device time (CUDA events on "
                    "the library stream); fusion_gain = gate-updates per state per pass"}


NOISE_T1, NOISE_T2 = 500.0, 250.0  # the reference's noise study defaults (noise_convergence_study.py)


def noise_instance(seed):
    """Config 5's circuit shape (n=20, p=4 QAOA on a random 3-regular graph)
    at one fixed parameter point, with schedule_noise() applied: the noisy
    QAOA ensemble of the reference's noise study, at config-5 size."""
    from paper_2001_10554_b200 import noise
    from paper_2001_10554_b200.circuit import build_qaoa_circuit, qaoa_bindings
    from paper_2001_10554_b200.workloads import random_3regular_graph

    rng = np.random.default_rng(seed)
    graph = random_3regular_graph(QAOA_N, rng)
    point = rng.uniform(0, np.pi, size=2 * QAOA_P)
    circ = build_qaoa_circuit(graph, QAOA_P).bind(qaoa_bindings(QAOA_P, point))
    return graph, noise.schedule_noise(circ)


def cpu_noise_sample(circ, graph, seed, threads):
    """Oracle port on the host: `threads` trajectories concurrently, each the
    reference's scalar path (numpy Philox per noise gate, gate by gate)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import circuit as ocirc
    from oracle import noise as onoise
    from oracle import statevector as osv

    n = circ.num_qubits
    edges = list(graph.edges)
    glist = []
    for g in circ.gates:
        if g.kind == "diagcost":
            glist.append({"kind": "diagcost", "param": g.param, "edges": edges})
        else:
            glist.append({"kind": g.kind, "qubits": g.qubits, "param": g.param,
                          "duration": g.duration})

    def one(t):
        prog = onoise.bind_trajectory(glist, NOISE_T1, NOISE_T2, seed, t)
        return osv.maxcut_expectation(ocirc.run(n, prog), edges)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        vals = list(ex.map(one, range(threads)))
    dt = time.perf_counter() - t0
    return len(vals) / dt, dt, vals


def run_noise(args, dist, comm, world, rank, local):
    """Noise trajectories in pool mode (cli.py:288-339):
    512 trajectories of the noisy config-5 QAOA circuit per step, one pool
    round -- per-trajectory noise matrices drawn on the host in one pass,
    the whole round applied as fused tile programs with per-state tables,
    <C> per trajectory read back.  Trajectories are split across GPUs in
    contiguous blocks (no state exchange); trajectory t equals a serial run
    of index t bit for bit."""
    from paper_2001_10554_b200 import noise, runtime

    n, S = QAOA_N, QAOA_POOL
    first, count = runtime.split_pool(S, rank, world)
    graph, circ = noise_instance(args.seed)
    model = noise.NoiseModel(NOISE_T1, NOISE_T2)
    ctx = runtime.make_context(None, n, num_states=count, device=local, fuse=fuse_mode(args),
                               seed=args.seed, noise_model=model)
    ctx.norm_check_interval = 0
    # a second pool of the same shape: round k+1's program is built and enqueued
    # while round k runs (runtime.run_noise_ensemble(shadow=...) does the same)
    shadow = runtime.make_context(None, n, num_states=count, device=local, fuse=fuse_mode(args),
                                  seed=args.seed, noise_model=model)
    shadow.norm_check_interval = 0
    ctxs = [ctx, shadow]
    st = ctx.state
    edges = np.asarray(graph.edges, dtype=np.int32)
    durations = [g.duration for g in circ.gates if g.kind == "noise"]
    from concurrent.futures import ThreadPoolExecutor

    pool = ThreadPoolExecutor(1)

    def draw(k):
        # round k's trajectories: k*S + first .. k*S + first + count - 1
        batch = noise.StreamBatch(noise.trajectory_stream(args.seed, k * S + first + s)
                                  for s in range(count))
        return noise.circuit_noise_matrices(durations, model, batch)

    round_no = [0]
    pending = [pool.submit(draw, 0)]

    behind = [None]  # the context whose round is still on the device

    def drain():
        c, behind[0] = behind[0], None
        return c.pool.observable(3, 0, edges) if c is not None else None

    def step():
        # the next round's host draws (worker thread) and this round's program
        # build overlap the previous round's device work; its <C> values are
        # read back once this round is enqueued
        k = round_no[0]
        round_no[0] += 1
        c = ctxs[k % 2]
        mats = pending[0].result()
        if behind[0] is not None:  # no interleaving of the two pools' kernels
            c.state.wait_event(behind[0].state.sync_event(0))
        runtime.reset_state(c)
        runtime.run_circuit(c, circ, noise_matrices=mats)
        c.state.record_sync_event(0)
        pending[0] = pool.submit(draw, k + 1)
        vals = drain()
        behind[0] = c
        return vals

    for _ in range(args.warmup):
        step()
    drain()  # the timed region starts with an empty pipeline ...
    for c in ctxs:
        c.state.synchronize()
    barrier(dist)
    clocks = ClockSampler(local)
    clocks.start()
    for c in ctxs:
        c.state.launch_log(True)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    values = drain()  # ... and ends with the last round's values on the host
    for c in ctxs:
        c.state.synchronize()
    wall = time.perf_counter() - t0
    logs = []
    for c in ctxs:
        c.state.launch_log(False)
        logs.append(c.state.read_launch_log())
    launch_ms = np.concatenate([l[0] for l in logs])
    launch_kind = np.concatenate([l[1] for l in logs])
    clock = clocks.stop()
    wall = max_over_ranks(dist, wall)
    gates_per_circuit = len(circ.gates)
    noise_gates = sum(g.kind == "noise" for g in circ.gates)
    trajectories = S * args.steps
    value = trajectories * gates_per_circuit * (2.0 ** n) / 2.0 ** 30 / wall
    kinds = {}
    for k, t in zip(launch_kind, launch_ms):
        kinds.setdefault(int(k), []).append(float(t))
    dev_ms = sum(sum(v) for v in kinds.values())
    peak, peak_src = measured_peak()
    gates_per_step = count * len(circ.gates)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import cpu_baseline as cb

        tps, dt, _ = cpu_noise_sample(circ, graph, args.seed, cb.threads())
        cpu = {"value": tps * gates_per_circuit * (2.0 ** n) / 2.0 ** 30, "unit": UNIT,
               "cores": cb.threads(), "kind": "port",
               "sample": f"{cb.threads()} noisy trajectories (n={n}, {gates_per_circuit} gates "
                         f"incl. {noise_gates} noise gates, + <C>) on {cb.threads()} host "
                         f"threads, oracle port, {dt:.2f} s",
               "trajectories_per_s": tps}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c128 (f64 pairs)", "data": "synthetic",
            "config": {"workload": f"noise ensemble: {S} trajectories per step of the noisy "
                                   f"config-5 QAOA circuit (n={n}, p={QAOA_P}, schedule_noise, "
                                   f"T1={NOISE_T1}, T2={NOISE_T2}), <C> per trajectory",
                       "pool": S, "per_gpu": count, "gates_per_circuit": gates_per_circuit,
                       "noise_gates": noise_gates, "fused": not args.no_fuse,
                       "numerics": args.numerics},
            "trajectories_per_s": trajectories / wall,
            "mean_cut": float(np.mean(values)),
            "roofline": pool_roofline(kinds, 32.0 * (2 ** n) * count, count * (2 ** n),
                                      gates_per_step / count, peak, peak_src, "noise", args.steps),
            "kernel_share": {LAUNCH_KINDS.get(k, str(k)): {"launches": len(v),
                                                           "share": float(np.sum(v) / dev_ms)}
                             for k, v in kinds.items()},
            "device_ms_per_step": dev_ms / args.steps,
            "gpu_launches": int(len(launch_ms)),
            "clocks": clock,
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT,
                    "h2d_bytes_per_step": int(count * noise_gates * 64),
                    "d2h_bytes_per_step": int(8 * count),
                    "note": "the step itself is end to end: noise matrices up, <C> down"},
        }
        print(json.dumps(line))
    barrier(dist)
    return 0


def spawn_ranks(args) -> int:
    """`--gpus N` without torchrun: re-run this command under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous)
    and hand back its exit code; rank 0 prints the JSON line."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
