"""The reference's acceptance criteria (pkg/tests/test_acceptance.py) run
against the B200 core: oracle equivalence over rank counts (1), per-rank
memory layout (3), T1/T2 decay anchors (5), running-mean convergence (6), the
PSO/QAOA desk study (7) and determinism (8).  Criterion 2 (exchange
accounting) is test_gpu_parity.test_exchange_accounting_matches_reference and
criterion 4 (pool partitioning) is test_host_logic's build_pool test."""
import math
import time

import numpy as np
import pytest

from paper_2001_10554_b200 import noise as N
from paper_2001_10554_b200 import optimize as opt
from paper_2001_10554_b200 import runtime, statevector as sv
from paper_2001_10554_b200.circuit import Circuit, GateSpec
from paper_2001_10554_b200.graphs import make_graph

from conftest import bits_equal, max_dev
from oracle import circuit as ocirc

pytestmark = pytest.mark.gpu

RING8 = [(q, (q + 1) % 8) for q in range(8)]


def random_circuit(n, count, rng):
    specs, plain = [], []
    for _ in range(count):
        r = rng.random()
        if r < 0.45:
            k = ("h", "x", "y", "z")[int(rng.integers(4))]
            q = int(rng.integers(n))
            specs.append(GateSpec(k, (q,)))
            plain.append({"kind": k, "qubits": (q,)})
        elif r < 0.75:
            k = ("rx", "ry", "rz")[int(rng.integers(3))]
            q, th = int(rng.integers(n)), float(rng.uniform(0, 2 * np.pi))
            specs.append(GateSpec(k, (q,), th))
            plain.append({"kind": k, "qubits": (q,), "param": th})
        elif r < 0.93:
            k = ("cx", "cz")[int(rng.integers(2))]
            c, t = (int(x) for x in rng.choice(n, size=2, replace=False))
            specs.append(GateSpec(k, (c, t)))
            plain.append({"kind": k, "qubits": (c, t)})
        else:
            g = float(rng.uniform(0, 2 * np.pi))
            specs.append(GateSpec("diagcost", (), g, graph=make_graph(n, RING8)))
            plain.append({"kind": "diagcost", "param": g, "edges": RING8})
    return Circuit(n, tuple(specs)), plain


def test_criterion_1_oracle_equivalence():
    """100 random 50-gate circuits at n=8 on 1/2/4/8 emulated ranks."""
    rng = np.random.default_rng(20260401)
    t0 = time.perf_counter()
    for trial in range(100):
        circ, plain = random_circuit(8, 50, rng)
        expected = ocirc.run(8, plain)
        for ranks in (1, 2, 4, 8):
            got = runtime.simulate_circuit(circ, num_ranks=ranks)
            assert max_dev(got, expected) < 1e-12, (trial, ranks)
            assert bits_equal(got, expected), (trial, ranks)
    assert time.perf_counter() - t0 < 300.0


def test_criterion_3_memory_layout():
    def rank_fn(comm):
        ctx = runtime.make_context(comm, 12, 1)
        return ctx.partition.amplitudes.size

    assert runtime.run_spmd(4, rank_fn) == [2 ** 10] * 4
    part = sv.allocate_partition(9, num_local_qubits=6, rank_index=3)
    assert part.amplitudes.size == 2 ** 6
    assert sv.full_state_bytes(30) == 2 ** (3 + 1 + 30)


def _trajectory_values(model, plus, duration, count, master_seed):
    """One noise gate on qubit 0 of `count` single-qubit states, state k
    drawing from RandomStream(master_seed, "state", k) -- one pool program."""
    ctx = runtime.make_context(None, 1, count, noise_model=model)
    if plus:
        ctx.pool.state.upload(np.full(2 * count, 1 / math.sqrt(2), dtype=np.complex128))
    else:
        runtime.reset_state(ctx)
    batch = N.StreamBatch(N.RandomStream(master_seed, "state", k) for k in range(count))
    runtime.apply_gate(ctx, GateSpec("noise", (0,), duration=duration), noise_stream=batch)
    a = ctx.pool.amplitudes()
    if plus:  # <X> = 2 Re(conj(a0) a1)
        return 2 * (a[:, 0].conjugate() * a[:, 1]).real
    return np.abs(a[:, 0]) ** 2 - np.abs(a[:, 1]) ** 2  # <Z>


def test_criterion_5_noise_physics():
    model = N.NoiseModel(500.0, 250.0)
    target = math.exp(-1.0)
    xs = _trajectory_values(model, True, 250.0, 2000, 501)
    se = xs.std(ddof=1) / math.sqrt(xs.size)
    assert abs(xs.mean() - target) < 3 * se
    zs = _trajectory_values(model, False, 500.0, 2000, 502)
    se = zs.std(ddof=1) / math.sqrt(zs.size)
    assert abs(zs.mean() - target) < 3 * se


def test_criterion_6_convergence_scaling():
    model = N.NoiseModel(500.0, 250.0)
    running = np.array([np.cumsum(v) / np.arange(1, v.size + 1) for v in
                        (_trajectory_values(model, True, 250.0, 1000, 2000 + s)
                         for s in range(20))])
    grid = np.unique(np.round(np.logspace(1, 3, 12)).astype(int))
    spread = running[:, grid - 1].std(axis=0, ddof=1)
    slope, _ = np.polyfit(np.log(grid), np.log(spread), 1)
    assert 0.4 <= -slope <= 0.6


def test_criterion_7_pso_study():
    """PSO over QAOA (p=2) on 20 random 3-regular 8-vertex graphs, R in
    {4, 8, 16}, budget 1000 evaluations: monotone traces, mean final ratio
    >= 0.8 and above the first batch.  The pool holds one state per
    particle, so each batch is one program."""
    seed = 2026
    base = N.RandomStream(seed, "pool", 0)
    graphs = [opt.random_3regular_graph(8, base.split(2 * k)) for k in range(20)]
    t0 = time.perf_counter()
    for R in (4, 8, 16):
        ctx = runtime.make_context(None, 8, R, seed=seed)
        finals, firsts = [], []
        for k, graph in enumerate(graphs):
            trace = opt.run_pso_qaoa(ctx, graph, 2, R, 1000, base.split(2 * k + 1))
            ratios = [row.global_best_ratio for row in trace]
            assert all(b >= a for a, b in zip(ratios, ratios[1:]))
            firsts.append(ratios[0])
            finals.append(ratios[-1])
        assert float(np.mean(finals)) >= 0.8
        assert float(np.mean(finals)) > float(np.mean(firsts))
    assert time.perf_counter() - t0 < 600.0


def test_criterion_8_determinism():
    """Bit-identical results across reruns, rank counts and pool layouts."""
    rng = np.random.default_rng(8)
    circ, _ = random_circuit(10, 80, rng)
    first = runtime.simulate_circuit(circ, num_ranks=4)
    assert bits_equal(first, runtime.simulate_circuit(circ, num_ranks=4))
    assert bits_equal(first, runtime.simulate_circuit(circ, num_ranks=1))
    model = N.NoiseModel(30.0, 15.0)
    noisy = N.schedule_noise(circ)
    pool = runtime.make_context(None, 10, 3, seed=9)
    _, v3 = runtime.run_noise_ensemble(pool, noisy, model, 6, lambda c: runtime.measure_z(c, 2))
    one = runtime.make_context(None, 10, 1, seed=9)
    _, v1 = runtime.run_noise_ensemble(one, noisy, model, 6, lambda c: runtime.measure_z(c, 2))
    assert np.array_equal(v1, v3)
