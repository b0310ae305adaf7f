"""GPU parity of QS_FUSE_FACTORED (include/qsb200.h, csrc/factor.cu).

The factored rewrite computes the same operator as the reference's gate-by-gate
numpy update (statevector.py:144-150) with different rounding, so the bar is
the north_star tolerance, not bit equality: max |d amplitude| <= 1e-12
(absolute) and expectation values within 1e-10 relative.  The oracle and the
reference's golden vectors are the checkers, as in test_gpu_parity.py.
"""
import numpy as np
import pytest

import paper_2001_10554_b200 as qs
from paper_2001_10554_b200 import _native as N
from paper_2001_10554_b200 import runtime
from paper_2001_10554_b200.circuit import Circuit, build_qaoa_circuit, qaoa_bindings
from paper_2001_10554_b200.graphs import make_graph

from conftest import bits_equal, golden, max_dev

from oracle import circuit as ocirc
from oracle import gates as ogates

pytestmark = pytest.mark.gpu
TOL = 1e-12       # amplitudes, absolute (north_star)
RTOL_OBS = 1e-10  # expectation values, relative (north_star)
FACT = "factored"

H = np.array([[1, 1], [1, -1]], dtype=np.complex128) / np.sqrt(2)
X = np.array([[0, 1], [1, 0]], dtype=np.complex128)


def mixed_program(n, count, rng):
    """Everything the rewrite distinguishes: Haar (both shear forms), exactly
    anti-diagonal (X), exactly diagonal (RZ, phase), rotations, controlled
    Haar / CNOT (mixing the target), CPhase (diagonal controlled), cut phases."""
    edges = [(0, 3), (2, 7), (5, 11), (1, n - 1), (4, 9)]
    out = []
    for _ in range(count):
        r = rng.random()
        q = int(rng.integers(n))
        if r < 0.45:
            out.append({"kind": "custom", "qubits": (q,), "matrix": ogates.random_unitary_2x2(rng)})
        elif r < 0.52:
            out.append({"kind": "custom", "qubits": (q,), "matrix": X})
        elif r < 0.60:
            out.append({"kind": "custom", "qubits": (q,), "matrix": H})
        elif r < 0.68:
            out.append({"kind": "custom", "qubits": (q,),
                        "matrix": ogates.rz(float(rng.uniform(0, 6.3)))})
        elif r < 0.74:
            out.append({"kind": "custom", "qubits": (q,),
                        "matrix": ogates.rx(float(rng.uniform(0, 6.3)))})
        else:
            t = int(rng.integers(n - 1))
            t = t if t < q else t + 1
            rr = rng.random()
            if rr < 0.4:
                u = ogates.random_unitary_2x2(rng)
            elif rr < 0.7:
                u = X
            else:
                u = np.diag([1.0, np.exp(1j * rng.uniform(0, 6.3))]).astype(np.complex128)
            if rng.random() < 0.15:
                out.append({"kind": "diagcost", "param": float(rng.uniform(0, 6.28)),
                            "edges": edges})
            else:
                out.append({"kind": "cu", "qubits": (q, t), "matrix": u})
    return out, edges


def run_queue(n, prog, edges, psi0, fuse):
    st = N.DeviceState(n, n)
    st.upload(psi0)
    graph = make_graph(n, edges)
    q = runtime.GateQueue(st, fuse=fuse)
    for g in prog:
        if g["kind"] == "custom":
            q.one_qubit(g["qubits"][0], g["matrix"])
        elif g["kind"] == "cu":
            q.controlled(*g["qubits"], g["matrix"])
        else:
            q.cut_phase(graph, g["param"])
    passes = q.flush()
    return st.download(), passes


@pytest.mark.parametrize("n", [12, 14, 17])
def test_factored_random_programs_within_tolerance(n):
    rng = np.random.default_rng(700 + n)
    for trial in range(3):
        prog, edges = mixed_program(n, 90, rng)
        psi0 = ogates.random_state(n, rng)
        expect = ocirc.run(n, prog, psi0)
        got, passes = run_queue(n, prog, edges, psi0, FACT)
        assert max_dev(got, expect) <= TOL, f"n={n} trial={trial}"
        assert passes < len(prog)


def test_factored_layer_is_not_the_exact_path():
    """The rewrite really runs (different rounding) and stays within 1e-12."""
    n = 14
    rng = np.random.default_rng(3)
    prog = [{"kind": "custom", "qubits": (q,), "matrix": ogates.random_unitary_2x2(rng)}
            for q in range(n)]
    psi0 = ogates.random_state(n, rng)
    exact, _ = run_queue(n, prog, [], psi0, True)
    fact, _ = run_queue(n, prog, [], psi0, FACT)
    assert bits_equal(exact, ocirc.run(n, prog, psi0))
    assert not bits_equal(exact, fact)
    assert max_dev(exact, fact) <= TOL


def test_factored_only_diagonals_and_only_x():
    n = 13
    rng = np.random.default_rng(4)
    psi0 = ogates.random_state(n, rng)
    for prog in (
        [{"kind": "custom", "qubits": (q,), "matrix": ogates.rz(0.1 + q)} for q in range(n)],
        [{"kind": "custom", "qubits": (q % n,), "matrix": X} for q in range(2 * n + 1)],
        [{"kind": "custom", "qubits": (5,), "matrix": H}] * 7,
    ):
        got, _ = run_queue(n, prog, [], psi0, FACT)
        assert max_dev(got, ocirc.run(n, prog, psi0)) <= TOL


def test_factored_long_program_rescales():
    """1400 Hadamards: the shear scales multiply to 2^-700, beyond the 2^-600
    guard, so the rewrite inserts scalar passes; the state stays normal."""
    n = 12
    rng = np.random.default_rng(5)
    psi0 = ogates.random_state(n, rng)
    prog = [{"kind": "custom", "qubits": (int(q),), "matrix": H}
            for q in rng.integers(0, n, size=1400)]
    got, _ = run_queue(n, prog, [], psi0, FACT)
    assert max_dev(got, ocirc.run(n, prog, psi0)) <= TOL


KINDS = {0: "h", 1: "rx", 2: "rz", 3: "cx"}


def decode(arr):
    from paper_2001_10554_b200.circuit import GateSpec
    out = []
    for kind, q0, q1, param in arr:
        k = KINDS[int(kind)]
        if k == "cx":
            out.append(GateSpec("cx", (int(q0), int(q1))))
        elif k == "h":
            out.append(GateSpec("h", (int(q0),)))
        else:
            out.append(GateSpec(k, (int(q0),), float(param)))
    return out


@pytest.mark.parametrize("ranks", [1, 2, 4])
def test_factored_config1_n12_golden(ranks):
    g = golden("golden_cfg1_n12.npz")
    circ = Circuit(12, tuple(decode(g["gates"])))
    psi = runtime.simulate_circuit(circ, num_ranks=ranks, fuse=FACT)
    assert max_dev(psi, g["state"]) <= TOL


def test_factored_config1_n20_golden():
    g = golden("golden_cfg1_n20.npz")
    circ = Circuit(20, tuple(decode(g["gates"])))
    ctx = runtime.make_context(None, 20, fuse=FACT)
    runtime.run_circuit(ctx, circ)
    psi = ctx.state.download()
    assert max_dev(psi[g["sample_idx"]], g["sample"]) <= TOL
    probs = [runtime.measure_probability(ctx, q) for q in range(20)]
    np.testing.assert_allclose(probs, g["probs"], rtol=RTOL_OBS, atol=0)


def test_factored_qaoa_pool_matches_reference():
    """Config 5 through the pool: per-state RX tables stay exact, the shared
    Hadamard layer is factored, the cut phases commute with its diagonals."""
    g = golden("golden_cfg5.npz")
    graph = make_graph(20, g["edges"])
    depth = 4
    circ = build_qaoa_circuit(graph, depth)
    params = g["params"]
    S = len(params)
    tables = {}
    for s in range(S):
        for name, v in qaoa_bindings(depth, params[s]).items():
            tables.setdefault(name, np.empty(S))[s] = v
    ctx = runtime.make_context(None, 20, num_states=S, fuse=FACT)
    runtime.run_circuit_pool(ctx, circ, tables)
    values = runtime.measure_maxcut(ctx, graph)
    np.testing.assert_allclose(values, g["values"], rtol=RTOL_OBS, atol=0)


@pytest.mark.slow
def test_factored_n26_sweep_vs_oracle_and_n28_roundtrip():
    # n=26: two config-2 sweeps (every qubit, fused passes) in both numerics
    # against the CPU oracle over the same 52 gates: exact bit-equal,
    # factored within 1e-12
    from oracle import cpu_baseline
    n = 26
    rng = np.random.default_rng(9)
    us = [ogates.random_unitary_2x2(rng) for _ in range(n)]

    def fresh(seed):
        st = N.DeviceState(n, n)
        N.call("qs_init_gaussian", st.handle, seed)
        norm = st.observable(N.QS_OBS_NORM)[0]
        N.call("qs_scale", st.handle, 1.0 / np.sqrt(norm))
        return st

    expect = fresh(11).download()
    for _ in range(2):
        for k in range(n):
            cpu_baseline.apply_1q_threaded(expect, k, us[k])
    for fuse in (True, FACT):
        st = fresh(11)
        q = runtime.GateQueue(st, fuse=fuse)
        for _ in range(2):
            for k in range(n):
                q.one_qubit(k, us[k])
        q.flush()
        got = st.download()
        del st
        if fuse is True:
            assert bits_equal(got, expect)
        else:
            assert max_dev(got, expect) <= TOL
            assert not bits_equal(got, expect)
    del expect
    # n=28: forward sweep then the adjoint sweep backward returns the start
    n = 28
    st = N.DeviceState(n, n)
    N.call("qs_init_gaussian", st.handle, 12)
    norm = st.observable(N.QS_OBS_NORM)[0]
    N.call("qs_scale", st.handle, 1.0 / np.sqrt(norm))
    start = st.download()
    us = [ogates.random_unitary_2x2(rng) for _ in range(n)]
    q = runtime.GateQueue(st, fuse=FACT)
    for k in range(n):
        q.one_qubit(k, us[k])
    q.flush()
    mid = st.observable(N.QS_OBS_NORM)[0]
    for k in reversed(range(n)):
        q.one_qubit(k, us[k].conj().T)
    q.flush()
    back = st.download()
    assert abs(mid - 1.0) < 1e-10
    assert max_dev(back, start) <= TOL


def test_state_diff_matches_host():
    """qs_state_diff (the bench's numerics_error) against numpy."""
    n = 14
    rng = np.random.default_rng(5)
    a, b = ogates.random_state(n, rng), ogates.random_state(n, rng)
    sa, sb = N.DeviceState(n, n), N.DeviceState(n, n)
    sa.upload(a)
    sb.upload(b)
    d = sa.diff(sb)
    assert d["max_abs"] == pytest.approx(float(np.max(np.abs(a - b))), rel=1e-14)
    assert d["rel_l2"] == pytest.approx(float(np.linalg.norm(a - b) / np.linalg.norm(b)),
                                        rel=1e-12)
    assert d["ref_max"] == pytest.approx(float(np.max(np.abs(b))), rel=1e-14)


def test_factored_pool_per_state_gates():
    """Per-state matrices in pool mode: RX(theta_s) factors with the same
    diagonals for every state (per-state shears + per-state scalars), per-state
    Haar matrices do not (they stay exact); shared gates and cut phases mix in."""
    from oracle import statevector as osv
    rng = np.random.default_rng(8)
    n, S = 13, 6
    edges = [(0, 3), (2, 7), (5, 11), (1, 12)]
    graph = make_graph(n, edges)
    states = np.stack([ogates.random_state(n, rng) for _ in range(S)])
    pool = runtime.PoolState(n, S, fuse=FACT)
    pool.state.upload(states)
    expected = states.copy()
    for step in range(40):
        q = int(rng.integers(n))
        r = rng.random()
        if r < 0.45:
            us = np.stack([ogates.rx(float(x)) for x in rng.uniform(0, 2 * np.pi, S)])
        elif r < 0.6:
            us = np.stack([ogates.random_unitary_2x2(rng) for _ in range(S)])
        elif r < 0.85:
            us = np.stack([ogates.random_unitary_2x2(rng)] * S)
        else:
            gam = rng.uniform(0, np.pi, S)
            pool.queue.cut_phase(graph, gam)
            for s in range(S):
                osv.apply_cut_phase(expected[s], edges, float(gam[s]))
            continue
        pool.queue.one_qubit(q, us)
        for s in range(S):
            osv.apply_1q(expected[s], q, us[s])
    # nearly anti-diagonal states (t = tan(theta/2) up to ~1e8): large shears
    for q in (0, 7, 12):
        th = np.array([np.pi - 1e-7, 0.3, np.pi + 2e-8, 2.0, np.pi - 3e-9, 5.9])
        us = np.stack([ogates.rx(float(x)) for x in th])
        pool.queue.one_qubit(q, us)
        for s in range(S):
            osv.apply_1q(expected[s], q, us[s])
    got = pool.amplitudes()
    assert max_dev(got, expected) <= TOL


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("remap", [False, True])
@pytest.mark.parametrize("large", [False, True])
def test_factored_config4_distributed(P, remap, large, monkeypatch):
    """Config 4 recipe at n=14 over 2/4 emulated ranks (m = 13/12, so the local
    programs are factored): local shears, global-qubit exchanges (or qubit
    remapping) and case-(c) CNOTs, against the oracle's full state.  `large`:
    the schedule of large states (lean-first passes, batched diagonal flush,
    CNOT passes on k_perm) forced at n=16 (m = 15/14)."""
    from paper_2001_10554_b200.circuit import GateSpec
    n = 16 if large else 14
    if large:
        monkeypatch.setenv("QSB_LEAN_FIRST_M", "12")
    rng = np.random.default_rng(40 + P)
    psi0 = ogates.random_state(n, rng)
    seq, prog = [], []
    for layer in range(3):
        for q in range(n):
            u = ogates.random_unitary_2x2(rng)
            seq.append(GateSpec("custom", (q,), matrix=u))
            prog.append({"kind": "custom", "qubits": (q,), "matrix": u})
        for q in range(n // 2):
            seq.append(GateSpec("cx", (q, n - 1 - q)))
            prog.append({"kind": "cx", "qubits": (q, n - 1 - q)})
    circ = Circuit(n, tuple(seq))
    expect = ocirc.run(n, prog, psi0)

    def rank_fn(comm):
        ctx = runtime.make_context(comm, n, 1, 0, fuse=FACT, remap=remap)
        m = ctx.topology.num_local_qubits
        ctx.partition.amplitudes = psi0[comm.rank << m:(comm.rank + 1) << m]
        ctx.norm_check_interval = 0
        runtime.run_circuit(ctx, circ)
        return runtime.gather_group_state(ctx)

    out = runtime.run_spmd(P, rank_fn, timeout=120.0)[0]
    assert max_dev(out, expect) <= TOL


def test_factored_pool_per_state_rescaling():
    """25 per-state shears with c ~ 2e-9 (t ~ 5e8): the per-state scales pass
    2^-600, so the rewrite inserts per-state scalar ops mid-program (and the
    amplitudes, grown by up to 5e8 per shear, stay finite)."""
    from oracle import statevector as osv
    rng = np.random.default_rng(21)
    n, S = 12, 3
    states = np.stack([ogates.random_state(n, rng) for _ in range(S)])
    pool = runtime.PoolState(n, S, fuse=FACT)
    pool.state.upload(states)
    expected = states.copy()
    for k in range(25):
        q = k % n
        th = np.array([np.pi - 4e-9, np.pi + 4e-9, 1.0 + k])
        us = np.stack([ogates.rx(float(x)) for x in th])
        pool.queue.one_qubit(q, us)
        for s in range(S):
            osv.apply_1q(expected[s], q, us[s])
    got = pool.amplitudes()
    assert np.all(np.isfinite(got))
    assert max_dev(got, expected) <= TOL


def test_factored_pool_per_state_diagonals_noise_like():
    """Per-state gates whose diagonals differ between states (noise-trajectory
    rotations rz.ry.rx with random angles) interleaved with shared and per-state
    RX gates and cut phases: per-state pre-diagonals and pending diagonals."""
    from oracle import statevector as osv
    rng = np.random.default_rng(31)
    n, S = 13, 5
    edges = [(0, 4), (3, 9), (6, 12), (2, 11)]
    graph = make_graph(n, edges)
    states = np.stack([ogates.random_state(n, rng) for _ in range(S)])
    pool = runtime.PoolState(n, S, fuse=FACT)
    pool.state.upload(states)
    expected = states.copy()
    for step in range(60):
        q = int(rng.integers(n))
        r = rng.random()
        if r < 0.4:
            us = np.stack([ogates.rz(a) @ ogates.ry(b) @ ogates.rx(c)
                           for a, b, c in rng.uniform(0, 0.3, size=(S, 3))])
        elif r < 0.6:
            us = np.stack([ogates.rx(float(x)) for x in rng.uniform(0, 2 * np.pi, S)])
        elif r < 0.8:
            us = np.stack([ogates.random_unitary_2x2(rng)] * S)
        elif r < 0.9:
            us = np.stack([ogates.rz(float(rng.uniform(0, 6)))] * S)
        else:
            gam = rng.uniform(0, np.pi, S)
            pool.queue.cut_phase(graph, gam)
            for s in range(S):
                osv.apply_cut_phase(expected[s], edges, float(gam[s]))
            continue
        shared = all(np.array_equal(us[0], u) for u in us)
        pool.queue.one_qubit(q, us[0] if shared else us)
        for s in range(S):
            osv.apply_1q(expected[s], q, us[s])
    got = pool.amplitudes()
    assert max_dev(got, expected) <= TOL


def test_factored_pool_per_state_diagonal_gates():
    """Per-state gates that are diagonal for every state (per-state RZ(gamma_s)
    between CNOTs, pure dephasing, fused products that come out diagonal) fold
    into the per-state pending diagonals and scalars; none may be dropped
    (CNOT, per-state RZ, CNOT + 10 H lost the RZ)."""
    from oracle import statevector as osv
    rng = np.random.default_rng(41)
    n, S = 12, 4
    states = np.stack([ogates.random_state(n, rng) for _ in range(S)])
    cx = X
    # the advisor's harness: CNOT, per-state RZ, CNOT, then 10 Hadamards
    pool = runtime.PoolState(n, S, fuse=FACT)
    pool.state.upload(states)
    expected = states.copy()
    pool.queue.controlled(0, 1, cx)
    rz = np.stack([ogates.rz(float(g)) for g in rng.uniform(0, 2 * np.pi, S)])
    pool.queue.one_qubit(1, rz)
    pool.queue.controlled(0, 1, cx)
    for q in range(2, 12):
        pool.queue.one_qubit(q, H)
    for s in range(S):
        osv.apply_controlled(expected[s], 0, 1, cx)
        osv.apply_1q(expected[s], 1, rz[s])
        osv.apply_controlled(expected[s], 0, 1, cx)
        for q in range(2, 12):
            osv.apply_1q(expected[s], q, H)
    got = pool.amplitudes()
    assert max_dev(got, expected) <= TOL
    # random mix with per-state diagonals everywhere (and a per-state product
    # noise . T . noise that comes out diagonal)
    pool = runtime.PoolState(n, S, fuse=FACT)
    pool.state.upload(states)
    expected = states.copy()
    T = np.diag([1.0, np.exp(0.25j * np.pi)]).astype(np.complex128)
    for step in range(80):
        q = int(rng.integers(n))
        r = rng.random()
        if r < 0.3:
            us = np.stack([ogates.rz(float(a)) for a in rng.uniform(0, 2 * np.pi, S)])
        elif r < 0.4:
            a = rng.uniform(0, 1, S)
            us = np.stack([ogates.rz(float(x)) @ T @ ogates.rz(float(-2 * x)) for x in a])
        elif r < 0.6:
            us = np.stack([ogates.rx(float(x)) for x in rng.uniform(0, 2 * np.pi, S)])
        elif r < 0.75:
            us = np.stack([ogates.random_unitary_2x2(rng)] * S)
        else:
            t = int(rng.integers(n - 1))
            t = t if t < q else t + 1
            pool.queue.controlled(q, t, cx)
            for s in range(S):
                osv.apply_controlled(expected[s], q, t, cx)
            continue
        pool.queue.one_qubit(q, us)
        for s in range(S):
            osv.apply_1q(expected[s], q, us[s])
    got = pool.amplitudes()
    assert max_dev(got, expected) <= TOL


def test_factored_pool_two_rescales_keep_their_place():
    """Two or more mid-program per-state rescales under the default re-order:
    each must stay between the shears around it (pulled to the
    front, their product underflowed the state to zero)."""
    from oracle import statevector as osv
    rng = np.random.default_rng(43)
    n, S = 16, 2
    states = np.stack([ogates.random_state(n, rng) for _ in range(S)])
    pool = runtime.PoolState(n, S, fuse=FACT)
    pool.state.upload(states)
    expected = states.copy()
    for layer in range(8):
        for q in range(n):
            th = np.array([np.pi - 3e-9, np.pi + 5e-9]) + 1e-10 * layer
            us = np.stack([ogates.rx(float(x)) for x in th])
            pool.queue.one_qubit(q, us)
            for s in range(S):
                osv.apply_1q(expected[s], q, us[s])
    got = pool.amplitudes()
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got)) > 1e-6
    assert max_dev(got, expected) <= TOL


def test_factored_lean_first_schedule(monkeypatch):
    """Large states keep passes of lean kinds (shears, product diagonals, cut
    phases) free of controlled gates, which would move the whole pass to k_tile
    (QSB_LEAN_FIRST_M lowers the m >= 24 threshold for this test): same results
    within tolerance as the mixed schedule, on config-4-like layers and random
    mixed programs."""
    rng = np.random.default_rng(4242)
    n = 14
    progs = []
    layer = [{"kind": "custom", "qubits": (q,), "matrix": ogates.random_unitary_2x2(rng)}
             for q in range(n)]
    layer += [{"kind": "cu", "qubits": (q, n - 1 - q), "matrix": X} for q in range(n // 2)]
    layer2 = [{"kind": "custom", "qubits": (q,), "matrix": ogates.random_unitary_2x2(rng)}
              for q in range(n)]
    progs.append((layer + layer2 + layer, [(0, 3)]))
    progs.append(mixed_program(n, 120, rng))
    for prog, edges in progs:
        psi0 = ogates.random_state(n, rng)
        expect = ocirc.run(n, prog, psi0)
        monkeypatch.setenv("QSB_LEAN_FIRST_M", "12")
        got, passes_lean = run_queue(n, prog, edges, psi0, FACT)
        assert max_dev(got, expect) <= TOL
        monkeypatch.setenv("QSB_LEAN_FIRST_M", "99")
        got2, passes_mixed = run_queue(n, prog, edges, psi0, FACT)
        assert max_dev(got2, expect) <= TOL
        assert passes_lean >= passes_mixed


@pytest.mark.parametrize("n", [14, 16, 19])
def test_factored_cnot_passes_run_as_permutations(n, monkeypatch):
    """A pass of CNOTs only in a factored program is one gather per
    2^13-amplitude box (k_perm, launch kind 9): chains, repeated targets,
    targets among qubits 0..3, controls inside and outside the box, several
    layers -- against the oracle."""
    monkeypatch.setenv("QSB_LEAN_FIRST_M", "12")
    rng = np.random.default_rng(900 + n)
    prog = []
    for layer in range(3):
        prog += [{"kind": "custom", "qubits": (q,), "matrix": ogates.random_unitary_2x2(rng)}
                 for q in range(n)]
        if layer == 0:    # config 4's pairs
            pairs = [(q, n - 1 - q) for q in range(n // 2)]
        elif layer == 1:  # a chain through low and high qubits, a repeated target
            pairs = [(0, 5), (5, n - 1), (n - 1, 2), (2, n - 2), (7, n - 2), (n - 3, 1), (1, 9)]
        else:
            pairs = []
            while len(pairs) < 12:
                c, t = (int(x) for x in rng.integers(0, n, size=2))
                if c != t:
                    pairs.append((c, t))
        prog += [{"kind": "cu", "qubits": p, "matrix": X} for p in pairs]
    psi0 = ogates.random_state(n, rng)
    expect = ocirc.run(n, prog, psi0)
    st = N.DeviceState(n, n)
    st.upload(psi0)
    st.launch_log(True)
    q = runtime.GateQueue(st, fuse=FACT)
    for g in prog:
        if g["kind"] == "custom":
            q.one_qubit(g["qubits"][0], g["matrix"])
        else:
            q.controlled(*g["qubits"], g["matrix"])
    q.flush()
    got = st.download()
    st.launch_log(False)
    _, kinds = st.read_launch_log()
    assert 9 in set(int(k) for k in kinds), kinds
    assert max_dev(got, expect) <= TOL


def test_factored_cnot_only_program_is_a_permutation():
    """A program of CNOTs alone (the local CNOTs of a distributed layer between
    two exchanges) counts as factored and runs on k_perm: bit-identical to the
    oracle on a state without zeros (a permutation moves the bits unchanged)."""
    n = 15
    rng = np.random.default_rng(77)
    psi0 = ogates.random_state(n, rng)
    pairs = [(q, n - 1 - q) for q in range(n // 2)] + [(3, 1), (n - 1, 0), (6, 2)]
    prog = [{"kind": "cu", "qubits": p, "matrix": X} for p in pairs]
    expect = ocirc.run(n, prog, psi0)
    st = N.DeviceState(n, n)
    st.upload(psi0)
    st.launch_log(True)
    q = runtime.GateQueue(st, fuse=FACT)
    for g in prog:
        q.controlled(*g["qubits"], g["matrix"])
    q.flush()
    got = st.download()
    st.launch_log(False)
    _, kinds = st.read_launch_log()
    assert set(int(k) for k in kinds) == {9}, kinds
    assert bits_equal(got, expect)


@pytest.mark.parametrize("n", [13, 16])
def test_factored_controlled_gates_on_one_pair_fuse(n):
    """Consecutive controlled gates on one (control, target) pair -- config 3's
    CNOT, CPhase(phi), controlled-Haar per pair -- become one controlled gate
    with the product matrix in the factored mode; triples, interrupted triples
    (a gate on the control or the target in between), reversed pairs and
    per-state matrices in a pool, against the oracle."""
    from oracle import statevector as osv
    rng = np.random.default_rng(3100 + n)
    prog = []
    for k in range(40):
        c, t = (int(x) for x in rng.choice(n, 2, replace=False))
        phi = float(rng.uniform(0, 2 * np.pi))
        cp = np.diag([1.0, np.exp(1j * phi)]).astype(np.complex128)
        triple = [X, cp, ogates.random_unitary_2x2(rng)]
        for j, u in enumerate(triple):
            prog.append({"kind": "cu", "qubits": (c, t), "matrix": u})
            r = rng.random()
            if j < 2 and r < 0.15:    # a 1q gate on the target breaks the run
                prog.append({"kind": "custom", "qubits": (t,), "matrix": ogates.random_unitary_2x2(rng)})
            elif j < 2 and r < 0.3:   # ... or one on the control
                prog.append({"kind": "custom", "qubits": (c,), "matrix": ogates.rz(0.3 + k)})
            elif j < 2 and r < 0.4:   # ... or the reversed pair
                prog.append({"kind": "cu", "qubits": (t, c), "matrix": X})
        if k % 5 == 0:
            prog.append({"kind": "custom", "qubits": (int(rng.integers(n)),), "matrix": H})
    psi0 = ogates.random_state(n, rng)
    expect = ocirc.run(n, prog, psi0)
    got, passes = run_queue(n, prog, [(0, 1)], psi0, FACT)
    assert max_dev(got, expect) <= TOL
    # a pool with per-state controlled matrices in the middle of a triple
    S = 3
    states = np.stack([ogates.random_state(n, rng) for _ in range(S)])
    pool = runtime.PoolState(n, S, fuse=FACT)
    pool.state.upload(states)
    expected = states.copy()
    for k in range(12):
        c, t = (int(x) for x in rng.choice(n, 2, replace=False))
        us = [X, np.stack([ogates.random_unitary_2x2(rng) for _ in range(S)]),
              np.diag([1.0, np.exp(1j * (0.7 + k))]).astype(np.complex128)]
        for u in us:
            pool.queue.controlled(c, t, u)
            for s in range(S):
                osv.apply_controlled(expected[s], c, t, u[s] if u.ndim == 3 else u)
        q = int(rng.integers(n))
        pool.queue.one_qubit(q, H)
        for s in range(S):
            osv.apply_1q(expected[s], q, H)
    assert max_dev(pool.amplitudes(), expected) <= TOL
