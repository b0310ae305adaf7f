"""GPU parity: the CUDA path through the C ABI vs the reference's own outputs
(golden fixtures made by tests/golden/make_golden.py) and vs the oracle.

The contract (BASELINE north_star): max |d amplitude| <= 1e-12 and
expectation values within 1e-10 relative.  Because the kernels spell out
numpy's complex arithmetic (FMA recipe) and the reductions
follow tree_sum's association, the results are expected to be bit-identical,
and most tests assert exactly that on top of the tolerance.
"""
import hashlib

import numpy as np
import pytest

import paper_2001_10554_b200 as qs
from paper_2001_10554_b200 import distribution as dist
from paper_2001_10554_b200 import runtime, statevector as sv
from paper_2001_10554_b200.circuit import Circuit, GateSpec, build_qaoa_circuit, qaoa_bindings
from paper_2001_10554_b200.graphs import make_graph

from conftest import bits_equal, golden, max_dev

from oracle import circuit as ocirc
from oracle import gates as ogates
from oracle import statevector as osv

pytestmark = pytest.mark.gpu
TOL = 1e-12      # amplitudes, absolute (north_star)
RTOL_OBS = 1e-10  # expectation values, relative (north_star)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.complex128).tobytes()).hexdigest()


def test_device_present():
    assert qs.device_count() >= 1, "no CUDA device: the B200 core has no CPU fallback"


# ---- local kernels vs the reference's own outputs --------------------------------------
def test_one_qubit_every_target_bit_exact():
    g = golden("golden_1q.npz")
    n = 10
    for q in range(n):
        p = sv.StatePartition(n, n, 0, g["psi0"].copy())
        sv.apply_local_one_qubit_gate(p, q, g["us"][q])
        assert max_dev(p.amplitudes, g["outs"][q]) <= TOL
        assert bits_equal(p.amplitudes, g["outs"][q]), f"q={q} not bit-exact"


def test_one_qubit_chain_bit_exact():
    g = golden("golden_1q.npz")
    p = sv.StatePartition(10, 10, 0, g["psi0"].copy())
    for q, u in zip(g["chain_q"], g["chain_u"]):
        sv.apply_local_one_qubit_gate(p, int(q), u)
    assert bits_equal(p.amplitudes, g["chain_out"])


def test_controlled_cnot_cphase_cu_bit_exact():
    g = golden("golden_ctrl.npz")
    for (c, t), u, out in zip(g["pairs"], g["mats"], g["outs"]):
        p = sv.StatePartition(10, 10, 0, g["psi0"].copy())
        sv.apply_local_controlled_gate(p, int(c), int(t), u)
        assert max_dev(p.amplitudes, out) <= TOL
        assert bits_equal(p.amplitudes, out), f"controlled ({c},{t}) not bit-exact"


def test_cut_phase_bit_exact():
    g = golden("golden_phase_obs.npz")
    graph = make_graph(10, g["edges"])
    for gamma, out in zip(g["gammas"], g["outs"]):
        p = sv.StatePartition(10, 10, 0, g["psi0"].copy())
        sv.apply_diagonal_phase(p, sv.CutPhase(graph, gamma))
        assert bits_equal(p.amplitudes, out)


def test_observables_tree_order_exact():
    g = golden("golden_phase_obs.npz")
    graph = make_graph(10, g["edges"])
    for k, s in enumerate(g["states"]):
        p = sv.StatePartition(10, 10, 0, s.copy())
        assert sv.norm_squared(p) == g["norm"][k]
        assert sv.maxcut_expectation(p, graph) == g["cut"][k]
        for q in range(10):
            assert sv.get_probability(p, q) == g["prob"][k][q]
            assert sv.z_expectation(p, q) == g["z"][k][q]
    # per-rank partials of a 4-way split (m = 8) and their group reduction
    s0 = g["states"][0]
    for r in range(4):
        p = sv.StatePartition(10, 8, r, s0[r << 8:(r + 1) << 8].copy())
        assert sv.norm_squared(p) == g["part_norm"][r]
        assert sv.maxcut_expectation(p, graph) == g["part_cut"][r]
        for q in range(10):
            assert sv.get_probability(p, q) == g["part_prob"][r][q]
            assert sv.z_expectation(p, q) == g["part_z"][r][q]
    assert sv.tree_sum(g["part_norm"]) == g["norm"][0]


# ---- configs --------------------------------------------------------------------------
KINDS = {0: "h", 1: "rx", 2: "rz", 3: "cx"}


def decode(arr):
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


@pytest.mark.parametrize("fuse", [False, True])
def test_config1_n12_full_state(fuse):
    g = golden("golden_cfg1_n12.npz")
    circ = Circuit(12, tuple(decode(g["gates"])))
    psi = runtime.simulate_circuit(circ, num_ranks=1, fuse=fuse)
    assert max_dev(psi, g["state"]) <= TOL
    assert bits_equal(psi, g["state"])


@pytest.mark.parametrize("fuse", [False, True])
def test_config1_n20_reference_hash(fuse):
    g = golden("golden_cfg1_n20.npz")
    circ = Circuit(20, tuple(decode(g["gates"])))
    ctx = runtime.make_context(None, 20, fuse=fuse)
    runtime.run_circuit(ctx, circ)
    psi = ctx.state.download()
    assert max_dev(psi[g["sample_idx"]], g["sample"]) <= TOL
    probs = [runtime.measure_probability(ctx, q) for q in range(20)]
    np.testing.assert_allclose(probs, g["probs"], rtol=RTOL_OBS, atol=0)
    assert sha(psi) == str(g["sha"]), "config-1 state differs from the reference bit pattern"
    assert probs == list(g["probs"])


@pytest.mark.parametrize("ranks", [1, 2, 4])
def test_config1_n12_distributed_emulated(ranks):
    g = golden("golden_cfg1_n12.npz")
    circ = Circuit(12, tuple(decode(g["gates"])))
    psi = runtime.simulate_circuit(circ, num_ranks=ranks)
    assert bits_equal(psi, g["state"])


def test_config3_controlled_sequence():
    g = golden("golden_cfg3_n12.npz")
    p = sv.StatePartition(12, 12, 0, g["psi0"].copy())
    for (c, t), u in zip(g["pairs"], g["mats"]):
        sv.apply_local_controlled_gate(p, int(c), int(t), u)
    assert max_dev(p.amplitudes, g["out"]) <= TOL
    assert bits_equal(p.amplitudes, g["out"])


@pytest.mark.parametrize("p", [0, 1, 2, 3])
@pytest.mark.parametrize("mode", ["fused", "gatewise"])
def test_config4_emulated_ranks(p, mode):
    """Config 4 recipe at m=10 over P=2^p emulated ranks on one GPU: local
    gates, global-qubit exchanges (peer kernel) and case-(c) CNOTs."""
    g = golden("golden_cfg4_m10.npz")
    P, n = 1 << p, 10 + p
    psi0, us, ref = g[f"psi0_p{p}"], g[f"us_p{p}"], g[f"out_p{p}"]
    seq = []
    k = 0
    for layer in range(4):
        for q in range(n):
            seq.append(GateSpec("custom", (q,), matrix=us[k]))
            k += 1
        for q in range(n // 2):
            seq.append(GateSpec("cx", (q, n - 1 - q)))
    circ = Circuit(n, tuple(seq))

    def rank_fn(comm):
        ctx = runtime.make_context(comm, n, 1, 0, fuse=(mode == "fused"))
        m = ctx.topology.num_local_qubits
        ctx.partition.amplitudes = psi0[comm.rank << m:(comm.rank + 1) << m]
        ctx.norm_check_interval = 0
        runtime.run_circuit(ctx, circ)
        return ctx.state.download(), ctx.state.counters()

    res = runtime.run_spmd(P, rank_fn, timeout=120.0)
    out = np.concatenate([r[0] for r in res])
    assert max_dev(out, ref) <= TOL
    assert bits_equal(out, ref)
    for r, (msgs, amps) in enumerate(x[1] for x in res):
        assert msgs == 0 if P == 1 else msgs > 0


def test_exchange_accounting_matches_reference():
    """Reference criterion 2: n=12, p=2 -- local gates move nothing, each global
    gate is 2 messages and 2*16*2^9 bytes per rank."""
    import json
    import os
    from conftest import GOLDEN

    meta = json.load(open(os.path.join(GOLDEN, "golden_accounting.json")))
    ref = golden("golden_accounting_state.npz")
    u = ref["u"]

    def rank_fn(comm):
        ctx = runtime.make_context(comm, 12, 1, 0)
        sv.init_uniform(ctx.partition)
        obs = {}
        for q in range(12):
            before = ctx.state.counters()
            dist.apply_one_qubit_gate(ctx.partition, ctx.topology, comm, q, u)
            after = ctx.state.counters()
            obs[str(q)] = [after[0] - before[0], 16 * (after[1] - before[1])]
        return obs, ctx.state.download()

    res = runtime.run_spmd(4, rank_fn)
    for r, (obs, _) in enumerate(res):
        assert obs == {k: list(v) for k, v in meta["per_rank"][r].items()}
    assert bits_equal(np.concatenate([x[1] for x in res]), ref["out"])


def test_config5_qaoa_pool_matches_reference():
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
    ctx = runtime.make_context(None, 20, num_states=S)
    runtime.run_circuit_pool(ctx, circ, tables)
    values = runtime.measure_maxcut(ctx, graph)
    np.testing.assert_allclose(values, g["values"], rtol=RTOL_OBS, atol=0)
    assert list(values) == list(g["values"])
    amps = ctx.pool.amplitudes()
    for s in range(S):
        assert sha(amps[s]) == str(g["shas"][s])


def test_qaoa_n10_full_states_and_register_api():
    g = golden("golden_cfg5.npz")
    graph = make_graph(10, g["edges10"])
    for pos, st, val in zip(g["params10"], g["states10"], g["values10"]):
        reg = qs.QubitRegister(10)
        for q in range(10):
            reg.ApplyHadamard(q)
        for k in range(2):
            reg.ApplyDiagonalCutPhase(graph, pos[k])
            for q in range(10):
                reg.ApplyRotationX(q, 2.0 * pos[2 + k])
        assert reg.MaxCutExpectation(graph) == val
        assert bits_equal(reg.GetAmplitudes(), st)


# ---- fused planner vs oracle at tile-capable sizes --------------------------------------
def random_program(n, count, rng, with_phase=True):
    edges = [(0, 3), (2, 7), (5, 11), (1, n - 1), (4, 9)]
    out = []
    for _ in range(count):
        r = rng.random()
        if r < 0.6:
            out.append({"kind": "cu" if False else "custom", "qubits": (int(rng.integers(n)),),
                        "matrix": ogates.random_unitary_2x2(rng)})
        elif r < 0.85:
            c = int(rng.integers(n))
            t = int(rng.integers(n - 1))
            t = t if t < c else t + 1
            out.append({"kind": "cu", "qubits": (c, t), "matrix": ogates.random_unitary_2x2(rng)})
        elif with_phase:
            out.append({"kind": "diagcost", "param": float(rng.uniform(0, 6.28)), "edges": edges})
    return out, edges


@pytest.mark.parametrize("n", [12, 14, 17])
def test_fused_program_matches_oracle(n):
    rng = np.random.default_rng(100 + n)
    prog, edges = random_program(n, 80, rng)
    psi0 = ogates.random_state(n, rng)
    expect = ocirc.run(n, prog, psi0)
    graph = make_graph(n, edges)
    for fuse in (True, False):
        st = qs._native.DeviceState(n, n)
        st.upload(psi0)
        q = runtime.GateQueue(st, fuse=fuse)
        for gspec in prog:
            if gspec["kind"] == "custom":
                q.one_qubit(gspec["qubits"][0], gspec["matrix"])
            elif gspec["kind"] == "cu":
                q.controlled(*gspec["qubits"], gspec["matrix"])
            else:
                q.cut_phase(graph, gspec["param"])
        passes = q.flush()
        got = st.download()
        assert max_dev(got, expect) <= TOL
        assert bits_equal(got, expect), f"fuse={fuse} n={n}"
        if fuse:
            assert passes < len(prog)


def test_pool_per_state_matrices_match_independent_runs():
    rng = np.random.default_rng(5)
    n, S = 13, 6
    states = np.stack([ogates.random_state(n, rng) for _ in range(S)])
    pool = runtime.PoolState(n, S)
    pool.state.upload(states)
    expected = states.copy()
    for step in range(25):
        q = int(rng.integers(n))
        us = np.stack([ogates.random_unitary_2x2(rng) for _ in range(S)])
        pool.queue.one_qubit(q, us)
        for s in range(S):
            osv.apply_1q(expected[s], q, us[s])
    got = pool.amplitudes()
    assert bits_equal(got, expected)


# ---- edge cases --------------------------------------------------------------------------
def test_errors_map_to_reference_exceptions():
    p = sv.allocate_partition(4, num_local_qubits=2, rank_index=0)
    with pytest.raises(sv.LocalityError):
        sv.apply_local_one_qubit_gate(p, 2, np.eye(2))
    with pytest.raises(ValueError):
        sv.apply_local_one_qubit_gate(p, -1, np.eye(2))
    with pytest.raises(ValueError):
        sv.apply_local_controlled_gate(p, 1, 1, np.eye(2))
    with pytest.raises(sv.LocalityError):
        sv.apply_local_controlled_gate(p, 0, 3, np.eye(2))
    with pytest.raises(ValueError):
        sv.init_basis_state(p, 16)
    with pytest.raises(ValueError):
        sv.get_probability(p, 4)
    with pytest.raises(ValueError):
        sv.StatePartition(3, 0, 0, None)
    with pytest.raises(ValueError):
        sv.StatePartition(3, 2, 2, None)


def test_known_answers():
    p = sv.init_basis_state(sv.allocate_partition(1), 0)
    sv.apply_local_one_qubit_gate(p, 0, qs.gates.HADAMARD)
    np.testing.assert_allclose(p.amplitudes, [1 / np.sqrt(2)] * 2)
    p = sv.init_basis_state(sv.allocate_partition(4), 0)
    sv.apply_local_one_qubit_gate(p, 1, qs.gates.PAULI_X)
    assert p.amplitudes[2] == 1.0 and np.count_nonzero(p.amplitudes) == 1
    p = sv.init_basis_state(sv.allocate_partition(2), 2)
    sv.apply_local_controlled_gate(p, 1, 0, qs.gates.PAULI_X)
    assert p.amplitudes[3] == 1.0
    p = sv.init_uniform(sv.allocate_partition(3))
    assert np.isclose(sv.maxcut_expectation(p, qs.graphs.triangle()), 1.5)
    p = sv.init_basis_state(sv.allocate_partition(5), 0b00011)
    edges = [(u, v) for u in (0, 1) for v in (2, 3, 4)]
    assert sv.maxcut_expectation(p, make_graph(5, edges)) == 6.0


def test_smallest_states_and_empty_program():
    # n = 1 (single pair), m = 1 distributed over 2 ranks with a global gate
    st = qs._native.DeviceState(1, 1)
    assert st.apply_program([], np.zeros(1)) == 0
    psi0 = np.array([0.6, 0.8j], dtype=np.complex128)
    u = ogates.random_unitary_2x2(np.random.default_rng(1))

    def rank_fn(comm):
        p = sv.StatePartition(2, 1, comm.rank, psi0.copy() if comm.rank == 0 else
                              np.array([0.0, 0.0], dtype=np.complex128))
        comm.attach(p)
        topo = dist.RankTopology(2, 2)
        dist.apply_one_qubit_gate(p, topo, comm, 1, u)
        dist.apply_controlled_gate(p, topo, comm, 0, 1, u)
        return p.amplitudes.copy()

    out = np.concatenate(runtime.run_spmd(2, rank_fn))
    full = np.concatenate([psi0, np.zeros(2, dtype=np.complex128)])
    expect = ocirc.run(2, [{"kind": "custom", "qubits": (1,), "matrix": u},
                           {"kind": "cu", "qubits": (0, 1), "matrix": u}], full, ranks=2)
    assert bits_equal(out, expect)


def test_idle_rank_with_non_power_of_two_world():
    g = golden("golden_cfg1_n12.npz")
    circ = Circuit(12, tuple(decode(g["gates"])))
    psi = runtime.simulate_circuit(circ, num_ranks=3)
    assert bits_equal(psi, g["state"])


def test_mismatched_collective_times_out():
    def rank_fn(comm):
        ctx = runtime.make_context(comm, 3, 1, 0)
        q = 2 if comm.rank == 0 else 0
        dist.apply_one_qubit_gate(ctx.partition, ctx.topology, comm, q, qs.gates.PAULI_X)

    with pytest.raises(RuntimeError) as err:
        runtime.run_spmd(2, rank_fn, timeout=0.5)
    assert isinstance(err.value.__cause__, dist.TransportTimeout)


def test_norm_drift_detected():
    ctx = runtime.make_context(None, 4)
    ctx.norm_check_interval = 10
    bad = GateSpec("custom", (0,), matrix=np.array([[1.1, 0], [0, 1]], dtype=np.complex128))
    with pytest.raises(runtime.NormDriftError):
        for _ in range(10):
            runtime.apply_gate(ctx, bad)


# ---- full-size, size-independent properties ----------------------------------------------
@pytest.mark.slow
def test_n28_sampled_pairs_roundtrip_and_norm():
    n = 28
    st = qs._native.DeviceState(n, n)
    qs._native.call("qs_init_gaussian", st.handle, 7)
    norm = st.observable(qs._native.QS_OBS_NORM)[0]
    qs._native.call("qs_scale", st.handle, 1.0 / np.sqrt(norm))
    psi0 = st.download()
    rng = np.random.default_rng(3)
    # single gates: every output pair depends only on its input pair -> exact sample check
    for q in (0, 1, 4, 13, 27):
        u = ogates.random_unitary_2x2(rng)
        before = st.download()
        st.apply_program([qs._native.QsGate(0, q, -1, 0, 0, 0)], u.view(np.float64).ravel(),
                         fuse=False)
        after = st.download()
        j = rng.integers(0, 1 << (n - 1), size=1 << 20, dtype=np.int64)
        lo = ((j >> q) << (q + 1)) | (j & ((1 << q) - 1))
        hi = lo + (1 << q)
        a, b = osv.pair_update(before[lo], before[hi], u)
        assert bits_equal(after[lo], a) and bits_equal(after[hi], b), f"q={q}"
    # fused sweep forward, then the adjoint sweep backward: identity within 1e-12
    start = st.download()
    us = [ogates.random_unitary_2x2(rng) for _ in range(n)]
    q = runtime.GateQueue(st, fuse=True)
    for k in range(n):
        q.one_qubit(k, us[k])
    q.flush()
    mid_norm = st.observable(qs._native.QS_OBS_NORM)[0]
    for k in reversed(range(n)):
        q.one_qubit(k, us[k].conj().T)
    q.flush()
    back = st.download()
    assert abs(mid_norm - 1.0) < 1e-10
    assert max_dev(back, start) <= TOL
    assert not bits_equal(psi0, after)


@pytest.mark.slow
def test_n30_controlled_gates_properties():
    """Config 3 at full size: sampled control=1 pairs are bit-exact against the
    oracle's pair update, control=0 amplitudes are untouched, CNOT twice and
    CPhase(phi)CPhase(-phi) return the state (CNOT exactly, CPhase to 1e-12)."""
    from paper_2001_10554_b200 import _native as N
    n = 30
    st = N.DeviceState(n, n)
    N.call("qs_init_gaussian", st.handle, 11)
    rng = np.random.default_rng(8)
    cases = [(0, 1), (1, 0), (5, 29), (29, 5), (13, 14)]
    for c, t in cases:
        u = ogates.random_unitary_2x2(rng)
        before = st.download()
        st.apply_program([N.QsGate(1, t, c, 0, 0, 0)], u.view(np.float64).ravel(), fuse=False)
        after = st.download()
        j = rng.integers(0, 1 << (n - 2), size=1 << 18, dtype=np.int64)
        lo_b, hi_b = min(c, t), max(c, t)
        x = ((j >> lo_b) << (lo_b + 1)) | (j & ((1 << lo_b) - 1))
        x = ((x >> hi_b) << (hi_b + 1)) | (x & ((1 << hi_b) - 1))
        lo = x | (1 << c)
        hi = lo | (1 << t)
        a, b = osv.pair_update(before[lo], before[hi], u)
        assert bits_equal(after[lo], a) and bits_equal(after[hi], b), (c, t)
        untouched = x  # control bit 0, target bit 0
        assert bits_equal(after[untouched], before[untouched])
        assert bits_equal(after[untouched | (1 << t)], before[untouched | (1 << t)])
    start = st.download()
    X = qs.gates.PAULI_X.view(np.float64).ravel()
    for _ in range(2):
        st.apply_program([N.QsGate(1, 17, 3, 0, 0, 0)], X, fuse=False)
    assert bits_equal(st.download(), start)
    phi = 1.234
    st.apply_program([N.QsGate(1, 9, 22, 0, 0, 0)], qs.gates.cphase(phi).view(np.float64).ravel(),
                     fuse=False)
    st.apply_program([N.QsGate(1, 9, 22, 0, 0, 0)], qs.gates.cphase(-phi).view(np.float64).ravel(),
                     fuse=False)
    assert max_dev(st.download(), start) <= TOL


@pytest.mark.slow
def test_full_pool_512x20_sample_vs_oracle():
    """Config 5 at full size: 512 pooled n=20 QAOA circuits in one batch; a
    sample of states checked bit for bit against the oracle, all <C> finite."""
    g = golden("golden_cfg5.npz")
    graph = make_graph(20, g["edges"])
    depth, S = 4, 512
    rng = np.random.default_rng(21)
    params = rng.uniform(0, np.pi, size=(S, 2 * depth))
    tables = {}
    for s in range(S):
        for name, v in qaoa_bindings(depth, params[s]).items():
            tables.setdefault(name, np.empty(S))[s] = v
    ctx = runtime.make_context(None, 20, num_states=S)
    runtime.run_circuit_pool(ctx, build_qaoa_circuit(graph, depth), tables)
    values = runtime.measure_maxcut(ctx, graph)
    assert values.shape == (S,) and np.all(np.isfinite(values))
    amps = ctx.pool.amplitudes()
    edges = [tuple(e) for e in g["edges"]]
    for s in (0, 255, 511):
        prog = [{"kind": "h", "qubits": (q,)} for q in range(20)]
        for k in range(depth):
            prog.append({"kind": "diagcost", "param": params[s][k], "edges": edges})
            prog += [{"kind": "rx", "qubits": (q,), "param": 2.0 * params[s][depth + k]}
                     for q in range(20)]
        expect = ocirc.run(20, prog)
        assert bits_equal(amps[s], expect)
        assert values[s] == osv.maxcut_expectation(expect, edges)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_config4_qubit_remapping_bit_exact(p):
    """Qubit remapping (global qubits swapped into local positions, half the
    exchange traffic) reproduces the reference's run_spmd output bit for bit
    once the canonical layout is restored."""
    g = golden("golden_cfg4_m10.npz")
    P, n = 1 << p, 10 + p
    psi0, us, ref = g[f"psi0_p{p}"], g[f"us_p{p}"], g[f"out_p{p}"]
    seq, k = [], 0
    for layer in range(4):
        for q in range(n):
            seq.append(GateSpec("custom", (q,), matrix=us[k]))
            k += 1
        for q in range(n // 2):
            seq.append(GateSpec("cx", (q, n - 1 - q)))
    circ = Circuit(n, tuple(seq))

    def rank_fn(comm):
        ctx = runtime.make_context(comm, n, 1, 0, fuse=True, remap=True)
        m = ctx.topology.num_local_qubits
        ctx.partition.amplitudes = psi0[comm.rank << m:(comm.rank + 1) << m]
        runtime.run_circuit(ctx, circ)
        moved = ctx.state.counters()[1]
        full = runtime.gather_group_state(ctx)
        return full, moved, ctx.qubit_layout.is_identity()

    res = runtime.run_spmd(P, rank_fn, timeout=120.0)
    assert bits_equal(res[0][0], ref)
    assert all(r[2] for r in res)  # layout restored on read


def test_remapped_observables_match_plain():
    g = golden("golden_cfg1_n12.npz")
    circ = Circuit(12, tuple(decode(g["gates"])))
    graph = make_graph(12, [(0, 11), (3, 10), (5, 6)])

    def rank_fn(comm):
        ctx = runtime.make_context(comm, 12, 1, 0, remap=True)
        runtime.run_circuit(ctx, circ)
        probs = [runtime.measure_probability(ctx, q) for q in (0, 9, 10, 11)]
        return probs, runtime.measure_maxcut(ctx, graph), runtime.measure_norm_squared(ctx)

    out = runtime.run_spmd(4, rank_fn)
    psi = g["state"]
    assert out[0][0] == [osv.get_probability(psi, q) for q in (0, 9, 10, 11)]
    assert out[0][1] == osv.maxcut_expectation(psi, graph.edges)
    assert out[0][2] == osv.norm_squared(psi)


@pytest.mark.parametrize("n,m,rank,S", [(20, 20, 0, 1), (14, 12, 3, 1), (13, 13, 0, 5), (10, 10, 0, 2)])
def test_marginals_one_pass_bit_identical(n, m, rank, S):
    from paper_2001_10554_b200 import _native as N
    rng = np.random.default_rng(n + m + rank)
    st = N.DeviceState(n, m, rank, S)
    st.upload(np.concatenate([ogates.random_state(m, rng) for _ in range(S)]))
    marg = st.marginals()
    host = st.download().reshape(S, -1)
    for s in range(S):
        for q in range(n):
            assert marg[s, q] == st.observable(N.QS_OBS_PROB, q)[s]
            assert marg[s, q] == osv.get_probability(host[s], q, n=n, rank=rank)


def test_measure_probabilities_matches_reference_report():
    g = golden("golden_cfg1_n20.npz")
    circ = Circuit(20, tuple(decode(g["gates"])))
    ctx = runtime.make_context(None, 20)
    runtime.run_circuit(ctx, circ)
    assert list(runtime.measure_probabilities(ctx)) == list(g["probs"])

    def rank_fn(comm):
        c = runtime.make_context(comm, 20, 1, 0)
        runtime.run_circuit(c, circ)
        return runtime.measure_probabilities(c)

    out = runtime.run_spmd(4, rank_fn)
    assert list(out[0]) == list(g["probs"])


def test_exchange_amplitudes_full_duplex():
    rng = np.random.default_rng(12)
    n = 16
    a, b = ogates.random_state(n, rng), ogates.random_state(n, rng)
    p = sv.StatePartition(n, n, 0, a.copy())
    out = np.empty_like(a)
    p.state.exchange_host(b, out, chunk=1000)  # ragged last chunk
    assert bits_equal(out, a)
    assert bits_equal(sv.read_amplitudes(p), b)
    sv.exchange_amplitudes(p, a, out)
    assert bits_equal(out, b) and bits_equal(p.amplitudes, a)


@pytest.mark.slow
def test_n33_max_single_gpu_size_layer_roundtrip():
    """Config 4's per-GPU size (2^33 amplitudes, 128 GiB) on one GPU: a
    single gate on the top qubit is bit-exact on sampled pairs; one fused
    config-4 layer (Haar on all 33 qubits + CX(q, 32-q)) keeps the norm and
    its adjoint layer returns sampled blocks to within 1e-12."""
    from paper_2001_10554_b200 import _native as N
    n = 33
    st = N.DeviceState(n, n)
    N.call("qs_init_gaussian", st.handle, 5)
    norm = st.observable(N.QS_OBS_NORM)[0]
    N.call("qs_scale", st.handle, 1.0 / np.sqrt(norm))
    rng = np.random.default_rng(33)
    blk = 1 << 12
    offs = [int(o) * blk for o in rng.integers(0, (1 << (n - 1)) // blk, size=24)]

    def read(offsets):
        return [st.download(offset=o, count=blk).copy() for o in offsets]

    # top qubit: pairs (o + i, o + i + 2^32)
    u = ogates.random_unitary_2x2(rng)
    lo_before, hi_before = read(offs), read([o + (1 << 32) for o in offs])
    st.apply_program([N.QsGate(0, n - 1, -1, 0, 0, 0)], u.view(np.float64).ravel(), fuse=False)
    lo_after, hi_after = read(offs), read([o + (1 << 32) for o in offs])
    for lb, hb, la, ha in zip(lo_before, hi_before, lo_after, hi_after):
        a, b = osv.pair_update(lb, hb, u)
        assert bits_equal(la, a) and bits_equal(ha, b)
    # one config-4 layer and its adjoint
    samples = offs + [o + (1 << 32) for o in offs]
    start = read(samples)
    us = [ogates.random_unitary_2x2(rng) for _ in range(n)]
    X = qs.gates.PAULI_X
    q = runtime.GateQueue(st, fuse=True)
    for k in range(n):
        q.one_qubit(k, us[k])
    for c in range(n // 2):
        q.controlled(c, n - 1 - c, X)
    q.flush()
    assert abs(st.observable(N.QS_OBS_NORM)[0] - 1.0) < 1e-10
    for c in reversed(range(n // 2)):
        q.controlled(c, n - 1 - c, X)
    for k in reversed(range(n)):
        q.one_qubit(k, np.ascontiguousarray(us[k].conj().T))
    q.flush()
    back = read(samples)
    assert max(max_dev(b, s) for b, s in zip(back, start)) <= TOL
    del st
