"""The drop-in contract on the device, beyond the reference's own suite
(tests/test_gpu_ref_suite.py): rank-group pools (S states, each sharded over
2^k thread ranks, pool.py:118-128 with runtime.py:64-83), the write-tracking
partition mirror, arbitrary phase callables, the reference's transport
accounting of exchanges, and global-qubit gates queued without host syncs."""
import numpy as np
import pytest

from paper_2001_10554_b200 import runtime
from paper_2001_10554_b200 import statevector as sv
from paper_2001_10554_b200.circuit import Circuit, GateSpec, build_qaoa_circuit, qaoa_bindings
from paper_2001_10554_b200.graphs import make_graph

from conftest import bits_equal, max_dev
from oracle import circuit as ocirc
from oracle import gates as og

pytestmark = pytest.mark.gpu


def _layer_circuit(n, rng, layers=3):
    seq, prog = [], []
    for _ in range(layers):
        for q in range(n):
            u = og.random_unitary_2x2(rng)
            seq.append(GateSpec("custom", (q,), matrix=u))
            prog.append({"kind": "custom", "qubits": (q,), "matrix": u})
        for q in range(n // 2):
            seq.append(GateSpec("cx", (q, n - 1 - q)))
            prog.append({"kind": "cx", "qubits": (q, n - 1 - q)})
    return Circuit(n, tuple(seq)), prog


@pytest.mark.parametrize("world,states", [(4, 2), (8, 2), (8, 4), (6, 2)])
def test_rank_group_pool_states_sharded(world, states):
    """S states, each over world//S ranks (rounded down to a power of two):
    every group's state equals the oracle; per-state QAOA tables bind by group."""
    n = 10
    rng = np.random.default_rng(world * 10 + states)
    circ, prog = _layer_circuit(n, rng)
    expect = ocirc.run(n, prog, np.eye(1 << n, dtype=np.complex128)[0])

    def rank_fn(t):
        ctx = runtime.make_context(t, n, states, seed=3)
        runtime.run_circuit(ctx, circ)
        out = [runtime.gather_group_state(ctx, g) for g in range(states)]
        norms = runtime.pool_sum(ctx, 0.0 if ctx.is_idle else runtime.measure_norm_squared(ctx))
        return out, norms, ctx.layout.ranks_per_state, ctx.is_idle

    res = runtime.run_spmd(world, rank_fn, timeout=120.0)
    out, norms, rps, _ = res[0]
    assert rps == 1 << ((world // states).bit_length() - 1)
    for g in range(states):
        assert bits_equal(out[g], expect), g
    assert all(abs(r[1] - states) < 1e-9 for r in res)
    assert all(r[0] == [None] * states for r in res[1:])


def test_rank_group_pool_qaoa_tables_bind_by_group():
    graph = make_graph(8, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (7, 0)])
    circ = build_qaoa_circuit(graph, 2)
    pos = np.random.default_rng(2).uniform(0, np.pi, size=(4, 4))
    tables = {k: np.array([qaoa_bindings(2, p)[k] for p in pos])
              for k in qaoa_bindings(2, pos[0])}

    def rank_fn(t):
        ctx = runtime.make_context(t, 8, 4, seed=0)   # 8 ranks: 4 groups of 2
        runtime.run_circuit_pool(ctx, circ, tables)
        v = runtime.measure_maxcut(ctx, graph)
        return runtime.pool_gather(ctx, v)

    pooled = runtime.run_spmd(8, rank_fn, timeout=120.0)[0]
    for s in range(4):
        ctx = runtime.make_context(None, 8, 1)
        runtime.run_circuit(ctx, circ, qaoa_bindings(2, pos[s]))
        assert abs(pooled[s] - runtime.measure_maxcut(ctx, graph)) < 1e-12


def test_batched_pool_extension_matches_rank_groups():
    """num_states > world: one batched allocation per rank (shim extension);
    same values as the reference's one-state-per-group layout."""
    graph = make_graph(6, [(0, 1), (1, 2), (2, 0), (3, 4), (4, 5), (5, 3)])
    circ = build_qaoa_circuit(graph, 1)
    pos = np.random.default_rng(4).uniform(0, np.pi, size=(6, 2))
    tables = {k: np.array([qaoa_bindings(1, p)[k] for p in pos]) for k in ("gamma1", "beta1")}

    def batched(t):
        ctx = runtime.make_context(t, 6, 6, seed=0)   # 2 ranks, 3 states each
        assert ctx.num_states == 3
        runtime.run_circuit_pool(ctx, circ, tables)
        v = runtime.measure_maxcut(ctx, graph)
        return runtime.pool_gather(ctx, v), runtime.pool_sum(ctx, v)

    def groups(t):
        ctx = runtime.make_context(t, 6, 6, seed=0)   # 6 ranks, one state each
        runtime.run_circuit_pool(ctx, circ, tables)
        v = runtime.measure_maxcut(ctx, graph)
        return runtime.pool_gather(ctx, v), runtime.pool_sum(ctx, v)

    b = runtime.run_spmd(2, batched, timeout=60.0)
    g = runtime.run_spmd(6, groups, timeout=60.0)
    assert bits_equal(b[0][0], g[0][0])
    assert b[0][1] == b[1][1] == g[0][1]


def test_mirror_read_then_gate_uploads_nothing():
    n = 16
    part = sv.allocate_partition(n)
    sv.init_uniform(part)
    st = part.state
    before = st.uploads
    amps = part.amplitudes          # download, no upload
    _ = float(np.abs(amps).sum())   # reads
    _ = amps[3:9].copy()
    sv.apply_local_one_qubit_gate(part, 3, og.H)
    assert st.uploads == before, "a read forced a re-upload"
    # a write through the mirror (or a view of it) is uploaded exactly once
    a = part.amplitudes
    view = a[:8]
    view[:] = 0.0
    sv.apply_local_one_qubit_gate(part, 0, og.H)
    assert st.uploads == before + (1 << n)
    got = part.amplitudes
    assert np.all(got[:8] == 0.0)
    # in-place operators and ufunc out= count as writes
    ref_norm = 4 * float(np.sum(np.abs(got) ** 2))
    part.amplitudes *= 2.0
    norm = sv.norm_squared(part)
    assert st.uploads == before + 2 * (1 << n)
    assert abs(norm - ref_norm) < 1e-12
    np.multiply(part.amplitudes, 0.5, out=part.amplitudes)
    assert abs(sv.norm_squared(part) - ref_norm / 4) < 1e-12


def test_diagonal_phase_callable_bit_identical_to_reference_expression():
    n = 12
    rng = np.random.default_rng(6)
    psi = og.random_state(n, rng)
    for m, r in ((12, 0), (10, 2)):
        lo = r << m
        part = sv.StatePartition(n, m, r, psi[lo:lo + (1 << m)].copy())
        f = (lambda idx: np.cos(0.37 * np.asarray(idx, dtype=np.float64)) + 0.1)
        sv.apply_diagonal_phase(part, f)
        ref = psi[lo:lo + (1 << m)].copy()
        ref *= np.exp(-1j * f(np.arange(lo, lo + (1 << m), dtype=np.uint64)))
        assert bits_equal(part.amplitudes, ref)


@pytest.mark.parametrize("mode", ["peer", "nccl"])
def test_exchange_accounting_in_reference_terms(mode):
    """TransportCounters after one global gate: 2 messages, 2 * 2^(m-1)
    amplitudes per rank (test_distribution.py:121-135); chunked: 2 per chunk."""
    from paper_2001_10554_b200 import distribution as dist
    n, P = 8, 4
    if mode == "nccl":
        pytest.skip("NCCL self-exchange is covered in test_gpu_nccl.py")

    def body(t):
        topo = dist.RankTopology(P, n)
        comm = dist.GroupComm(t, 0, P)
        part = sv.allocate_partition(n, topo.num_local_qubits, comm.rank)
        sv.init_uniform(part)
        comm.attach(part)
        before = t.counters.snapshot()
        dist.apply_one_qubit_gate(part, topo, comm, n - 1, og.H)
        mid = t.counters.delta(before)
        dist.apply_one_qubit_gate(part, topo, comm, n - 2, og.H, chunk=8)
        return mid, t.counters.delta(before)

    for mid, tot in runtime.run_spmd(P, body, timeout=60.0):
        half = 1 << (n - 2 - 1)
        assert (mid.messages_sent, mid.amplitudes_sent) == (2, 2 * half)
        assert tot.messages_sent == 2 + 2 * (half // 8)


def test_global_gates_queue_without_host_sync():
    """A run of global-qubit gates on 2 emulated ranks returns to the host
    before the GPU is done (the exchange kernels are ordered by CUDA events,
    not by host stream syncs), and the result equals the single-rank run bit
    for bit (P-invariance, test_distribution.py:261-270)."""
    from paper_2001_10554_b200 import _native as N
    n = 28
    rng = np.random.default_rng(8)
    us = [og.random_unitary_2x2(rng) for _ in range(6)]

    def body(t):
        ctx = runtime.make_context(t, n, 1)
        N.call("qs_init_gaussian", ctx.state.handle, 77)  # keyed by global index
        ctx.norm_check_interval = 0
        ctx.state.synchronize()
        for u in us:
            runtime.apply_gate(ctx, GateSpec("custom", (n - 1,), matrix=u))
            runtime.apply_gate(ctx, GateSpec("custom", (3,), matrix=u))
        ctx.queue.flush()
        busy = ctx.state.busy()
        return busy, runtime.gather_group_state(ctx)

    res = runtime.run_spmd(2, body, timeout=300.0)
    assert any(r[0] for r in res), "the host waited for the GPU after the exchanges"
    single = runtime.run_spmd(1, body, timeout=300.0)[0][1]
    assert bits_equal(res[0][1], single)
