"""Edge cases of the fused path beyond test_gpu_parity: pools with per-state
tables mixed with controlled gates and cut phases (every tile variant), long
programs that hit the planner's pass/round limits, odd pool sizes, tiles of
exactly one state, graphs without edges -- each bit-exact against the oracle."""
import numpy as np
import pytest

from paper_2001_10554_b200 import _native as N
from paper_2001_10554_b200 import runtime, statevector as sv
from paper_2001_10554_b200.graphs import make_graph, phase_lut

from conftest import bits_equal
from oracle import gates as ogates
from oracle import statevector as osv

pytestmark = pytest.mark.gpu


def oracle_apply(expected, kind, args):
    if kind == "1q":
        q, us = args
        for s in range(expected.shape[0]):
            osv.apply_1q(expected[s], q, us[s])
    elif kind == "ctrl":
        c, t, us = args
        for s in range(expected.shape[0]):
            osv.apply_controlled(expected[s], c, t, us[s])
    else:
        edges, gammas = args
        for s in range(expected.shape[0]):
            osv.apply_cut_phase(expected[s], edges, float(gammas[s]))


@pytest.mark.parametrize("n,S,steps", [(12, 3, 150), (13, 5, 120), (15, 2, 90)])
def test_pool_tables_controls_and_phases(n, S, steps):
    """Per-state matrices and LUTs together with shared ones, controlled gates
    whose control is in registers / elsewhere in the tile / outside it, and cut
    phases: exercises the PHASE/GENERIC/TABLES tile variants on pools whose
    tile count is not a multiple of the grid."""
    rng = np.random.default_rng(7 * n + S)
    edges = [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < 0.25]
    graph = make_graph(n, edges)
    states = np.stack([ogates.random_state(n, rng) for _ in range(S)])
    pool = runtime.PoolState(n, S)
    pool.state.upload(states)
    expected = states.copy()
    for _ in range(steps):
        r = rng.random()
        shared = rng.random() < 0.4
        if r < 0.55:
            q = int(rng.integers(n))
            u = ogates.random_unitary_2x2(rng)
            us = np.stack([u] * S) if shared else np.stack(
                [ogates.random_unitary_2x2(rng) for _ in range(S)])
            pool.queue.one_qubit(q, u if shared else us)
            oracle_apply(expected, "1q", (q, us))
        elif r < 0.85:
            c, t = (int(x) for x in rng.choice(n, size=2, replace=False))
            u = ogates.random_unitary_2x2(rng)
            us = np.stack([u] * S) if shared else np.stack(
                [ogates.random_unitary_2x2(rng) for _ in range(S)])
            pool.queue.controlled(c, t, u if shared else us)
            oracle_apply(expected, "ctrl", (c, t, us))
        else:
            g = float(rng.uniform(0, 6.2))
            gammas = np.full(S, g) if shared else rng.uniform(0, 6.2, size=S)
            pool.queue.cut_phase(graph, g if shared else gammas)
            oracle_apply(expected, "phase", (edges, gammas))
    assert bits_equal(pool.amplitudes(), expected)


def test_long_program_splits_into_passes():
    """300 gates on 12 qubits of one state: the planner must cut passes at
    the 64-gate and round limits; the result stays bit-exact."""
    n = 12
    rng = np.random.default_rng(3)
    psi = ogates.random_state(n, rng)
    st = N.DeviceState(n, n)
    st.upload(psi)
    q = runtime.GateQueue(st, fuse=True)
    exp = psi.copy()
    for _ in range(300):
        t = int(rng.integers(n))
        u = ogates.random_unitary_2x2(rng)
        q.one_qubit(t, u)
        osv.apply_1q(exp, t, u)
    passes = q.flush()
    assert passes >= 300 // 64
    assert bits_equal(st.download(), exp)


def test_graph_without_edges_and_isolated_vertices():
    n = 12
    rng = np.random.default_rng(4)
    psi = ogates.random_state(n, rng)
    p = sv.StatePartition(n, n, 0, psi.copy())
    empty = make_graph(n, [])
    sv.apply_cut_phase(p, empty, 0.7)          # exp(-i*0.7*0) = 1 for every amplitude
    exp = psi.copy()
    osv.apply_cut_phase(exp, [], 0.7)
    assert bits_equal(p.amplitudes, exp)
    assert sv.maxcut_expectation(p, empty) == 0.0
    star = make_graph(n, [(0, 5)])            # vertices other than 0 and 5 isolated
    assert sv.maxcut_expectation(p, star) == osv.maxcut_expectation(p.amplitudes, [(0, 5)])
    assert phase_lut(0.7, 0).shape == (1,)


def test_tile_of_exactly_one_state_and_pool_of_one():
    """m = 12: one tile per state (tiles_per_state = 1), pools of 1 and 7."""
    n = 12
    rng = np.random.default_rng(9)
    for S in (1, 7):
        states = np.stack([ogates.random_state(n, rng) for _ in range(S)])
        pool = runtime.PoolState(n, S) if S > 1 else None
        st = pool.state if pool else N.DeviceState(n, n)
        st.upload(states)
        q = pool.queue if pool else runtime.GateQueue(st)
        exp = states.copy()
        for k in range(40):
            t = int(rng.integers(n))
            u = ogates.random_unitary_2x2(rng)
            q.one_qubit(t, u)
            for s in range(S):
                osv.apply_1q(exp[s], t, u)
        q.flush()
        assert bits_equal(st.download().reshape(S, -1), exp)


def test_apply_gate_pool_binds_state_values():
    """runtime.apply_gate_pool (runtime.py:175-189): state s binds table[s];
    equal to running each binding on its own state."""
    from paper_2001_10554_b200.circuit import GateSpec
    from paper_2001_10554_b200.graphs import make_graph

    n, S = 12, 3
    rng = np.random.default_rng(12)
    graph = make_graph(n, [(0, 3), (3, 7), (7, 11), (2, 5)])
    gates = [GateSpec("h", (q,)) for q in range(n)]
    gates += [GateSpec("diagcost", (), "$g", graph=graph), GateSpec("rx", (4,), "$b"),
              GateSpec("cphase", (1, 9), "$p")]
    tables = {"g": rng.uniform(0, 3, S), "b": rng.uniform(0, 3, S), "p": rng.uniform(0, 3, S)}
    ctx = runtime.make_context(None, n, S)
    for g in gates:
        runtime.apply_gate_pool(ctx, g, None if g.slot is None else tables[g.slot])
    got = ctx.pool.amplitudes()
    for s in range(S):
        one = runtime.make_context(None, n, 1)
        for g in gates:
            runtime.apply_gate(one, g if g.slot is None else
                               GateSpec(g.kind, g.qubits, float(tables[g.slot][s]), graph=g.graph))
        one.flush()
        assert bits_equal(got[s], one.state.download())


def test_oversize_state_fails_loudly():
    """2^36 amplitudes (1 TiB) cannot be allocated: a clean error, and the
    device stays usable."""
    with pytest.raises(Exception) as err:
        N.DeviceState(36, 36)
    assert "memory" in str(err.value).lower() or "alloc" in str(err.value).lower()
    st = N.DeviceState(12, 12)
    N.call("qs_init_basis", st.handle, 5)
    assert st.download()[5] == 1.0


@pytest.mark.parametrize("a,c", [(0, 1), (2, 9), (11, 3), (0, 12)])
def test_swap_qubits_local_is_a_permutation(a, c):
    """qs_swap_qubits_local (remapping's local swap) exchanges qubit a and c
    of every state: the amplitude at i moves to i with bits a and c swapped."""
    n, S = 13, 3
    rng = np.random.default_rng(a * 31 + c)
    states = np.stack([ogates.random_state(n, rng) for _ in range(S)])
    st = N.DeviceState(n, n, 0, S)
    st.upload(states)
    N.call("qs_swap_qubits_local", st.handle, a, c)
    got = st.download().reshape(S, -1)
    idx = np.arange(1 << n)
    ba, bc = (idx >> a) & 1, (idx >> c) & 1
    src = idx ^ ((ba ^ bc) << a) ^ ((ba ^ bc) << c)
    assert bits_equal(got, states[:, src])
