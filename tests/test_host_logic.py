"""Host-side logic of the drop-in shim, checked on CPU against the reference's
semantics (routing, topology, pool layout, IR, matrices, phase LUTs)."""
import numpy as np
import pytest

from paper_2001_10554_b200 import circuit, distribution as dist, gates, graphs, pool, runtime
from paper_2001_10554_b200 import statevector as sv
from paper_2001_10554_b200 import workloads

from conftest import bits_equal, golden

from oracle import gates as og


def test_topology_and_index_math():
    topo = dist.RankTopology(5, 6)
    assert topo.effective_ranks == 4 and topo.num_local_qubits == 4
    with pytest.raises(ValueError):
        dist.RankTopology(4, 2)
    assert dist.rank_and_offset(5, dist.RankTopology(2, 3)) == (1, 1)
    assert dist.rank_and_offset(13, dist.RankTopology(4, 4)) == (3, 1)
    t = dist.RankTopology(8, 6)
    for q in range(3, 6):
        for r in range(8):
            p = dist.exchange_partner(r, q, t)
            assert p != r and dist.exchange_partner(p, q, t) == r
    with pytest.raises(ValueError):
        dist.exchange_partner(0, 0, dist.RankTopology(2, 3))


def expected_route(rank, n, m, c, t):
    """The reference's four cases (distribution.py:195-230) restated."""
    if c < m and t < m:
        return "local_controlled"
    if c >= m:
        if not (rank >> (c - m)) & 1:
            return "skip"
        return "local_one_qubit" if t < m else "exchange"
    return "exchange"


@pytest.mark.parametrize("world,n", [(2, 4), (4, 5), (8, 6)])
def test_controlled_routing_all_cases(world, n):
    topo = dist.RankTopology(world, n)
    m = topo.num_local_qubits
    for rank in range(world):
        for c in range(n):
            for t in range(n):
                if c == t:
                    with pytest.raises(ValueError):
                        dist.route_controlled(rank, topo, c, t)
                    continue
                r = dist.route_controlled(rank, topo, c, t)
                assert r[0] == expected_route(rank, n, m, c, t)
                if r[0] == "exchange":
                    d = 1 << (t - m)
                    assert r[1] == rank ^ d and r[2] == ((rank & d) == 0)
                    assert r[3] == (c if c < m else None)
    assert dist.route_controlled(5, dist.RankTopology(6, 5), 0, 4) == ("idle",)


def test_one_qubit_routing():
    topo = dist.RankTopology(4, 5)
    assert dist.route_one_qubit(0, topo, 2) == ("local",)
    assert dist.route_one_qubit(1, topo, 4) == ("exchange", 3, True)
    assert dist.route_one_qubit(3, topo, 3) == ("exchange", 2, False)
    with pytest.raises(ValueError):
        dist.route_one_qubit(0, topo, 5)


def test_tree_sums_match_reference_association():
    g = golden("golden_phase_obs.npz")
    assert sv.tree_sum(g["part_norm"]) == g["norm"][0]
    x = np.random.default_rng(1).standard_normal(13)
    from oracle import statevector as osv
    assert sv.tree_sum_values(x) == osv.tree_sum_values(x)
    assert sv.tree_sum(x[:8]) == osv.tree_sum(x[:8])


def test_pool_layout_worked_examples():
    ten = pool.build_pool(80, 10)
    assert (ten.num_states, ten.ranks_per_state, ten.active_ranks) == (10, 8, 80)
    one = pool.build_pool(80, 1)
    assert (one.ranks_per_state, one.total_ranks - one.active_ranks) == (64, 16)
    three = pool.build_pool(7, 3)
    assert three.ranks_per_state == 2 and three.is_idle(6)
    with pytest.raises(ValueError):
        pool.build_pool(2, 3)


def test_split_pool_is_contiguous_cover():
    for S in (1, 7, 512):
        for world in (1, 2, 3, 8):
            blocks = [runtime.split_pool(S, r, world) for r in range(world)]
            covered = []
            for first, count in blocks:
                covered.extend(range(first, first + count))
            assert covered == list(range(S))


def test_qaoa_ir():
    g = workloads.random_3regular_graph(20, np.random.default_rng(0))
    assert len(g.edges) == 30
    assert all(sum(1 for e in g.edges if v in e) == 3 for v in range(20))
    c = circuit.build_qaoa_circuit(g, 4)
    assert len(c.gates) == 104
    b = circuit.qaoa_bindings(2, [0.1, 0.2, 0.3, 0.4])
    assert b == {"gamma1": 0.1, "beta1": 0.6, "gamma2": 0.2, "beta2": 0.8}
    with pytest.raises(circuit.UnboundParameterError):
        c.require_bound()


def test_config1_recipe_matches_golden_encoding():
    gl = workloads.config1_gates(12, 10, 20260809)
    enc = golden("golden_cfg1_n12.npz")["gates"]
    assert len(gl) == len(enc) == 175
    kinds = {"h": 0, "rx": 1, "rz": 2, "cx": 3}
    for gspec, row in zip(gl, enc):
        assert kinds[gspec.kind] == row[0] and gspec.qubits[0] == row[1]
        if gspec.kind in ("rx", "rz"):
            assert gspec.param == row[3]
    assert len(workloads.config1_gates(20, 10, 1)) == 295


def test_gate_matrices_bit_identical_to_reference_recipe():
    for t in (0.0, 0.3, 1.7, 5.9):
        assert bits_equal(gates.rx(t), og.rx(t))
        assert bits_equal(gates.ry(t), og.ry(t))
        assert bits_equal(gates.rz(t), og.rz(t))
    assert bits_equal(gates.HADAMARD, og.H)
    assert gates.is_unitary(gates.cphase(0.4))
    with pytest.raises(ValueError):
        gates.gate_matrix(np.eye(3))


def test_phase_lut_bits_match_reference_expression():
    gamma = 0.7312
    lut = graphs.phase_lut(gamma, 30)
    cuts = np.arange(31, dtype=np.float64)
    ref = np.exp(-1j * np.asarray(gamma * cuts, dtype=np.float64))
    assert bits_equal(lut, ref)


def test_haar_recipe_matches_reference_oracle():
    a = workloads.haar_2x2(np.random.default_rng(9))
    b = og.random_unitary_2x2(np.random.default_rng(9))
    assert bits_equal(a, b)
    assert gates.is_unitary(a)


class _FakeState:
    num_states = 3


def test_gate_queue_table_layout():
    q = runtime.GateQueue(_FakeState(), fuse=True)
    u = np.stack([og.random_unitary_2x2(np.random.default_rng(i)) for i in range(3)])
    q.one_qubit(4, gates.HADAMARD)
    q.one_qubit(5, u)
    q.controlled(1, 2, gates.PAULI_X)
    g = graphs.make_graph(4, [(0, 1), (2, 3)])
    q.cut_phase(g, [0.1, 0.2, 0.3])
    kinds = [(x.kind, x.target, x.control, x.offset, x.stride) for x in q.gates]
    assert kinds == [(0, 4, -1, 0, 0), (0, 5, -1, 8, 8), (1, 2, 1, 32, 0), (2, 0, -1, 40, 6)]
    mats = np.concatenate(q.tables)
    assert bits_equal(mats[8:32].view(np.complex128).reshape(3, 2, 2), u)
    assert mats.size == 40 + 18


def test_cut_phase_callable_matches_reference_function():
    g = graphs.make_graph(5, [(0, 1), (1, 4), (2, 3)])
    phase = sv.CutPhase(g, 0.37)
    idx = np.arange(32, dtype=np.uint64)
    from oracle import statevector as osv
    assert np.array_equal(phase(idx), 0.37 * osv.cut_counts(g.edges, idx))


def test_batched_matrices_and_luts_bit_identical_to_scalar():
    th = np.random.default_rng(4).uniform(0, 2 * np.pi, 257)
    for kind, fn in (("rx", gates.rx), ("ry", gates.ry), ("rz", gates.rz)):
        assert bits_equal(gates.rotation_batch(kind, th), np.stack([fn(float(t)) for t in th]))
    assert bits_equal(graphs.phase_lut_batch(th, 30),
                      np.stack([graphs.phase_lut(float(t), 30) for t in th]))


def test_drop_in_api_surface():
    """The hot-path names of qpool's modules exist in the shim (reference
    statevector.py, distribution.py, runtime.py, pool.py, gates.py)."""
    import paper_2001_10554_b200 as qs
    expected = {
        "statevector": ["LocalityError", "StatePartition", "allocate_partition",
                        "full_state_bytes", "init_basis_state", "init_uniform", "pair_update",
                        "apply_local_one_qubit_gate", "apply_local_controlled_gate",
                        "apply_diagonal_phase", "norm_squared", "get_probability",
                        "z_expectation", "maxcut_expectation", "tree_sum", "combine_pair",
                        "tree_sum_values"],
        "distribution": ["DEFAULT_CHUNK_AMPLITUDES", "RankTopology", "rank_and_offset",
                         "exchange_partner", "GroupComm", "single_rank_comm",
                         "apply_one_qubit_gate", "apply_controlled_gate", "group_reduce_sum",
                         "measure_probability", "measure_norm_squared", "measure_maxcut",
                         "measure_z", "TransportTimeout"],
        "runtime": ["NormDriftError", "RankContext", "make_context", "reset_state", "apply_gate",
                    "run_circuit", "run_circuit_pool", "measure_probability", "measure_maxcut",
                    "measure_z", "gather_group_state", "run_spmd", "simulate_circuit",
                    "NORM_CHECK_INTERVAL", "NORM_TOL"],
        "pool": ["PoolLayout", "build_pool"],
        "gates": ["HADAMARD", "PAULI_X", "PAULI_Y", "PAULI_Z", "IDENTITY", "rx", "ry", "rz",
                  "is_unitary", "gate_matrix", "FIXED_GATES", "ROTATION_GATES"],
        "graphs": ["Graph", "make_graph", "triangle"],
    }
    for mod, names in expected.items():
        m = getattr(qs, mod)
        missing = [n for n in names if not hasattr(m, n)]
        assert not missing, (mod, missing)


def test_pool_helpers_follow_reference_tree_order():
    from paper_2001_10554_b200 import pool, runtime
    from paper_2001_10554_b200.statevector import tree_sum_values

    vals = np.random.default_rng(2).standard_normal(7)
    assert pool.incoherent_sum_over_pool(0.3, pool.build_pool(1, 1), None) == 0.3
    # world 7, 3 states of 2 ranks (rank 6 idle): every rank gets the tree sum
    # of the group leaders' values, rank 0 the values in group order
    import threading
    from paper_2001_10554_b200 import transport as tp
    fab = tp.InProcessFabric(7, timeout=5.0)
    layout = pool.build_pool(7, 3)
    out = [None] * 7

    def run(r):
        t = fab.endpoint(r)
        g = layout.group_of_rank(r)
        mine = 0.0 if g is None else float(vals[g])
        out[r] = (pool.incoherent_sum_over_pool(mine, layout, t),
                  pool.gather_state_values(mine, layout, t))

    ts = [threading.Thread(target=run, args=(r,)) for r in range(7)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(o[0] == tree_sum_values(vals[:3]) for o in out)
    assert np.array_equal(out[0][1], vals[:3]) and all(o[1] is None for o in out[1:])
    assert runtime.pool_sum(None, vals) == tree_sum_values(vals)
    assert runtime.pool_sum(None, 0.25) == 0.25
    assert np.array_equal(runtime.pool_gather(None, vals, 3), vals[:3])
    s = pool.RandomStream(3, pool.SCOPE_POOL, 0)
    assert np.array_equal(pool.uniform_randoms(s, 4, 0.0, 2.0),
                          pool.RandomStream(3, pool.SCOPE_POOL, 0).uniform(4, 0.0, 2.0))
