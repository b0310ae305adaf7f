"""The uniform-start fold (DeviceState.defer_basis / apply_program,
qs_apply_program_on_constant in include/qsb200.h): a program that starts with
H on every qubit of a freshly reset |0..0> runs from the constant state
H^(x)n |0..0> instead of resetting and running the Hadamard passes.

CPU part: the constant is what the reference's arithmetic produces
(statevector.py:144-150 restated by oracle/statevector.py), bit for bit, and the
detection only fires on a complete leading Hadamard layer.  GPU part: the
folded program equals the oracle bit for bit in the exact mode (fill + k_tile)
and within 1e-12 in the factored mode (constant generated in the first lean
pool pass), and a deferred reset is seen by every other access.
"""
import numpy as np
import pytest

from paper_2001_10554_b200 import _native as N
from paper_2001_10554_b200 import gates as G

from oracle import gates as ogates
from oracle import statevector as osv


def _gate(kind, target, offset, stride=0, control=-1):
    return N.QsGate(kind, target, control, 0, offset, stride)


@pytest.mark.parametrize("n", [1, 2, 5, 12, 20])
def test_hadamard_chain_is_the_reference_arithmetic(n):
    v = N.hadamard_chain(n)
    m = min(n, 12)  # the chain is the same for every qubit count: check the oracle up to n=12
    psi = np.zeros(1 << m, dtype=np.complex128)
    psi[0] = 1.0
    rng = np.random.default_rng(n)
    for q in rng.permutation(m):
        osv.apply_1q(psi, int(q), G.HADAMARD)
    want = np.full(1 << m, N.hadamard_chain(m) + 0j)
    assert np.array_equal(psi.view(np.uint64), want.view(np.uint64))  # signed zeros too
    assert abs(v - 2.0 ** (-n / 2.0)) <= 4 * n * np.finfo(float).eps * v


def test_leading_hadamard_layer_detection():
    n = 4
    h = G.HADAMARD.view(np.float64).reshape(-1)
    x = np.array([[0, 1], [1, 0]], dtype=np.complex128).view(np.float64).reshape(-1)
    mats = np.concatenate([h, x])
    layer = [_gate(N.QS_KIND_1Q, q, 0) for q in (2, 0, 3, 1)]
    assert N.leading_hadamard_layer(layer, mats, n) == n
    assert N.leading_hadamard_layer(layer + [_gate(N.QS_KIND_1Q, 0, 8)], mats, n) == n
    assert N.leading_hadamard_layer(layer[:3], mats, n) == 0                       # a qubit missing
    assert N.leading_hadamard_layer(layer[:3] + [layer[0]], mats, n) == 0          # a repeat
    assert N.leading_hadamard_layer([_gate(N.QS_KIND_1Q, 1, 8)] + layer, mats, n) == 0  # X first
    per_state = [_gate(N.QS_KIND_1Q, q, 0, stride=8) for q in range(n)]
    assert N.leading_hadamard_layer(per_state, mats, n) == 0                       # per-state tables
    ctrl = layer[:3] + [_gate(N.QS_KIND_CTRL, 1, 0, control=0)]
    assert N.leading_hadamard_layer(ctrl, mats, n) == 0
    minus = mats.copy()
    minus[0] = -minus[0]
    assert N.leading_hadamard_layer(layer, minus, n) == 0                          # not H's bits


# ---- GPU ---------------------------------------------------------------------------


def _qaoa_like(n, S, rng, layers=2):
    """H layer, then per layer a per-state cut phase and per-state RX mixers."""
    edges = [(0, 3), (2, 7), (5, 11), (1, n - 1), (4, 9), (6, 10)]
    prog = [("h", q) for q in rng.permutation(n)]
    for _ in range(layers):
        prog.append(("cut", rng.uniform(0, np.pi, S)))
        beta = rng.uniform(0, np.pi, S)
        prog += [("rx", int(q), beta) for q in range(n)]
    return prog, edges


def _run_pool(pool, prog, graph):
    for op in prog:
        if op[0] == "h":
            pool.queue.one_qubit(int(op[1]), G.HADAMARD)
        elif op[0] == "cut":
            pool.queue.cut_phase(graph, op[1])
        else:
            pool.queue.one_qubit(op[1], np.stack([ogates.rx(float(2 * b)) for b in op[2]]))


def _oracle_pool(n, S, prog, edges, index=0):
    out = np.zeros((S, 1 << n), dtype=np.complex128)
    out[:, index] = 1.0
    for op in prog:
        for s in range(S):
            if op[0] == "h":
                osv.apply_1q(out[s], int(op[1]), G.HADAMARD)
            elif op[0] == "cut":
                osv.apply_cut_phase(out[s], edges, float(op[1][s]))
            else:
                osv.apply_1q(out[s], op[1], ogates.rx(float(2 * op[2][s])))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("fuse", [True, "factored", False])
def test_uniform_start_pool_matches_oracle(fuse):
    from paper_2001_10554_b200 import runtime
    from paper_2001_10554_b200.graphs import make_graph

    rng = np.random.default_rng(77)
    n, S = 13, 5
    prog, edges = _qaoa_like(n, S, rng)
    graph = make_graph(n, edges)
    expect = _oracle_pool(n, S, prog, edges)
    pool = runtime.PoolState(n, S, fuse=fuse)
    for rep in range(2):  # fresh pool, then after an explicit deferred reset on a used pool
        if rep:
            pool.queue.discard()
            pool.state.defer_basis(0)
        _run_pool(pool, prog, graph)
        got = pool.amplitudes()
        assert pool.state._pending_basis is None and pool.state.uniform_folds == rep + 1
        if fuse == "factored":
            assert float(np.max(np.abs(got - expect))) <= 1e-12
        else:
            assert np.array_equal(got.view(np.uint64), expect.view(np.uint64))


@pytest.mark.gpu
def test_no_fold_without_a_fresh_zero_state():
    from paper_2001_10554_b200 import runtime
    from paper_2001_10554_b200.graphs import make_graph

    rng = np.random.default_rng(78)
    n, S = 12, 3
    prog, edges = _qaoa_like(n, S, rng, layers=1)
    graph = make_graph(n, edges)
    # basis state 5: the layer is not a uniform state
    pool = runtime.PoolState(n, S, fuse=True)
    pool.state.defer_basis(5)
    _run_pool(pool, prog, graph)
    got = pool.amplitudes()
    assert pool.state.uniform_folds == 0
    expect = _oracle_pool(n, S, prog, edges, index=5)
    assert np.array_equal(got.view(np.uint64), expect.view(np.uint64))
    # an upload between the reset and the program: the reset lands first, the program
    # runs on the uploaded state
    states = np.stack([ogates.random_state(n, rng) for _ in range(S)])
    pool.state.defer_basis(0)
    pool.state.upload(states)
    assert pool.state._pending_basis is None
    _run_pool(pool, prog, graph)
    got = pool.amplitudes()
    assert pool.state.uniform_folds == 0
    expect = states.copy()
    for op in prog:
        for s in range(S):
            if op[0] == "h":
                osv.apply_1q(expect[s], int(op[1]), G.HADAMARD)
            elif op[0] == "cut":
                osv.apply_cut_phase(expect[s], edges, float(op[1][s]))
            else:
                osv.apply_1q(expect[s], op[1], ogates.rx(float(2 * op[2][s])))
    assert np.array_equal(got.view(np.uint64), expect.view(np.uint64))


@pytest.mark.gpu
def test_deferred_reset_is_seen_by_reads_and_observables():
    n = 12
    st = N.DeviceState(n, n, 0, 2)
    st.upload(np.stack([ogates.random_state(n, np.random.default_rng(s)) for s in range(2)]))
    st.defer_basis(3)
    out = st.download().reshape(2, -1)
    want = np.zeros((2, 1 << n), dtype=np.complex128)
    want[:, 3] = 1.0
    assert np.array_equal(out, want)
    st.defer_basis(0)
    assert np.array_equal(st.observable(N.QS_OBS_NORM), np.ones(2))
    with pytest.raises(ValueError):
        st.defer_basis(1 << n)


@pytest.mark.gpu
def test_program_on_constant_equals_fill_then_program():
    """The C entry point on a single state: shared-matrix program (k_tile / k_fact
    paths take the fill), exact and factored, against init_constant + program."""
    rng = np.random.default_rng(5)
    n = 14
    gates, tabs, off = [], [], 0
    for _ in range(30):
        u = ogates.random_unitary_2x2(rng)
        gates.append(_gate(N.QS_KIND_1Q, int(rng.integers(n)), off))
        tabs.append(u.view(np.float64).reshape(-1))
        off += 8
    mats = np.concatenate(tabs)
    arr = (N.QsGate * len(gates))(*gates)
    e = np.zeros(2, dtype=np.int32)
    c = (0.25, -0.125)
    for fuse in (N.FUSE_NONE, N.FUSE_EXACT, N.FUSE_FACTORED):
        a = N.DeviceState(n, n)
        b = N.DeviceState(n, n)
        N.call("qs_init_constant", a.handle, c[0], c[1])
        N.call("qs_apply_program", a.handle, arr, len(gates), N.dptr(mats), mats.size, N.iptr(e), 0, fuse)
        N.call("qs_apply_program_on_constant", b.handle, c[0], c[1], arr, len(gates), N.dptr(mats),
               mats.size, N.iptr(e), 0, fuse)
        assert np.array_equal(a.download().view(np.uint64), b.download().view(np.uint64))
    b = N.DeviceState(n, n)
    N.call("qs_apply_program_on_constant", b.handle, c[0], c[1], arr, 0, N.dptr(mats), mats.size,
           N.iptr(e), 0, N.FUSE_EXACT)
    assert np.array_equal(b.download(), np.full(1 << n, complex(*c)))


@pytest.mark.gpu
def test_register_api_hadamard_layer_is_folded():
    """The paper-style register: Initialize("base", 0) +
    ApplyHadamard on every qubit runs from the uniform state; the amplitudes are
    the reference's product chain bit for bit, and a later gate sees them."""
    from paper_2001_10554_b200.register import QubitRegister

    n = 13
    reg = QubitRegister(n, "base", 0)
    for q in range(n):
        reg.ApplyHadamard(q)
    reg.ApplyPauliZ(0)
    reg.queue.flush()
    assert reg.state.uniform_folds == 1
    got = reg.state.download()
    v = N.hadamard_chain(n)
    want = np.full(1 << n, v + 0j)
    want[1::2] = -v
    assert np.array_equal(got.real, want.real) and not got.imag.any()
