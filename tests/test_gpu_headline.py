"""Parity of the headline at its own size: one BASELINE config-2 sweep at
n=30 (16 GiB; a Haar 2x2 on every qubit 0..29 in turn, statevector.py:162-177,
inputs by the recipes of tests/oracles.py:92-101) on the device, in the
bit-identical mode and in the factored numerics the bench times, against the
CPU oracle run over the same 30 gates on the GPU box's host cores
(oracle.cpu_baseline.apply_1q_threaded, bit-identical to the faithful
restatement, tests/test_oracle.py).

The initial state is the device's counter-based Gaussian (normalised on the
device) -- regenerated bit-identically for each mode, so the host holds only
the oracle's 16 GiB; device results are compared chunk by chunk.
Bars (north_star): exact mode bit-equal; factored mode max|d| <= 1e-12, with
the relative errors ||d||_2/||psi||_2 and max|d|/max|psi| reported."""
import json
import os

import numpy as np
import pytest

from paper_2001_10554_b200 import _native as N
from paper_2001_10554_b200 import runtime

from oracle import cpu_baseline
from oracle import gates as og

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-12
N_QUBITS = 30
CHUNK = 1 << 26


def _fresh_state(n, seed):
    st = N.DeviceState(n, n)
    N.call("qs_init_gaussian", st.handle, seed)
    norm = st.observable(N.QS_OBS_NORM)[0]
    N.call("qs_scale", st.handle, 1.0 / np.sqrt(norm))
    return st


def _sweep(st, us, fuse):
    q = runtime.GateQueue(st, fuse=fuse)
    for k, u in enumerate(us):
        q.one_qubit(k, u)
    return q.flush()


def _compare(st, expect):
    """Chunked download: max|d|, sum|d|^2, bit equality, max|psi|, sum|psi|^2."""
    total = expect.size
    buf = np.empty(CHUNK, dtype=np.complex128)
    mx, sd, mb, sb, equal = 0.0, 0.0, 0.0, 0.0, True
    for off in range(0, total, CHUNK):
        k = min(CHUNK, total - off)
        got = st.download(buf[:k], offset=off, count=k)
        ref = expect[off:off + k]
        d = np.abs(got - ref)
        mx = max(mx, float(d.max()))
        sd += float(np.dot(d, d))
        a = np.abs(ref)
        mb = max(mb, float(a.max()))
        sb += float(np.dot(a, a))
        if equal:
            equal = bool(np.array_equal(got.view(np.uint64), ref.view(np.uint64)))
    return {"max_abs": mx, "rel_l2": (sd / sb) ** 0.5, "rel_max": mx / mb, "bit_equal": equal}


@pytest.mark.timeout(1800)
def test_config2_sweep_n30_exact_and_factored_vs_oracle():
    n = N_QUBITS
    rng = np.random.default_rng(20260809)
    us = [og.random_unitary_2x2(rng) for _ in range(n)]
    seed = 2026
    st = _fresh_state(n, seed)
    expect = st.download()
    del st
    for k, u in enumerate(us):  # the oracle, on every host core
        cpu_baseline.apply_1q_threaded(expect, k, u)
    report = {"n": n, "gates": n, "seed": seed, "oracle_threads": cpu_baseline.threads()}
    for mode, fuse in (("exact", True), ("factored", "factored")):
        st = _fresh_state(n, seed)
        passes = _sweep(st, us, fuse)
        res = _compare(st, expect)
        res["passes"] = passes
        report[mode] = res
        del st
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "headline_parity_n30.json"), "w") as fh:
        json.dump(report, fh, indent=1)
    print(json.dumps(report))
    assert report["exact"]["bit_equal"], report
    assert report["factored"]["max_abs"] <= TOL, report
    assert not report["factored"]["bit_equal"]  # the factored rewrite really ran


@pytest.mark.timeout(900)
def test_config4_layer_n33_product_state():
    """Config 4's N=1 point (n=33, 128 GiB): the lean passes whose tiles hold
    qubit 32, the CNOT pass folded into the last of them and the k_perm pass,
    checked through a size-independent property -- a Haar layer takes the
    uniform product state to the product state of the gates' first-column
    sums, and the CNOT layer permutes its indices -- on sampled index ranges,
    factored mode (1e-12 absolute; the amplitudes are ~1e-5)."""
    n = 33
    try:
        st = N.DeviceState(n, n)
    except MemoryError as exc:
        pytest.skip(f"no room for a 2^{n} state: {exc}")
    rng = np.random.default_rng(3333)
    us = [og.random_unitary_2x2(rng) for _ in range(n)]
    pairs = [(q, n - 1 - q) for q in range(n // 2)]
    X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
    N.call("qs_init_constant", st.handle, 2.0 ** (-n / 2.0), 0.0)
    q = runtime.GateQueue(st, fuse="factored")
    for k in range(n):
        q.one_qubit(k, us[k])
    for c, t in pairs:
        q.controlled(c, t, X)
    passes = q.flush()
    assert passes <= 6
    # per-qubit factors of the product state after the Haar layer
    f = np.array([(u @ np.array([1.0, 1.0])) / np.sqrt(2.0) for u in us])  # f[q][bit]

    def expect(idx):
        idx = np.asarray(idx, dtype=np.uint64)
        src = idx.copy()
        for c, t in reversed(pairs):  # out[i] = in[f_1(f_2(..f_k(i)))]
            src ^= ((src >> np.uint64(c)) & np.uint64(1)) << np.uint64(t)
        out = np.ones(idx.shape, dtype=np.complex128)
        for k in range(n):
            out *= f[k][((src >> np.uint64(k)) & np.uint64(1)).astype(np.int64)]
        return out

    worst = 0.0
    for off in (0, 12345 * 4096, (1 << 32) + 777 * 512, (1 << 33) - 8192,
                int(rng.integers(0, (1 << 33) - 8192)) & ~511):
        got = st.download(offset=off, count=8192)
        want = expect(np.arange(off, off + 8192, dtype=np.uint64))
        worst = max(worst, float(np.max(np.abs(got - want))))
    assert worst <= 1e-12, worst
    assert worst <= 1e-9 * 2.0 ** (-n / 2.0) * 1e3  # ~1e-11 relative to the amplitude scale
    norm = float(st.observable(N.QS_OBS_NORM)[0])
    assert abs(norm - 1.0) <= 1e-10
