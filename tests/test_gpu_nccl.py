"""The NCCL exchange path (qs_exchange_gate_nccl: the reference's three-step
Fig. 3 scheme, chunked and double-buffered) exercised on one GPU through a
single-rank communicator: a rank that exchanges with itself sends its upper
half and receives it back as the "partner" half, so the exchange gate equals a
local gate on qubit m-1 -- checked bit for bit against the oracle, with and
without a local control, over several chunk counts."""
import ctypes

import numpy as np
import pytest

from paper_2001_10554_b200 import _native as N

from conftest import bits_equal
from oracle import gates as ogates
from oracle import statevector as osv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_state():
    m = 14
    st = N.DeviceState(m + 1, m, 0, 1, 0)
    uid = (ctypes.c_ubyte * 128)()
    try:
        N.call("qs_nccl_unique_id", uid)
        N.call("qs_comm_init", st.handle, uid, 1, 0)
    except N.NativeError as exc:  # pragma: no cover - depends on the image
        pytest.skip(f"NCCL unavailable: {exc}")
    yield st, m
    N.call("qs_comm_destroy", st.handle)


@pytest.mark.parametrize("chunk_log2", [7, 10, 13, 9])  # growing, then shrinking chunks
@pytest.mark.parametrize("control", [-1, 0, 5, 12])
def test_self_exchange_equals_local_gate_on_top_qubit(nccl_state, chunk_log2, control):
    st, m = nccl_state
    rng = np.random.default_rng(100 * chunk_log2 + control)
    psi = ogates.random_state(m, rng)
    u = ogates.random_unitary_2x2(rng)
    st.upload(psi)
    N.call("qs_exchange_gate_nccl", st.handle, 0, 1, N.dptr(np.ascontiguousarray(u).view(np.float64)),
           control, 1 << chunk_log2)
    got = st.download()
    exp = psi.copy()
    if control < 0:
        osv.apply_1q(exp, m - 1, u)
    else:
        osv.apply_controlled(exp, control, m - 1, u)
    assert bits_equal(got, exp)
