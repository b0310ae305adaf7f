"""ctypes binding of libqsb200.so (the C ABI in include/qsb200.h).

This module is the only place the Python shim touches native code.  There is
no CPU fallback: if the library or a CUDA device is missing, every compute
call raises.  Status codes map onto the reference's exception types
(statevector.LocalityError, ValueError, transport.TransportError).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libqsb200.so")

QS_OK, QS_ERR_VALUE, QS_ERR_LOCALITY, QS_ERR_CUDA, QS_ERR_COMM, QS_ERR_NOMEM = range(6)
QS_KIND_1Q, QS_KIND_CTRL, QS_KIND_CUTPHASE = 0, 1, 2
QS_OBS_NORM, QS_OBS_PROB, QS_OBS_Z, QS_OBS_MAXCUT = 0, 1, 2, 3

# Every symbol include/qsb200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "qs_abi_version", "qs_last_error", "qs_device_count", "qs_counters", "qs_host_sync_count",
    "qs_state_create", "qs_state_destroy", "qs_state_info", "qs_state_device_ptr",
    "qs_synchronize", "qs_state_upload", "qs_state_download", "qs_state_exchange_host",
    "qs_init_zero", "qs_init_basis", "qs_init_constant", "qs_init_gaussian", "qs_scale",
    "qs_apply_diagonal", "qs_state_diff",
    "qs_apply_1q", "qs_apply_controlled", "qs_apply_cut_phase", "qs_apply_program",
    "qs_apply_program_on_constant", "qs_plan_program", "qs_last_program_passes", "qs_observable", "qs_marginals",
    "qs_exchange_gate_peer", "qs_exchange_gate_nccl", "qs_swap_qubits_peer",
    "qs_swap_qubits_local", "qs_state_ipc_handle", "qs_peer_open",
    "qs_peer_close", "qs_nccl_unique_id", "qs_comm_init", "qs_comm_destroy",
    "qs_event_record", "qs_event_elapsed_ms", "qs_launch_log", "qs_launch_log_read",
    "qs_compose_2x2", "qs_philox4x64", "qs_decompose_2x2",
    "qs_sync_event", "qs_sync_event_ipc", "qs_sync_event_open", "qs_sync_event_record",
    "qs_stream_wait_event", "qs_stream_busy",
)


class LocalityError(ValueError):
    """A kernel was asked to act on a qubit the local slice does not pair
    (reference statevector.py:25-26)."""


class TransportError(RuntimeError):
    """Exchange/communicator failure (reference transport.py:44-46)."""


class NativeError(RuntimeError):
    """CUDA failure inside libqsb200 (no device, launch error)."""


class QsGate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("target", ctypes.c_int32),
                ("control", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("offset", ctypes.c_uint64), ("stride", ctypes.c_uint64)]


_lib = None
_lock = threading.Lock()

_P = ctypes.c_void_p
_I = ctypes.c_int32
_U = ctypes.c_uint64
_D = ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)
_U64P = ctypes.POINTER(ctypes.c_uint64)
_IP = ctypes.POINTER(ctypes.c_int32)
_UP = ctypes.POINTER(ctypes.c_uint64)
_BP = ctypes.POINTER(ctypes.c_ubyte)

_SIGNATURES = {
    "qs_abi_version": ([], ctypes.c_int),
    "qs_last_error": ([], ctypes.c_char_p),
    "qs_device_count": ([_IP], ctypes.c_int),
    "qs_counters": ([_P, _UP, _UP], ctypes.c_int),
    "qs_host_sync_count": ([], ctypes.c_uint64),
    "qs_state_create": ([_I, _I, _I, _I, _I, ctypes.POINTER(_P)], ctypes.c_int),
    "qs_state_destroy": ([_P], ctypes.c_int),
    "qs_state_info": ([_P, _IP, _IP, _IP, _IP, _UP], ctypes.c_int),
    "qs_state_device_ptr": ([_P, ctypes.POINTER(_P)], ctypes.c_int),
    "qs_synchronize": ([_P], ctypes.c_int),
    "qs_state_upload": ([_P, _DP, _U, _U], ctypes.c_int),
    "qs_state_download": ([_P, _DP, _U, _U], ctypes.c_int),
    "qs_state_exchange_host": ([_P, _DP, _DP, _U], ctypes.c_int),
    "qs_init_zero": ([_P], ctypes.c_int),
    "qs_init_basis": ([_P, _U], ctypes.c_int),
    "qs_init_constant": ([_P, _D, _D], ctypes.c_int),
    "qs_init_gaussian": ([_P, _U], ctypes.c_int),
    "qs_scale": ([_P, _D], ctypes.c_int),
    "qs_apply_diagonal": ([_P, _DP, _U, _U], ctypes.c_int),
    "qs_state_diff": ([_P, _P, _DP], ctypes.c_int),
    "qs_apply_1q": ([_P, _I, _DP, _U], ctypes.c_int),
    "qs_apply_controlled": ([_P, _I, _I, _DP, _U], ctypes.c_int),
    "qs_apply_cut_phase": ([_P, _IP, _I, _DP, _U], ctypes.c_int),
    "qs_apply_program": ([_P, ctypes.POINTER(QsGate), _I, _DP, _U, _IP, _I, _I], ctypes.c_int),
    "qs_apply_program_on_constant": ([_P, _D, _D, ctypes.POINTER(QsGate), _I, _DP, _U, _IP, _I, _I],
                                     ctypes.c_int),
    "qs_plan_program": ([_I, ctypes.POINTER(QsGate), _I, _I, _IP, _I, _IP], ctypes.c_int),
    "qs_last_program_passes": ([_P, _IP], ctypes.c_int),
    "qs_observable": ([_P, _I, _I, _IP, _I, _DP], ctypes.c_int),
    "qs_marginals": ([_P, _DP], ctypes.c_int),
    "qs_compose_2x2": ([_DP, _DP, ctypes.c_int64, _DP], ctypes.c_int),
    "qs_decompose_2x2": ([_DP, _DP], ctypes.c_int),
    "qs_philox4x64": ([_U64P, _U64P, ctypes.c_int64, _U64P], ctypes.c_int),
    "qs_exchange_gate_peer": ([_P, _P, _I, _DP, _I], ctypes.c_int),
    "qs_exchange_gate_nccl": ([_P, _I, _I, _DP, _I, _U], ctypes.c_int),
    "qs_swap_qubits_peer": ([_P, _P, _I, _I], ctypes.c_int),
    "qs_swap_qubits_local": ([_P, _I, _I], ctypes.c_int),
    "qs_state_ipc_handle": ([_P, _BP], ctypes.c_int),
    "qs_peer_open": ([_P, _BP, ctypes.POINTER(_P)], ctypes.c_int),
    "qs_peer_close": ([_P, _P], ctypes.c_int),
    "qs_nccl_unique_id": ([_BP], ctypes.c_int),
    "qs_sync_event": ([_P, _I, ctypes.POINTER(_P)], ctypes.c_int),
    "qs_sync_event_ipc": ([_P, _I, _BP], ctypes.c_int),
    "qs_sync_event_open": ([_P, _BP, ctypes.POINTER(_P)], ctypes.c_int),
    "qs_sync_event_record": ([_P, _I], ctypes.c_int),
    "qs_stream_wait_event": ([_P, _P], ctypes.c_int),
    "qs_stream_busy": ([_P, _IP], ctypes.c_int),
    "qs_comm_init": ([_P, _BP, _I, _I], ctypes.c_int),
    "qs_comm_destroy": ([_P], ctypes.c_int),
    "qs_event_record": ([_P, _I], ctypes.c_int),
    "qs_event_elapsed_ms": ([_P, _I, _I, ctypes.POINTER(ctypes.c_float)], ctypes.c_int),
    "qs_launch_log": ([_P, _I], ctypes.c_int),
    "qs_launch_log_read": ([_P, ctypes.POINTER(ctypes.c_float), _IP, _I, _IP], ctypes.c_int),
}


def load(path: str | None = None):
    """Load (once) and return the ctypes handle of libqsb200.so."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # QSB_LIB: an alternative build of the same library (tools/exp variants)
        path = path or os.environ.get("QSB_LIB") or LIB_PATH
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -m paper_2001_10554_b200.build` "
                "(the B200 core has no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == QS_OK:
        return
    msg = (load().qs_last_error() or b"").decode(errors="replace")
    if rc == QS_ERR_VALUE:
        raise ValueError(msg)
    if rc == QS_ERR_LOCALITY:
        raise LocalityError(msg)
    if rc == QS_ERR_COMM:
        raise TransportError(msg)
    if rc == QS_ERR_NOMEM:
        raise MemoryError(msg)
    raise NativeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def host_sync_count() -> int:
    """Host-blocking CUDA calls the library has made in this process
    (qs_host_sync_count): stream/event/device synchronisations."""
    return int(load().qs_host_sync_count())


def device_count() -> int:
    n = ctypes.c_int32(0)
    rc = load().qs_device_count(ctypes.byref(n))
    return n.value if rc == QS_OK else 0


FUSE_NONE, FUSE_EXACT, FUSE_FACTORED = 0, 1, 2


def fuse_code(fuse) -> int:
    """False -> QS_FUSE_NONE, True -> QS_FUSE_EXACT (bit-identical to the
    reference), "factored" -> QS_FUSE_FACTORED (include/qsb200.h: Euler-
    factored 1q gates, within 1e-12 of the reference)."""
    if isinstance(fuse, str):
        if fuse == "factored":
            return FUSE_FACTORED
        if fuse == "exact":
            return FUSE_EXACT
        raise ValueError(f"unknown fuse mode {fuse!r}")
    if fuse is True or fuse is False or fuse is None:
        return FUSE_EXACT if fuse else FUSE_NONE
    code = int(fuse)
    if code not in (FUSE_NONE, FUSE_EXACT, FUSE_FACTORED):
        raise ValueError(f"unknown fuse mode {fuse!r}")
    return code


def decompose_2x2(u) -> tuple:
    """qs_decompose_2x2: u = k diag(1,za) R diag(1,zb) with R = scale *
    [[1,-t],[t,1]] (form is always 0)."""
    u = np.ascontiguousarray(u, dtype=np.complex128).reshape(2, 2)
    out = np.zeros(10)
    call("qs_decompose_2x2", dptr(u.view(np.float64).ravel()), dptr(out))
    return (complex(out[0], out[1]), complex(out[2], out[3]), complex(out[4], out[5]),
            int(out[6]), float(out[7]), float(out[8]))


def plan_program(num_local_qubits: int, gates, fuse: bool = True) -> list[int]:
    """First gate index of every pass the native planner would launch (CPU only)."""
    n = len(gates)
    arr = gates if isinstance(gates, ctypes.Array) else (QsGate * max(n, 1))(*gates)
    starts = (ctypes.c_int32 * max(n, 1))()
    count = ctypes.c_int32(0)
    call("qs_plan_program", num_local_qubits, arr, n, fuse_code(fuse), starts, max(n, 1),
         ctypes.byref(count))
    return list(starts[:count.value])


def dptr(a: np.ndarray):
    """float64 pointer to a C-contiguous array (complex128 or float64)."""
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(_DP)


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_IP)


def u64ptr(a: np.ndarray):
    if a.dtype != np.uint64 or not a.flags["C_CONTIGUOUS"]:
        raise ValueError("need a C-contiguous uint64 array")
    return a.ctypes.data_as(_U64P)


_H_BITS = (np.array([[1, 1], [1, -1]], dtype=np.complex128) / np.sqrt(2.0)).tobytes()


def leading_hadamard_layer(gates, mats: np.ndarray, num_qubits: int) -> int:
    """num_qubits when the program starts with one shared-matrix H (the bits of
    gates.HADAMARD, gates.py:15) on every qubit, in any order; 0 otherwise."""
    if len(gates) < num_qubits:
        return 0
    seen = 0
    for k in range(num_qubits):
        g = gates[k]
        if g.kind != QS_KIND_1Q or g.stride != 0 or not (0 <= g.target < num_qubits):
            return 0
        if (seen >> g.target) & 1:
            return 0
        if mats[g.offset:g.offset + 8].tobytes() != _H_BITS:
            return 0
        seen |= 1 << g.target
    return num_qubits


def hadamard_chain(num_qubits: int) -> float:
    """The amplitude of H^(x)n |0..0> as statevector.pair_update computes it
    gate by gate (statevector.py:144-150): n roundings of v * fl(1/sqrt 2)."""
    h = float(np.frombuffer(_H_BITS, dtype=np.float64)[0])
    v = 1.0
    for _ in range(num_qubits):
        v = v * h
    return v


class DeviceState:
    """Owning handle of one qs_state (num_states partitions of 2^m amplitudes)."""

    def __init__(self, num_qubits: int, num_local_qubits: int, rank_index: int = 0,
                 num_states: int = 1, device: int = 0):
        lib = load()
        h = _P()
        check(lib.qs_state_create(num_qubits, num_local_qubits, rank_index, num_states, device,
                                  ctypes.byref(h)))
        self._h = h
        self.num_qubits = num_qubits
        self.num_local_qubits = num_local_qubits
        self.rank_index = rank_index
        self.num_states = num_states
        self.device = device
        self.amps_per_state = 1 << num_local_qubits
        self._pending_basis = None

    @property
    def handle(self):
        """The qs_state pointer for a native call.  A deferred basis-state
        reset (defer_basis) is carried out first, so every access to the
        device state -- whatever the entry point -- sees the reset state."""
        if self._h is None:
            raise ValueError("state was destroyed")
        if self._pending_basis is not None:
            index, self._pending_basis = self._pending_basis, None
            check(load().qs_init_basis(self._h, index))
        return self._h

    def defer_basis(self, index: int = 0) -> None:
        """init_basis_state(index), carried out at the next access.  A program
        that arrives first and starts with H on every qubit of |0..0> runs from
        the uniform state instead (apply_program), and the reset is never
        written to HBM."""
        if self._h is None:
            raise ValueError("state was destroyed")
        if not (0 <= index < (1 << self.num_qubits)):
            raise ValueError(f"basis index {index} out of range for {self.num_qubits} qubits")
        self._pending_basis = int(index)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            load().qs_state_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- data movement --------------------------------------------------------
    uploads = 0  # amplitudes uploaded through this handle (host -> device)
    uniform_folds = 0  # programs run from the uniform state (reset + Hadamard layer folded)

    def upload(self, amps: np.ndarray, offset: int = 0) -> None:
        a = np.ascontiguousarray(amps, dtype=np.complex128).ravel()
        call("qs_state_upload", self.handle, dptr(a), offset, a.size)
        self.uploads += a.size

    def apply_diagonal(self, factors: np.ndarray, offset: int = 0) -> None:
        """psi[offset:offset+len] *= factors (qs_apply_diagonal)."""
        f = np.ascontiguousarray(factors, dtype=np.complex128).ravel()
        call("qs_apply_diagonal", self.handle, dptr(f), offset, f.size)

    def download(self, out: np.ndarray | None = None, offset: int = 0,
                 count: int | None = None) -> np.ndarray:
        total = self.amps_per_state * self.num_states
        if count is None:
            count = total - offset
        if out is None:
            out = np.empty(count, dtype=np.complex128)
        call("qs_state_download", self.handle, dptr(out), offset, count)
        return out

    def exchange_host(self, host_in: np.ndarray, host_out: np.ndarray, chunk: int = 1 << 24) -> None:
        """Download into host_out while uploading host_in (full duplex, chunked)."""
        call("qs_state_exchange_host", self.handle, dptr(host_in), dptr(host_out), chunk)
        self.uploads += host_in.size

    def synchronize(self) -> None:
        call("qs_synchronize", self.handle)

    def device_ptr(self) -> int:
        p = _P()
        call("qs_state_device_ptr", self.handle, ctypes.byref(p))
        return p.value

    # ---- cross-rank ordering (qs_sync_event*) ------------------------------------
    def sync_event(self, which: int) -> int:
        p = _P()
        call("qs_sync_event", self.handle, which, ctypes.byref(p))
        return p.value

    def sync_event_ipc(self, which: int) -> bytes:
        buf = (ctypes.c_ubyte * 64)()
        call("qs_sync_event_ipc", self.handle, which, buf)
        return bytes(buf)

    def open_sync_event(self, handle64: bytes) -> int:
        buf = (ctypes.c_ubyte * 64).from_buffer_copy(handle64)
        p = _P()
        call("qs_sync_event_open", self.handle, buf, ctypes.byref(p))
        return p.value

    def record_sync_event(self, which: int) -> None:
        call("qs_sync_event_record", self.handle, which)

    def wait_event(self, ev: int) -> None:
        call("qs_stream_wait_event", self.handle, ctypes.c_void_p(ev))

    def busy(self) -> bool:
        b = ctypes.c_int32(0)
        call("qs_stream_busy", self.handle, ctypes.byref(b))
        return bool(b.value)

    def diff(self, other: "DeviceState") -> dict:
        """Distance to `other` (same shape, same device): max|d|, ||d||_2,
        ||other||_2, max|other| and the relative forms."""
        out = np.zeros(4, dtype=np.float64)
        call("qs_state_diff", self.handle, other.handle, dptr(out))
        mx, sd, sb, mb = (float(x) for x in out)
        return {"max_abs": mx, "l2": sd ** 0.5, "ref_l2": sb ** 0.5, "ref_max": mb,
                "rel_l2": (sd / sb) ** 0.5 if sb > 0 else 0.0,
                "rel_max": mx / mb if mb > 0 else 0.0}

    def counters(self) -> tuple[int, int]:
        msgs, amps = ctypes.c_uint64(0), ctypes.c_uint64(0)
        call("qs_counters", self.handle, ctypes.byref(msgs), ctypes.byref(amps))
        return msgs.value, amps.value

    # ---- kernels ----------------------------------------------------------------
    def apply_program(self, gates: list[QsGate] | ctypes.Array, mats: np.ndarray,
                      edges: np.ndarray | None = None, fuse: bool = True) -> int:
        n = len(gates)
        mats = np.ascontiguousarray(mats, dtype=np.float64)
        uniform = None
        if self._pending_basis == 0 and self.num_qubits == self.num_local_qubits:
            lead = leading_hadamard_layer(gates, mats, self.num_qubits)
            if lead:
                # H^(x)n |0..0>: every amplitude is the same product chain in the
                # reference's arithmetic (each H multiplies the one non-zero
                # amplitude of its pair by fl(1/sqrt 2) and adds a signed zero)
                self._pending_basis = None
                self.uniform_folds += 1
                gates = list(gates)[lead:]
                n = len(gates)
                uniform = hadamard_chain(self.num_qubits)
        arr = gates if isinstance(gates, ctypes.Array) else (QsGate * n)(*gates)
        if edges is None:
            e = np.zeros(2, dtype=np.int32)
            ne = 0
        else:
            e = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1)
            ne = e.size // 2
            if ne == 0:
                e = np.zeros(2, dtype=np.int32)
        if uniform is not None:
            call("qs_apply_program_on_constant", self.handle, uniform, 0.0, arr, n, dptr(mats),
                 mats.size, iptr(e), ne, fuse_code(fuse))
        else:
            call("qs_apply_program", self.handle, arr, n, dptr(mats), mats.size, iptr(e), ne,
                 fuse_code(fuse))
        passes = ctypes.c_int32(0)
        call("qs_last_program_passes", self.handle, ctypes.byref(passes))
        return passes.value

    def observable(self, kind: int, q: int = 0, edges: np.ndarray | None = None) -> np.ndarray:
        out = np.empty(self.num_states, dtype=np.float64)
        e = np.zeros(2, dtype=np.int32) if edges is None else \
            np.ascontiguousarray(edges, dtype=np.int32).reshape(-1)
        ne = 0 if edges is None else e.size // 2
        if e.size == 0:
            e = np.zeros(2, dtype=np.int32)
        call("qs_observable", self.handle, kind, q, iptr(e), ne, dptr(out))
        return out

    def marginals(self) -> np.ndarray:
        """[num_states, n] probabilities P(q=1) in one pass (qs_marginals)."""
        out = np.empty(self.num_states * self.num_qubits, dtype=np.float64)
        call("qs_marginals", self.handle, dptr(out))
        return out.reshape(self.num_states, self.num_qubits)

    def launch_log(self, enable: bool) -> None:
        call("qs_launch_log", self.handle, 1 if enable else 0)

    def read_launch_log(self, cap: int = 1 << 16) -> tuple[np.ndarray, np.ndarray]:
        ms = (ctypes.c_float * cap)()
        kinds = (ctypes.c_int32 * cap)()
        count = ctypes.c_int32(0)
        call("qs_launch_log_read", self.handle, ms, kinds, cap, ctypes.byref(count))
        k = min(count.value, cap)
        return np.frombuffer(ms, dtype=np.float32, count=k).copy(), \
            np.frombuffer(kinds, dtype=np.int32, count=k).copy()

    def event_record(self, slot: int) -> None:
        call("qs_event_record", self.handle, slot)

    def event_elapsed_ms(self, a: int, b: int) -> float:
        ms = ctypes.c_float(0)
        call("qs_event_elapsed_ms", self.handle, a, b, ctypes.byref(ms))
        return float(ms.value)
