"""Device-resident state slices and the local kernels -- the drop-in for
qpool.statevector (reference pkg/src/qpool/statevector.py).

Same names, arguments, return values and exceptions as the reference; the
amplitudes live in B200 HBM inside libqsb200 and every kernel is a CUDA launch
through the C ABI (include/qsb200.h).  Layout is the reference's: rank r of a
2^p-rank group owns global indices [r*2^m, (r+1)*2^m), qubit 0 is the LSB.

``StatePartition.amplitudes`` is a host mirror: reading it downloads the
slice; the next device operation uploads the mirror back first (so code that
writes ``part.amplitudes[:] = x`` as the reference tests do keeps working)
and then drops it.  Large runs should not touch it inside a hot loop.
"""
from __future__ import annotations

import numpy as np

from . import _native
from ._native import LocalityError, DeviceState
from .graphs import edge_array, phase_lut

__all__ = [
    "LocalityError", "StatePartition", "allocate_partition", "full_state_bytes", "read_amplitudes",
    "exchange_amplitudes",
    "init_basis_state", "init_uniform", "pair_update", "apply_local_one_qubit_gate",
    "apply_local_controlled_gate", "apply_diagonal_phase", "apply_cut_phase", "CutPhase",
    "norm_squared", "get_probability", "z_expectation", "maxcut_expectation",
    "tree_sum", "combine_pair", "tree_sum_values",
]


# ---- host reductions over rank partials (statevector.py:29-71) --------------------
def tree_sum(values) -> float:
    """Perfect-binary-tree sum of a power-of-two-length array (statevector.py:29-45)."""
    x = np.asarray(values, dtype=np.float64).ravel()
    if x.size == 0:
        return 0.0
    if x.size & (x.size - 1):
        raise ValueError(f"tree_sum requires power-of-two length, got {x.size}")
    while x.size > 1:
        x = x[0::2] + x[1::2]
    return float(x[0])


def combine_pair(lo: float, hi: float) -> float:
    return lo + hi


def tree_sum_values(values) -> float:
    """Tree-order sum of any number of scalars, split at the largest power of
    two below the length (statevector.py:53-71)."""
    vals = [float(v) for v in values]
    if not vals:
        return 0.0

    def rec(lo: int, hi: int) -> float:
        k = hi - lo
        if k == 1:
            return vals[lo]
        split = 1 << ((k - 1).bit_length() - 1)
        return combine_pair(rec(lo, lo + split), rec(lo + split, hi))

    return rec(0, len(vals))


def pair_update(a: np.ndarray, b: np.ndarray, u: np.ndarray):
    """Host form of the 2x2 pair update (statevector.py:144-150); the device
    kernels evaluate exactly this expression.  Kept for API compatibility."""
    return u[0, 0] * a + u[0, 1] * b, u[1, 0] * a + u[1, 1] * b


# ---- partitions --------------------------------------------------------------------
class _HostMirror(np.ndarray):
    """Host copy of a device slice that notices writes.

    Item assignment, in-place operators, ufuncs with ``out=`` and the numpy
    functions that write into an argument -- on the mirror or on any view of
    it -- mark the owning partition dirty; only then does the next device
    operation upload it.  Reading never causes an upload (a
    16 GiB H2D after merely inspecting the state).  Copies are plain arrays."""

    def __array_finalize__(self, obj):
        self._owner = getattr(obj, "_owner", None)

    def _touch(self):
        owner = self._owner
        if owner is not None:
            owner._dirty = True

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        self._touch()

    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        args = [x.view(np.ndarray) if isinstance(x, _HostMirror) else x for x in inputs]
        outs = kwargs.get("out")
        if outs:
            kwargs["out"] = tuple(o.view(np.ndarray) if isinstance(o, _HostMirror) else o
                                  for o in outs)
        res = getattr(ufunc, method)(*args, **kwargs)
        if outs:
            for o in outs:
                if isinstance(o, _HostMirror):
                    o._touch()
            return outs[0] if len(outs) == 1 else outs
        return res

    _WRITERS = ("copyto", "place", "put", "putmask", "put_along_axis", "fill_diagonal")

    def __array_function__(self, func, types, args, kwargs):
        res = super().__array_function__(func, types, args, kwargs)
        if func.__name__ in self._WRITERS and args and isinstance(args[0], _HostMirror):
            args[0]._touch()
        if isinstance(res, _HostMirror) and res.base is None:
            res = res.view(np.ndarray)  # a fresh array, not a view of the slice
        return res

    def fill(self, value):
        super().fill(value)
        self._touch()

    def put(self, *a, **k):
        super().put(*a, **k)
        self._touch()

    def sort(self, *a, **k):
        super().sort(*a, **k)
        self._touch()

    def copy(self, order="C"):
        return np.array(self.view(np.ndarray), copy=True, order=order)


class StatePartition:
    """One rank's slice of 2^m amplitudes on a CUDA device (statevector.py:74-108).

    ``amplitudes`` (the reference's field, a constructor argument there) may be
    None here: the slice is then allocated on the device without a host copy.
    Reading ``amplitudes`` downloads a write-tracking host mirror; writes
    through it (``part.amplitudes[:] = x``, as the reference's tests do) are
    uploaded before the next device operation, reads are not."""

    def __init__(self, num_qubits: int, num_local_qubits: int, rank_index: int,
                 amplitudes: np.ndarray | None, *, device: int = 0):
        n, m, r = num_qubits, num_local_qubits, rank_index
        if not (0 < m <= n):
            raise ValueError(f"need 0 < num_local_qubits <= num_qubits, got m={m}, n={n}")
        if not (0 <= r < (1 << (n - m))):
            raise ValueError(f"rank_index {r} out of range for {n - m} rank bits")
        if amplitudes is not None:
            amplitudes = np.asarray(amplitudes)
            if amplitudes.shape != (1 << m,):
                raise ValueError(
                    f"amplitude slice must have length 2**{m}, got {amplitudes.shape}")
            if amplitudes.dtype != np.complex128:
                raise ValueError("amplitudes must be complex128")
        self.num_qubits = n
        self.num_local_qubits = m
        self.rank_index = r
        self.device = device
        self.state = DeviceState(n, m, r, 1, device)
        self._mirror: _HostMirror | None = None
        self._dirty = False
        if amplitudes is not None:
            self.state.upload(amplitudes)

    # reference properties
    @property
    def num_rank_bits(self) -> int:
        return self.num_qubits - self.num_local_qubits

    @property
    def global_offset(self) -> int:
        return self.rank_index << self.num_local_qubits

    def owned_indices(self) -> np.ndarray:
        base = self.global_offset
        return np.arange(base, base + (1 << self.num_local_qubits), dtype=np.uint64)

    @property
    def amplitudes(self) -> np.ndarray:
        if self._mirror is None:
            mirror = self.state.download().view(_HostMirror)
            mirror._owner = self
            self._mirror, self._dirty = mirror, False
        return self._mirror

    @amplitudes.setter
    def amplitudes(self, value) -> None:
        value = np.ascontiguousarray(value, dtype=np.complex128)
        if value.shape != (1 << self.num_local_qubits,):
            raise ValueError("amplitude slice has the wrong length")
        self._drop_mirror()
        self.state.upload(value)

    def _drop_mirror(self) -> None:
        if self._mirror is not None:
            self._mirror._owner = None  # later writes to it no longer reach the state
        self._mirror, self._dirty = None, False

    def sync_in(self, mutating: bool = True) -> DeviceState:
        """Before a device operation: upload the host mirror if it was written;
        a mutating operation then drops it (a read-only one keeps it)."""
        if self._mirror is not None and self._dirty:
            self.state.upload(self._mirror.view(np.ndarray))
            self._dirty = False
        if mutating:
            self._drop_mirror()
        return self.state

    def __repr__(self) -> str:
        return (f"StatePartition(num_qubits={self.num_qubits}, "
                f"num_local_qubits={self.num_local_qubits}, rank_index={self.rank_index}, "
                f"device={self.device})")


def read_amplitudes(partition: StatePartition, out: np.ndarray | None = None) -> np.ndarray:
    """Copy the slice into `out` (e.g. a pinned host buffer) or a new array;
    unlike ``.amplitudes`` no host mirror is kept."""
    st = partition.sync_in(False)
    return st.download(out)


def exchange_amplitudes(partition: StatePartition, new: np.ndarray, out: np.ndarray) -> None:
    """Read the slice into `out` while `new` replaces it -- one full-duplex,
    chunked transfer (pinned buffers recommended; they must not alias)."""
    partition.sync_in()
    if new.shape != (1 << partition.num_local_qubits,) or out.shape != new.shape:
        raise ValueError("amplitude buffers have the wrong length")
    partition.state.exchange_host(np.ascontiguousarray(new, dtype=np.complex128), out)


def allocate_partition(num_qubits: int, num_local_qubits: int | None = None,
                       rank_index: int = 0, *, device: int = 0) -> StatePartition:
    """A zeroed slice on the device (statevector.py:111-115)."""
    m = num_qubits if num_local_qubits is None else num_local_qubits
    part = StatePartition(num_qubits, m, rank_index, None, device=device)
    _native.call("qs_init_zero", part.state.handle)
    return part


def full_state_bytes(num_qubits: int) -> int:
    return 1 << (3 + 1 + num_qubits)


def init_basis_state(partition: StatePartition, index: int) -> StatePartition:
    if not (0 <= index < (1 << partition.num_qubits)):
        raise ValueError(
            f"basis index {index} out of range for {partition.num_qubits} qubits")
    partition._drop_mirror()
    if partition.num_local_qubits == partition.num_qubits:
        partition.state.defer_basis(index)  # carried out at the next access of the device state
    else:
        _native.call("qs_init_basis", partition.state.handle, index)
    return partition


def init_uniform(partition: StatePartition) -> StatePartition:
    partition._drop_mirror()
    # the value the reference assigns (statevector.py:140), evaluated on the host
    value = 2.0 ** (-partition.num_qubits / 2.0)
    _native.call("qs_init_constant", partition.state.handle, value, 0.0)
    return partition


def _u8(u) -> np.ndarray:
    m = np.ascontiguousarray(np.asarray(u, dtype=np.complex128))
    if m.shape != (2, 2):
        raise ValueError(f"gate matrix must be 2x2, got shape {m.shape}")
    return m


def apply_local_one_qubit_gate(partition: StatePartition, q: int, u) -> StatePartition:
    """In-place 2x2 on local qubit q (statevector.py:162-177) -- one HBM pass."""
    if q >= partition.num_local_qubits:
        raise LocalityError(
            f"qubit {q} is global for m={partition.num_local_qubits}; "
            "route through the distribution module")
    if q < 0:
        raise ValueError("negative qubit index")
    m = _u8(u)
    st = partition.sync_in()
    _native.call("qs_apply_1q", st.handle, q, _native.dptr(m), 0)
    return partition


def apply_local_controlled_gate(partition: StatePartition, control: int, target: int,
                                u) -> StatePartition:
    """2x2 on target pairs whose control bit is 1 (statevector.py:180-195)."""
    mloc = partition.num_local_qubits
    if control == target:
        raise ValueError("control and target must differ")
    if control >= mloc or target >= mloc:
        raise LocalityError("both qubits must be local for the local controlled kernel")
    if control < 0 or target < 0:
        raise ValueError("negative qubit index")
    m = _u8(u)
    st = partition.sync_in()
    _native.call("qs_apply_controlled", st.handle, control, target, _native.dptr(m), 0)
    return partition


class CutPhase:
    """The phase function ``lambda idx: gamma * cut_counts(graph, idx)`` that the
    reference passes to apply_diagonal_phase (runtime.py:131-133), in a form the
    device can evaluate (edge list + LUT)."""

    def __init__(self, graph, gamma: float):
        self.graph = graph
        self.gamma = float(gamma)

    def __call__(self, idx):
        from .graphs import cut_counts
        return self.gamma * cut_counts(self.graph, idx)


def apply_cut_phase(partition: StatePartition, graph, gamma: float) -> StatePartition:
    edges = edge_array(graph)
    lut = phase_lut(gamma, len(edges))
    st = partition.sync_in()
    _native.call("qs_apply_cut_phase", st.handle, _native.iptr(edges), len(edges),
                 _native.dptr(lut), 0)
    return partition


def apply_diagonal_phase(partition: StatePartition, phases) -> StatePartition:
    """psi_i *= exp(-1j * phases(i)) over the owned indices (statevector.py:198-206).

    A :class:`CutPhase` (the reference's in-tree phase function, runtime.py:
    131-133) runs entirely on the device (edge list + LUT).  Any other
    callable is the caller's host code: it is evaluated on the owned indices
    as the reference does, the factors exp(-1j * angles) are formed with the
    same numpy expression, and the device multiplies them in
    (qs_apply_diagonal) -- bit-identical to the reference."""
    if isinstance(phases, CutPhase):
        return apply_cut_phase(partition, phases.graph, phases.gamma)
    angles = np.asarray(phases(partition.owned_indices()), dtype=np.float64)
    factors = np.exp(-1j * angles)
    st = partition.sync_in()
    st.apply_diagonal(np.broadcast_to(factors, (1 << partition.num_local_qubits,)))
    return partition


# ---- observables (partial sums in tree order) ------------------------------------
def norm_squared(partition: StatePartition) -> float:
    return float(partition.sync_in(False).observable(_native.QS_OBS_NORM)[0])


def get_probability(partition: StatePartition, q: int) -> float:
    if not (0 <= q < partition.num_qubits):
        raise ValueError(f"qubit {q} out of range")
    return float(partition.sync_in(False).observable(_native.QS_OBS_PROB, q)[0])


def z_expectation(partition: StatePartition, q: int) -> float:
    if not (0 <= q < partition.num_qubits):
        raise ValueError(f"qubit {q} out of range")
    return float(partition.sync_in(False).observable(_native.QS_OBS_Z, q)[0])


def maxcut_expectation(partition: StatePartition, graph) -> float:
    if graph.num_vertices > partition.num_qubits:
        raise ValueError("graph vertices exceed qubit count")
    return float(partition.sync_in(False).observable(_native.QS_OBS_MAXCUT, 0, edge_array(graph))[0])
