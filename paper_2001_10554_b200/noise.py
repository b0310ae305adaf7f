"""Stochastic T1/T2 noise trajectories -- the drop-in for qpool.noise
(reference pkg/src/qpool/noise.py) and the keyed random streams it draws from
(qpool.pool.RandomStream, pool.py:27-78).

A noise gate of duration d is Rz(tz) @ Ry(ty) @ Rx(tx) with
tx, ty ~ N(0, d/T1) and tz ~ N(0, 2d(1/T2 - 1/(2 T1))), three normals drawn in
the order (tx, ty, tz) from the trajectory's state-scope stream
(noise.py:70-80).  The gate itself is an ordinary one-qubit update on the
device; in pool mode every state s carries its own trajectory stream and the
S matrices of one noise gate become a per-state table of a fused tile pass
(runtime.run_circuit / run_noise_ensemble), so a whole round of S trajectories
costs one program per circuit instead of S.

What stays on the host is parameter preparation, as in the reference: the
Philox draws, the inverse normal CDF and the 2x2 products.  They are
vectorised over the S streams here (one numpy expression per Philox round
instead of S generator constructions) and are bit-identical to the
reference's scalar path:

* ``philox4x64_uniform`` restates numpy's Philox4x64-10 bit generator
  (counter pre-incremented per 4-word block, ``random()`` = top 53 bits
  x 2^-53); tests/test_noise.py checks it word-for-word against
  ``np.random.Philox``.
* the normal draw is ``scipy.special.ndtri`` of the clipped uniforms, the
  reference's own call (pool.py:75-78).
* ``compose_2x2`` is the host product ``qs_compose_2x2`` in libqsb200
  (include/qsb200.h); it evaluates each entry as the FMA chain the
  reference's ``@`` (OpenBLAS zgemm) produced when the golden trajectories
  were generated, so noisy states match tests/golden/golden_noise.npz
  bit-for-bit on any host.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
from scipy.special import ndtri

from . import _native
from . import gates as G

__all__ = [
    "NoiseModel", "NOISELESS", "RandomStream", "StreamBatch", "SCOPE_POOL", "SCOPE_STATE",
    "SCOPE_LOCAL", "trajectory_stream", "noise_gate_matrix", "noise_gate_matrices",
    "schedule_noise", "philox4x64_uniform", "compose_2x2",
]

_MASK64 = (1 << 64) - 1
SCOPE_POOL, SCOPE_STATE, SCOPE_LOCAL = "pool", "state", "local"
_SCOPE_IDS = {SCOPE_POOL: 1, SCOPE_STATE: 2, SCOPE_LOCAL: 3}


def _splitmix64(x: int) -> int:
    """SplitMix64 finaliser used for key mixing (pool.py:27-31)."""
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


# ---- Philox4x64-10, vectorised over independent keys ---------------------------------
_M0 = np.uint64(0xD2E7470EE14C6C93)
_M1 = np.uint64(0xCA5A826395121157)
_W0 = np.uint64(0x9E3779B97F4A7C15)
_W1 = np.uint64(0xBB67AE8584CAA73B)
_LO32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def _mulhilo(a: np.uint64, b: np.ndarray):
    """(hi, lo) 64-bit halves of a*b, elementwise, from 32-bit partial products."""
    al, ah = a & _LO32, a >> _S32
    bl, bh = b & _LO32, b >> _S32
    ll, lh, hl, hh = al * bl, al * bh, ah * bl, ah * bh
    mid = (ll >> _S32) + (lh & _LO32) + (hl & _LO32)
    hi = hh + (lh >> _S32) + (hl >> _S32) + (mid >> _S32)
    return hi, a * b


def _philox_block(k0, k1, c0, c1):
    """Philox4x64-10 of counter (c0, c1, 0, 0) under key (k0, k1), arrays
    broadcast; the four output words.  Runs in libqsb200 (qs_philox4x64)."""
    shape = np.broadcast(k0, k1, c0, c1).shape
    keys = np.empty(shape + (2,), dtype=np.uint64)
    keys[..., 0], keys[..., 1] = k0, k1
    ctr = np.empty(shape + (2,), dtype=np.uint64)
    ctr[..., 0], ctr[..., 1] = c0, c1
    out = np.empty(shape + (4,), dtype=np.uint64)
    _native.call("qs_philox4x64", _native.u64ptr(keys), _native.u64ptr(ctr),
                 int(np.prod(shape, dtype=np.int64)), _native.u64ptr(out))
    return [out[..., j] for j in range(4)]


def philox_block_numpy(k0, k1, c0, c1):
    """The same Philox rounds in numpy (the restatement qs_philox4x64 is
    checked against in tests/test_noise.py)."""
    z = np.zeros(np.broadcast(k0, c0).shape, dtype=np.uint64)
    v = [c0 + z, c1 + z, z, z]
    with np.errstate(over="ignore"):
        for r in range(10):
            if r:
                k0 = k0 + _W0
                k1 = k1 + _W1
            hi0, lo0 = _mulhilo(_M0, v[0])
            hi1, lo1 = _mulhilo(_M1, v[2])
            v = [hi1 ^ v[1] ^ k0, lo1, hi0 ^ v[3] ^ k1, lo0]
    return v


def _to_unit(words: np.ndarray) -> np.ndarray:
    """numpy's next_double: top 53 bits x 2^-53."""
    return (words >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def philox4x64_uniform(keys: np.ndarray, counters: np.ndarray, count: int) -> np.ndarray:
    """[S, count] doubles in [0,1): what ``Generator(Philox(counter=[c,0,0,0],
    key=k)).random(count)`` returns for each (k, c) row.  numpy increments
    the 256-bit counter before every 4-word block, so block b is Philox of
    counter c+1+b."""
    keys = np.asarray(keys, dtype=np.uint64).reshape(-1, 2)
    ctr0 = np.asarray(counters, dtype=np.uint64).reshape(-1, 1)
    blocks = -(-count // 4)
    with np.errstate(over="ignore"):
        c0 = ctr0 + np.arange(1, blocks + 1, dtype=np.uint64)[None, :]
    c1 = (c0 < ctr0).astype(np.uint64)  # carry into the second counter word
    v = _philox_block(keys[:, :1], keys[:, 1:], c0, c1)
    words = np.stack(v, axis=2).reshape(keys.shape[0], blocks * 4)
    return _to_unit(words[:, :count])


def philox4x64_draws3(keys: np.ndarray, counters: np.ndarray, num_calls: int) -> np.ndarray:
    """[S, num_calls, 3]: the uniforms of `num_calls` consecutive
    ``stream.uniform(3)`` calls per stream (call j regenerates from counter
    c+3j, so it uses words 0..2 of block c+3j+1) -- one vectorised Philox
    pass for a whole circuit's noise draws."""
    keys = np.asarray(keys, dtype=np.uint64).reshape(-1, 2)
    ctr0 = np.asarray(counters, dtype=np.uint64).reshape(-1, 1)
    with np.errstate(over="ignore"):
        c0 = ctr0 + np.uint64(1) + np.uint64(3) * np.arange(num_calls, dtype=np.uint64)[None, :]
    c1 = (c0 < ctr0).astype(np.uint64)
    v = _philox_block(keys[:, :1], keys[:, 1:], c0, c1)
    return _to_unit(np.stack(v[:3], axis=2))


# ---- keyed streams ----------------------------------------------------------------------
@dataclass
class RandomStream:
    """Keyed, counter-based uniform stream (pool.py:34-78): Philox keyed by
    (seed, scope, scope_key, salt); each call regenerates from the counter and
    advances it by the draw count."""

    seed: int
    scope: str
    scope_key: int = 0
    salt: int = 0
    counter: int = 0

    def __post_init__(self) -> None:
        if self.scope not in _SCOPE_IDS:
            raise ValueError(f"unknown scope {self.scope!r}")

    def _key(self) -> list:
        mix = _splitmix64(_SCOPE_IDS[self.scope])
        mix = _splitmix64(mix ^ (self.scope_key & _MASK64))
        mix = _splitmix64(mix ^ (self.salt & _MASK64))
        return [self.seed & _MASK64, mix]

    def philox_key(self) -> list:
        """The key words numpy's Philox actually uses for ``key=self._key()``
        (pool.py:70): numpy converts the Python list with ``np.asarray``, so
        a list mixing a word below 2^63 with one above it goes through
        float64 and the large word loses its low bits.  Reproduced here so the
        draws stay identical to the reference's."""
        return [int(w) for w in np.asarray(self._key()).astype(np.uint64)]

    def split(self, salt: int) -> "RandomStream":
        return RandomStream(self.seed, self.scope, self.scope_key,
                            _splitmix64(self.salt ^ _splitmix64(salt)))

    def uniform(self, count: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        if not lo < hi:
            raise ValueError(f"need lo < hi, got [{lo}, {hi})")
        if count < 0:
            raise ValueError("negative draw count")
        u = philox4x64_uniform(np.array([self.philox_key()], dtype=np.uint64),
                               np.array([self.counter], dtype=np.uint64), count)[0]
        self.counter += count
        return lo + u * (hi - lo)

    def normal(self, count: int, std: float = 1.0) -> np.ndarray:
        u = np.clip(self.uniform(count), 1e-300, None)
        return ndtri(u) * std


class StreamBatch:
    """S independent RandomStreams drawn together (one per pool state).  Draws
    equal each member stream's own draws, and member counters advance with
    the batch."""

    def __init__(self, streams):
        self.streams = list(streams)
        if not self.streams:
            raise ValueError("empty stream batch")
        self._keys = np.array([s.philox_key() for s in self.streams], dtype=np.uint64)

    def __len__(self) -> int:
        return len(self.streams)

    def uniform(self, count: int) -> np.ndarray:
        if count < 0:
            raise ValueError("negative draw count")
        ctr = np.array([s.counter for s in self.streams], dtype=np.uint64)
        u = philox4x64_uniform(self._keys, ctr, count)
        for s in self.streams:
            s.counter += count
        return u

    def normal(self, count: int) -> np.ndarray:
        return ndtri(np.clip(self.uniform(count), 1e-300, None))

    def normal3_calls(self, num_calls: int) -> np.ndarray:
        """[S, num_calls, 3]: what `num_calls` successive normal(3) calls
        return, drawn in one pass; counters advance by 3*num_calls."""
        ctr = np.array([s.counter for s in self.streams], dtype=np.uint64)
        u = philox4x64_draws3(self._keys, ctr, num_calls)
        for s in self.streams:
            s.counter += 3 * num_calls
        return ndtri(np.clip(u, 1e-300, None))


def trajectory_stream(seed: int, trajectory_index: int) -> RandomStream:
    """State-scope stream of trajectory t (noise.py:60-69): independent of how
    trajectories are spread over pool states."""
    return RandomStream(seed, SCOPE_STATE, scope_key=trajectory_index)


# ---- the noise model --------------------------------------------------------------------
@dataclass(frozen=True)
class NoiseModel:
    """Relaxation (t1) and dephasing (t2) timescales in gate times (noise.py:32-55)."""

    t1: float
    t2: float

    def __post_init__(self) -> None:
        if not (self.t1 > 0 and self.t2 > 0):
            raise ValueError("timescales must be positive")
        if self.t2 > 2 * self.t1:
            raise ValueError(f"t2 ={self.t2} exceeds 2*t1 ={2 * self.t1}; "
                             "pure-dephasing rate would be negative")

    def variances(self, duration: float) -> tuple:
        if duration < 0:
            raise ValueError("negative noise duration")
        var_xy = duration / self.t1
        var_z = 2.0 * duration * (1.0 / self.t2 - 1.0 / (2.0 * self.t1))
        return var_xy, var_z


NOISELESS = NoiseModel(math.inf, math.inf)


def compose_2x2(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """[S,2,2] products a[s] @ b[s] (qs_compose_2x2; see the module docstring)."""
    a = np.ascontiguousarray(a, dtype=np.complex128).reshape(-1, 2, 2)
    b = np.ascontiguousarray(b, dtype=np.complex128).reshape(-1, 2, 2)
    if a.shape != b.shape:
        raise ValueError("compose_2x2 needs equal stacks")
    out = np.empty_like(a)
    _native.call("qs_compose_2x2", _native.dptr(a), _native.dptr(b), a.shape[0],
                 _native.dptr(out))
    return out


def _matrices_from_draws(draws: np.ndarray, duration: float, model: NoiseModel) -> np.ndarray:
    var_xy, var_z = model.variances(duration)
    sxy, sz = math.sqrt(var_xy), math.sqrt(var_z)
    tx = draws[:, 0] * sxy
    ty = draws[:, 1] * sxy
    tz = draws[:, 2] * sz
    # Rx acts first, so it sits rightmost: (Rz @ Ry) @ Rx (noise.py:80)
    return compose_2x2(compose_2x2(G.rotation_batch("rz", tz), G.rotation_batch("ry", ty)),
                       G.rotation_batch("rx", tx))


def noise_gate_matrix(duration: float, model: NoiseModel, stream: RandomStream) -> np.ndarray:
    """One stochastic rotation as a single 2x2 unitary (noise.py:70-80)."""
    var_xy, var_z = model.variances(duration)  # validates before drawing
    return _matrices_from_draws(stream.normal(3)[None, :], duration, model)[0]


def apply_noise_gate(partition, q: int, duration: float, model: NoiseModel,
                     stream: RandomStream):
    """One stochastic noise gate on a single-rank partition (noise.py:84-90):
    the matrix is drawn on the host from `stream`, the update is the local
    1q kernel on the device."""
    from . import statevector as sv
    return sv.apply_local_one_qubit_gate(partition, q, noise_gate_matrix(duration, model, stream))


def noise_gate_matrices(duration: float, model: NoiseModel, batch: StreamBatch) -> np.ndarray:
    """[S,2,2]: noise_gate_matrix for every stream of the batch, in one pass."""
    model.variances(duration)
    return _matrices_from_draws(batch.normal(3), duration, model)


def circuit_noise_matrices(durations, model: NoiseModel, stream) -> np.ndarray:
    """The matrices of G consecutive noise gates (durations in circuit order)
    drawn from one stream ([G,2,2]) or a StreamBatch ([G,S,2,2]) -- equal to
    calling noise_gate_matrix / noise_gate_matrices gate by gate, but with
    one Philox pass, one ndtri and one batch of 2x2 products for the whole
    circuit (the per-gate host cost of a pool round drops ~100x)."""
    durations = [float(d) for d in durations]
    scales = []
    for d in durations:
        vxy, vz = model.variances(d)
        scales.append((math.sqrt(vxy), math.sqrt(vxy), math.sqrt(vz)))
    single = not isinstance(stream, StreamBatch)
    batch = StreamBatch([stream]) if single else stream
    num, S = len(durations), len(batch)
    if num == 0:
        return np.zeros((0, 2, 2) if single else (0, S, 2, 2), dtype=np.complex128)
    ang = batch.normal3_calls(num) * np.array(scales)[None, :, :]  # [S, num, 3]
    ang = np.ascontiguousarray(ang.transpose(1, 0, 2)).reshape(num * S, 3)
    mats = compose_2x2(compose_2x2(G.rotation_batch("rz", ang[:, 2]),
                                   G.rotation_batch("ry", ang[:, 1])),
                       G.rotation_batch("rx", ang[:, 0])).reshape(num, S, 2, 2)
    return mats[:, 0] if single else mats


# ---- scheduling -------------------------------------------------------------------------
def _touched_qubits(gate) -> tuple:
    if gate.kind == "diagcost":
        return tuple(range(gate.graph.num_vertices))
    return tuple(sorted(gate.qubits))


def schedule_noise(circuit, model: NoiseModel | None = None):
    """Insert noise gates covering each qubit's elapsed time (noise.py:92-139):
    before each gate every touched qubit is covered up to the gate's end;
    after a qubit's last gate it gets one more noise gate from that gate's
    start to the circuit's end; idle qubits get one for the whole duration."""
    from .circuit import Circuit, GateSpec

    if not circuit.gates:
        return circuit
    for g in circuit.gates:
        if g.kind == "noise":
            raise ValueError("circuit already contains noise gates")
        if g.duration < 0:
            raise ValueError(f"gate {g.kind} has negative duration")
    last_gate_of: dict = {}
    for i, g in enumerate(circuit.gates):
        for q in _touched_qubits(g):
            last_gate_of[q] = i
    total_time = sum(g.duration for g in circuit.gates)
    covered = {q: 0.0 for q in range(circuit.num_qubits)}
    out = []
    now = 0.0
    for i, g in enumerate(circuit.gates):
        start, end = now, now + g.duration
        now = end
        touched = _touched_qubits(g)
        for q in touched:
            out.append(GateSpec("noise", (q,), duration=end - covered[q]))
            covered[q] = end
        out.append(g)
        for q in touched:
            if last_gate_of[q] == i:
                out.append(GateSpec("noise", (q,), duration=total_time - start))
    for q in range(circuit.num_qubits):
        if q not in last_gate_of:
            out.append(GateSpec("noise", (q,), duration=total_time))
    return Circuit(circuit.num_qubits, tuple(out))
