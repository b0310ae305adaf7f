"""Circuit execution over the B200 core -- the caller side of the boundary
(reference pkg/src/qpool/runtime.py: apply_gate 115-152, run_circuit
155-162, run_circuit_pool 192-209, measure_* 212-227, simulate_circuit
291-302).

Differences by design, not in results:
  * Gates are queued per device state and flushed as one program into
    libqsb200, whose native planner fuses consecutive local gates into
    shared-memory tile passes (one HBM read+write per pass).  Per-amplitude
    arithmetic and order are unchanged, so the state is bit-identical to
    gate-by-gate execution.  A global-qubit gate, an observable, or the
    every-100-gates norm check (runtime.py:146-152) flushes the queue.
  * Pool mode (pool.py / runtime.py:192-209) is one batched device state of
    S independent partitions per GPU with per-state matrix/LUT tables: one
    launch per fused pass for the whole pool instead of one circuit per rank
    group.  Pools are split across GPUs by contiguous state blocks (no state
    exchange).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native
from . import distribution as dist
from . import gates as gates_mod
from . import statevector as sv
from .graphs import edge_array, phase_lut, phase_lut_batch
from . import noise as noise_mod

NORM_CHECK_INTERVAL = 100
NORM_TOL = 1e-10


class NormDriftError(RuntimeError):
    """The running state stopped being normalized (runtime.py:40-41)."""


# ---- gate queue -> qs_apply_program ------------------------------------------------
class GateQueue:
    """Pending gates of one device state, flushed as one fused program."""

    def __init__(self, state: _native.DeviceState, fuse: bool = True):
        self.state = state
        self.fuse = fuse
        self.gates: list = []
        self.tables: list = []
        self.size = 0  # doubles
        self.edges: np.ndarray | None = None
        self.passes_total = 0
        self.gates_total = 0
        self.touched: set = set()  # physical positions the queued gates act on
        self._keyed: dict = {}     # table key -> (offset, stride) within this program

    def __len__(self) -> int:
        return len(self.gates)

    def discard(self) -> None:
        """Drop the pending gates without running them."""
        self.gates, self.tables, self.size, self.edges = [], [], 0, None
        self.touched = set()
        self._keyed = {}

    def _add(self, kind: int, target: int, control: int, table: np.ndarray, per_state: bool,
             key=None):
        """Queue a gate whose matrix/LUT table is `table`.  Gates passing the
        same `key` share one copy of the table in the program (e.g. the 20 RX
        mixers of a QAOA layer bound to the same per-state beta table)."""
        if key is not None and key in self._keyed:
            offset, stride = self._keyed[key]
            self.gates.append(_native.QsGate(kind, target, control, 0, offset, stride))
            return
        table = np.ascontiguousarray(table, dtype=np.float64).reshape(-1)
        stride = table.size // self.state.num_states if per_state else 0
        g = _native.QsGate(kind, target, control, 0, self.size, stride)
        if key is not None:
            self._keyed[key] = (self.size, stride)
        self.gates.append(g)
        self.tables.append(table)
        self.size += table.size

    def one_qubit(self, q: int, u, key=None) -> None:
        """u: (2,2) shared or (S,2,2) per state; `key` dedupes repeated tables."""
        u = np.ascontiguousarray(u, dtype=np.complex128)
        self._add(_native.QS_KIND_1Q, q, -1, u.view(np.float64), u.ndim == 3, key)
        self.touched.add(q)

    def controlled(self, c: int, t: int, u) -> None:
        u = np.ascontiguousarray(u, dtype=np.complex128)
        self._add(_native.QS_KIND_CTRL, t, c, u.view(np.float64), u.ndim == 3)
        self.touched.update((c, t))

    def cut_phase(self, graph, gamma) -> None:
        edges = edge_array(graph)
        if self.edges is not None and not np.array_equal(self.edges, edges):
            self.flush()
        self.edges = edges
        self.touched.update(int(x) for x in edges.ravel())
        gam = np.asarray(gamma, dtype=np.float64)
        if gam.ndim == 0:
            lut = phase_lut(float(gam), len(edges))
            self._add(_native.QS_KIND_CUTPHASE, 0, -1, lut.view(np.float64), False)
        else:
            luts = phase_lut_batch(gam, len(edges))
            self._add(_native.QS_KIND_CUTPHASE, 0, -1, luts.view(np.float64), True)

    def flush(self) -> int:
        if not self.gates:
            return 0
        mats = np.concatenate(self.tables) if self.tables else np.zeros(1)
        passes = self.state.apply_program(self.gates, mats, self.edges, self.fuse)
        self.passes_total += passes
        self.gates_total += len(self.gates)
        self.gates, self.tables, self.size = [], [], 0
        self.edges = None
        self.touched = set()
        self._keyed = {}
        return passes


def _matrix_for(gate) -> np.ndarray:
    kind = gate.kind
    if kind in gates_mod.FIXED_GATES:
        return gates_mod.FIXED_GATES[kind]
    if kind in gates_mod.ROTATION_GATES:
        return gates_mod.ROTATION_GATES[kind](_angle(gate))
    if kind in ("custom", "cu"):
        return gates_mod.gate_matrix(gate.matrix)
    if kind == "cx":
        return gates_mod.PAULI_X
    if kind == "cz":
        return gates_mod.PAULI_Z
    if kind == "cphase":
        return gates_mod.cphase(_angle(gate))
    raise ValueError(f"no matrix for gate kind {kind!r}")


def _angle(gate) -> float:
    if isinstance(gate.param, str):
        raise ValueError(f"gate {gate.kind} has unbound slot {gate.param}")
    return float(gate.param)


# ---- contexts ------------------------------------------------------------------------
@dataclass
class RankContext:
    """What one rank (one GPU or one emulated rank) needs to run circuits."""

    comm: dist.GroupComm
    num_qubits: int
    num_states: int = 1
    device: int = 0
    fuse: bool = True
    remap: bool = False
    norm_check_interval: int = NORM_CHECK_INTERVAL
    seed: int = 0
    noise_model: "noise_mod.NoiseModel | None" = None
    state_offset: int = 0  # global index of this context's first pool state
    topology: dist.RankTopology = field(init=False)
    layout: "dist.QubitLayout | None" = field(init=False, default=None)
    partition: sv.StatePartition | None = field(init=False, default=None)
    pool: "PoolState | None" = field(init=False, default=None)
    queue: GateQueue | None = field(init=False, default=None)
    gates_applied: int = field(init=False, default=0)
    _state_stream: object = field(init=False, default=None, repr=False)

    def __post_init__(self) -> None:
        size = self.comm.size if self.num_states == 1 else 1
        self.topology = dist.RankTopology(size, self.num_qubits)
        if self.num_states > 1 and self.comm.size > 1:
            raise ValueError("pool contexts hold whole states; split pools with split_pool()")
        if self.comm.rank < self.topology.effective_ranks:
            if self.num_states == 1:
                self.partition = sv.allocate_partition(
                    self.num_qubits, self.topology.num_local_qubits, self.comm.rank,
                    device=self.device)
                sv.init_basis_state(self.partition, 0)
                self.queue = GateQueue(self.partition.state, self.fuse)
                if self.remap and self.topology.rank_bits > 0:
                    self.layout = dist.QubitLayout(self.num_qubits,
                                                   self.topology.num_local_qubits)
            else:
                self.pool = PoolState(self.num_qubits, self.num_states, self.device, self.fuse)
                self.queue = self.pool.queue
        self.comm.attach(self.partition)

    @property
    def is_idle(self) -> bool:
        return self.queue is None

    @property
    def state_stream(self):
        """The state-scope stream of this context's state (runtime.py:79);
        pools get a StreamBatch with one stream per state."""
        if self._state_stream is None:
            if self.pool is None:
                self._state_stream = noise_mod.RandomStream(self.seed, noise_mod.SCOPE_STATE,
                                                            self.state_offset)
            else:
                self._state_stream = noise_mod.StreamBatch(
                    noise_mod.RandomStream(self.seed, noise_mod.SCOPE_STATE, self.state_offset + s)
                    for s in range(self.num_states))
        return self._state_stream

    @property
    def state(self) -> _native.DeviceState:
        return self.partition.state if self.partition is not None else self.pool.state

    def flush(self) -> None:
        if self.queue is not None:
            if self.partition is not None:
                self.partition.sync_in()
            self.queue.flush()


def make_context(comm: dist.GroupComm | None, num_qubits: int, num_states: int = 1,
                 device: int = 0, fuse: bool = True, remap: bool = False, *, seed: int = 0,
                 noise_model=None, state_offset: int = 0) -> RankContext:
    """remap=True: gates on global qubits first swap the qubit into a local
    position (half the traffic of the reference's exchange, and the gate then
    fuses with its neighbours); reads restore the canonical layout.
    seed/noise_model as the reference's make_context (runtime.py:90-99);
    state_offset: global index of the first pool state (split_pool)."""
    return RankContext(comm or dist.single_rank_comm(), num_qubits, num_states, device, fuse,
                       remap, seed=seed, noise_model=noise_model, state_offset=state_offset)


def reset_state(ctx: RankContext, index: int = 0) -> None:
    if ctx.is_idle:
        return
    ctx.queue.discard()
    if ctx.layout is not None:  # a fresh basis state: back to the canonical layout
        ctx.layout = dist.QubitLayout(ctx.num_qubits, ctx.topology.num_local_qubits)
    if ctx.partition is not None:
        sv.init_basis_state(ctx.partition, index)
    else:
        _native.call("qs_init_basis", ctx.pool.state.handle, index)
    ctx.gates_applied = 0


def _restore(ctx: RankContext) -> None:
    if ctx.layout is not None and not ctx.layout.is_identity():
        ctx.flush()
        dist.restore_layout(ctx.partition, ctx.comm, ctx.topology, ctx.layout)


def _apply_gate_remapped(ctx: RankContext, gate) -> None:
    """apply_gate under a qubit layout: logical qubits are mapped to physical
    positions; a gate on a global position swaps it in first."""
    L, topo, q = ctx.layout, ctx.topology, ctx.queue
    m = topo.num_local_qubits
    kind = gate.kind
    if kind == "diagcost":
        from .graphs import make_graph
        g = gate.graph
        phys = make_graph(ctx.num_qubits, [(L.phys[u], L.phys[v]) for u, v in g.edges])
        q.cut_phase(phys, _angle(gate))
        return
    if kind in ("cx", "cz", "cphase", "cu"):
        c, t = gate.qubits
        u = _matrix_for(gate)
        if L.phys[t] >= m:
            pc = L.phys[c]
            _swap_in(ctx, t, protected=(pc,) if pc < m else ())
        pc, pt = L.phys[c], L.phys[t]
        L.use(pt)
        if pc < m:
            q.controlled(pc, pt, u)
            return
        # control on a rank bit: the queued gate depends on this rank's bit pc,
        # so a later swap of pc (or pt) must not overtake it; mark both on every
        # rank so swap decisions stay identical
        if (ctx.comm.rank >> (pc - m)) & 1:
            q.one_qubit(pt, u)
        q.touched.update((pc, pt))
        return
    qb = gate.qubits[0]
    u = _matrix_for(gate)
    if L.phys[qb] >= m:
        _swap_in(ctx, qb)
    q.one_qubit(L.phys[qb], u)
    L.use(L.phys[qb])


def _swap_in(ctx: RankContext, qubit: int, protected=()) -> None:
    """Swap logical `qubit` (on a rank bit) into a local position: flush the
    queue, then evict the most recently used local position.  Repeated sweeps
    and layered circuits touch qubits cyclically, where the most recently used
    qubit is the one needed last (MRU is the optimal eviction for cyclic use).
    Half the slice crosses to the partner (k_swap_peer) instead of the whole
    slice of a pair exchange, and the gate itself then runs locally and fuses
    with the gates that follow.  (Swapping into an untouched slot without a
    flush was measured to double the swaps in sweeps, tools/exp/remap_policy.py.)"""
    L, m = ctx.layout, ctx.topology.num_local_qubits
    ctx.flush()
    p = L.phys[qubit]
    slot = next((l for l in reversed(L.recent) if l < m and l not in protected), None)
    if slot is None:
        slot = next(l for l in range(m - 1, -1, -1) if l not in protected)
    dist.swap_global_local(ctx.partition, ctx.comm, ctx.topology, L, p, slot)


def _noise_matrix(ctx: RankContext, gate, noise_stream):
    """The noise gate's matrix (noise.py:70-80): (2,2) for one state, (S,2,2)
    for a pool whose states draw from their own streams (runtime.py:122-126)."""
    if ctx.noise_model is None:
        raise ValueError("noise gate requires a noise model on the context")
    stream = ctx.state_stream if noise_stream is None else noise_stream
    if ctx.pool is not None:
        if not isinstance(stream, noise_mod.StreamBatch):
            stream = noise_mod.StreamBatch(stream)
        if len(stream) != ctx.num_states:
            raise ValueError(f"{len(stream)} noise streams for {ctx.num_states} states")
        return noise_mod.noise_gate_matrices(gate.duration, ctx.noise_model, stream)
    if isinstance(stream, noise_mod.StreamBatch):
        raise ValueError("a single-state context takes one noise stream")
    return noise_mod.noise_gate_matrix(gate.duration, ctx.noise_model, stream)


def _circuit_noise(ctx: RankContext, gates, noise_stream):
    """Pre-draw every noise gate of a circuit in one pass (same values, same
    stream advance as drawing gate by gate); None when there are none."""
    durations = [g.duration for g in gates if g.kind == "noise"]
    if not durations or ctx.is_idle:
        return None
    if ctx.noise_model is None:
        raise ValueError("noise gate requires a noise model on the context")
    stream = ctx.state_stream if noise_stream is None else noise_stream
    if ctx.pool is not None:
        if not isinstance(stream, noise_mod.StreamBatch):
            stream = noise_mod.StreamBatch(stream)
        if len(stream) != ctx.num_states:
            raise ValueError(f"{len(stream)} noise streams for {ctx.num_states} states")
    elif isinstance(stream, noise_mod.StreamBatch):
        raise ValueError("a single-state context takes one noise stream")
    return iter(noise_mod.circuit_noise_matrices(durations, ctx.noise_model, stream))


def apply_gate(ctx: RankContext, gate, noise_stream=None, *, noise_matrix=None) -> None:
    """Queue one gate; global-qubit gates flush and exchange (runtime.py:115-152).
    Noise gates draw their matrix from `noise_stream` (default: the context's
    state stream) -- or take a pre-drawn `noise_matrix` -- and then run as
    one-qubit gates."""
    if ctx.is_idle:
        return
    if gate.kind == "noise":
        u = _noise_matrix(ctx, gate, noise_stream) if noise_matrix is None else noise_matrix
        if u.ndim == 3:  # pool: per-state table, every qubit is local
            ctx.queue.one_qubit(gate.qubits[0], u)
            _count_and_check(ctx)
            return
        from .circuit import GateSpec
        gate = GateSpec("custom", gate.qubits, matrix=u)
    if ctx.layout is not None:
        _apply_gate_remapped(ctx, gate)
        # the drift check needs no canonical layout (any association is fine)
        _count_and_check(ctx, restore=False)
        return
    kind = gate.kind
    topo = ctx.topology
    q = ctx.queue
    if kind == "diagcost":
        q.cut_phase(gate.graph, _angle(gate))
    elif kind in ("cx", "cz", "cphase", "cu"):
        c, t = gate.qubits
        u = _matrix_for(gate)
        route = dist.route_controlled(ctx.comm.rank, topo, c, t)
        if route[0] == "local_controlled":
            q.controlled(c, t, u)
        elif route[0] == "local_one_qubit":
            q.one_qubit(t, u)
        elif route[0] == "exchange":
            ctx.flush()
            dist.apply_controlled_gate(ctx.partition, topo, ctx.comm, c, t, u)
    else:
        qb = gate.qubits[0]
        u = _matrix_for(gate)
        route = dist.route_one_qubit(ctx.comm.rank, topo, qb)
        if route[0] == "local":
            q.one_qubit(qb, u)
        else:
            ctx.flush()
            dist.apply_one_qubit_gate(ctx.partition, topo, ctx.comm, qb, u)
    _count_and_check(ctx)


def _count_and_check(ctx: RankContext, restore: bool = True) -> None:
    """Count one applied gate; every norm_check_interval gates check that
    norm^2 is still 1 (runtime.py:146-152) -- for a pool, every state's."""
    ctx.gates_applied += 1
    if ctx.norm_check_interval and ctx.gates_applied % ctx.norm_check_interval == 0:
        norm_sq = measure_norm_squared(ctx, restore=restore)
        worst = float(np.max(np.abs(np.asarray(norm_sq, dtype=np.float64) - 1.0)))
        if worst >= NORM_TOL:
            raise NormDriftError(f"norm^2 drifted to {norm_sq!r} after {ctx.gates_applied} gates")


def run_circuit(ctx: RankContext, circuit, bindings: dict | None = None,
                noise_stream=None, noise_matrices=None) -> None:
    """Queue and flush every gate (runtime.py:155-162).  `noise_matrices`:
    the circuit's noise gates already drawn (noise.circuit_noise_matrices),
    e.g. by a worker thread while the previous round ran."""
    bound = circuit.bind(bindings) if bindings else circuit
    bound.require_bound()
    pre = (iter(noise_matrices) if noise_matrices is not None
           else _circuit_noise(ctx, bound.gates, noise_stream))
    for gate in bound.gates:
        if gate.kind == "noise" and pre is not None:
            apply_gate(ctx, gate, noise_matrix=next(pre))
        else:
            apply_gate(ctx, gate, noise_stream=noise_stream)
    ctx.flush()


def _group_reduce(ctx: RankContext, partial: float) -> float:
    return dist.group_reduce_sum(partial, ctx.topology, ctx.comm)


def measure_norm_squared(ctx: RankContext, restore: bool = True):
    if ctx.is_idle:
        return 0.0
    if restore:
        _restore(ctx)
    ctx.flush()
    if ctx.pool is not None:
        return ctx.pool.observable(_native.QS_OBS_NORM)
    return _group_reduce(ctx, sv.norm_squared(ctx.partition))


def measure_probability(ctx: RankContext, q: int):
    if ctx.is_idle:
        return 0.0
    _restore(ctx)
    ctx.flush()
    if ctx.pool is not None:
        return ctx.pool.observable(_native.QS_OBS_PROB, q)
    return _group_reduce(ctx, sv.get_probability(ctx.partition, q))


def measure_probabilities(ctx: RankContext) -> np.ndarray:
    """P(q=1) for every qubit in one pass over the slice (qs_marginals); each
    value equals measure_probability(ctx, q).  Pools: [num_states, n]."""
    if ctx.is_idle:
        return np.zeros(ctx.num_qubits)
    _restore(ctx)
    ctx.flush()
    if ctx.pool is not None:
        return ctx.pool.state.marginals()
    if ctx.partition is not None:
        ctx.partition.sync_in()
    partial = ctx.state.marginals()[0]
    return np.array([_group_reduce(ctx, float(v)) for v in partial])


def measure_z(ctx: RankContext, q: int):
    if ctx.is_idle:
        return 0.0
    _restore(ctx)
    ctx.flush()
    if ctx.pool is not None:
        return ctx.pool.observable(_native.QS_OBS_Z, q)
    return _group_reduce(ctx, sv.z_expectation(ctx.partition, q))


def measure_maxcut(ctx: RankContext, graph):
    if ctx.is_idle:
        return 0.0
    _restore(ctx)
    ctx.flush()
    if ctx.pool is not None:
        return ctx.pool.observable(_native.QS_OBS_MAXCUT, 0, edge_array(graph))
    return _group_reduce(ctx, sv.maxcut_expectation(ctx.partition, graph))


def gather_group_state(ctx: RankContext) -> np.ndarray | None:
    """Full amplitude vector of the (single) state on rank 0 (runtime.py:239-258).
    Threaded communicators gather through the fabric; TorchComm through
    torch.distributed.gather_object."""
    if ctx.is_idle and not isinstance(ctx.comm, dist.TorchComm):
        return None
    if not ctx.is_idle:
        _restore(ctx)
        ctx.flush()
    mine = ctx.state.download() if not ctx.is_idle else None
    comm = ctx.comm
    if comm.size == 1:
        return mine
    if isinstance(comm, dist.ThreadComm):
        fab = comm.fabric
        with fab._lock:
            fab._gather.setdefault("state", {})[comm.rank] = mine
        comm.allgather(0.0, ctx.topology.effective_ranks)
        if comm.rank != 0:
            return None
        with fab._lock:
            parts = [fab._gather["state"][r] for r in range(ctx.topology.effective_ranks)]
        return np.concatenate(parts)
    import torch.distributed as tdist

    out = [None] * comm.size if comm.rank == 0 else None
    tdist.gather_object(mine, out, dst=comm._global(0), group=comm.group)
    if comm.rank != 0:
        return None
    return np.concatenate([p for p in out[: ctx.topology.effective_ranks]])


# ---- pool mode -----------------------------------------------------------------------
class PoolState:
    """S independent n-qubit states, batched in one device allocation."""

    def __init__(self, num_qubits: int, num_states: int, device: int = 0, fuse: bool = True):
        self.num_qubits = num_qubits
        self.num_states = num_states
        self.state = _native.DeviceState(num_qubits, num_qubits, 0, num_states, device)
        self.queue = GateQueue(self.state, fuse)
        _native.call("qs_init_basis", self.state.handle, 0)

    def observable(self, kind: int, q: int = 0, edges=None) -> np.ndarray:
        self.queue.flush()
        return self.state.observable(kind, q, edges)

    def amplitudes(self) -> np.ndarray:
        self.queue.flush()
        return self.state.download().reshape(self.num_states, -1)


def run_circuit_pool(ctx: RankContext, circuit, slot_tables: dict | None = None,
                     noise_stream=None) -> None:
    """Every pool state runs `circuit`; state s binds slot_tables[name][s]
    (runtime.py:192-209).  Per-state matrices/LUTs go to the device as tables;
    noise gates draw state s's matrix from stream s of `noise_stream` (a
    StreamBatch or a list of streams; default: the states' own streams)."""
    if not slot_tables:
        run_circuit(ctx, circuit, noise_stream=noise_stream)
        return
    if ctx.is_idle:
        return
    S = ctx.num_states
    for name, vals in slot_tables.items():
        if len(vals) != S:
            raise ValueError(f"table for ${name} has {len(vals)} entries for {S} states")
    tables = {k: np.asarray(v, dtype=np.float64) for k, v in slot_tables.items()}
    q = ctx.queue
    pre = _circuit_noise(ctx, circuit.gates, noise_stream)
    rot_cache: dict = {}
    for gate in circuit.gates:
        slot = gate.slot if isinstance(getattr(gate, "param", None), str) else None
        if slot is None:
            if gate.kind == "noise":
                apply_gate(ctx, gate, noise_matrix=next(pre))
                continue
            if ctx.pool is None:
                apply_gate(ctx, gate, noise_stream=noise_stream)
                continue
            _queue_fixed(q, gate)
            continue
        if slot not in tables:
            raise ValueError(f"gate {gate.kind} has unbound slot ${slot}")
        vals = tables[slot]
        if ctx.pool is None:
            # single state: bind value 0 (run_circuit semantics)
            from dataclasses import replace
            apply_gate(ctx, replace(gate, param=float(vals[0])), noise_stream=noise_stream)
            continue
        if gate.kind == "diagcost":
            q.cut_phase(gate.graph, vals)
        elif gate.kind in gates_mod.ROTATION_GATES:
            # one table per (rotation, slot): every gate bound to the slot shares it
            key = ("rot", gate.kind, slot)
            mats = rot_cache.get(key)
            if mats is None:
                mats = rot_cache[key] = gates_mod.rotation_batch(gate.kind, vals)
            q.one_qubit(gate.qubits[0], mats, key=(id(rot_cache), key))
        elif gate.kind == "cphase":
            mats = np.stack([gates_mod.cphase(float(v)) for v in vals])
            q.controlled(gate.qubits[0], gate.qubits[1], mats)
        else:
            raise ValueError(f"gate kind {gate.kind} takes no parameter")
    q.flush()


def run_noise_ensemble(ctx: RankContext, circuit, model, trajectories: int, observe,
                       seed: int | None = None, num_groups: int | None = None):
    """Noisy-trajectory ensemble (cli.py:288-339) on this context.

    Trajectory t runs on pool group t mod num_groups in round t div
    num_groups, drawing its noise from trajectory_stream(seed, t) -- so every
    trajectory is bit-identical to a serial single-state run with the same
    index, however the ensemble is spread.  A pool context runs all of its S
    states as one fused program per round.  `observe(ctx)` returns one value
    (single state) or S values (pool).  Circuits without noise gates get
    schedule_noise() first, as the CLI does.

    Returns (reference, values): the noiseless value (computed with the
    NOISELESS model and trajectory 0's stream) and a float array of length
    `trajectories` holding this context's trajectories (NaN elsewhere)."""
    if trajectories < 1:
        raise ValueError("--trajectories must be >= 1")
    if not any(g.kind == "noise" for g in circuit.gates):
        circuit = noise_mod.schedule_noise(circuit)
    seed = ctx.seed if seed is None else seed
    S = ctx.num_states if ctx.pool is not None else 1
    groups = S if num_groups is None else num_groups
    values = np.full(trajectories, np.nan)
    if ctx.is_idle:
        return None, values

    def streams(first: int):
        if ctx.pool is None:
            return noise_mod.trajectory_stream(seed, first)
        return noise_mod.StreamBatch(noise_mod.trajectory_stream(seed, first + s)
                                     for s in range(S))

    def run(model_, first, stream_fn):
        ctx.noise_model = model_
        reset_state(ctx)
        run_circuit(ctx, circuit, noise_stream=stream_fn(first))
        return np.atleast_1d(np.asarray(observe(ctx), dtype=np.float64))

    durations = [g.duration for g in circuit.gates if g.kind == "noise"]

    def draw(first):
        return noise_mod.circuit_noise_matrices(durations, model, streams(first))

    saved = ctx.noise_model
    try:
        if ctx.pool is None:
            ref = float(run(noise_mod.NOISELESS, 0, streams)[0])
        else:  # every state runs trajectory 0's (noiseless) draws
            ref = float(run(noise_mod.NOISELESS, 0, lambda _f: noise_mod.StreamBatch(
                noise_mod.trajectory_stream(seed, 0) for _ in range(S)))[0])
        firsts = [k * groups + ctx.state_offset for k in range(-(-trajectories // groups))]
        firsts = [f for f in firsts if f < trajectories]
        # round k+1's noise is drawn on a worker thread while round k runs
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(1) as ex:
            fut = ex.submit(draw, firsts[0]) if firsts else None
            for idx, first in enumerate(firsts):
                mats = fut.result()
                ctx.noise_model = model
                reset_state(ctx)
                run_circuit(ctx, circuit, noise_matrices=mats)
                if idx + 1 < len(firsts):
                    fut = ex.submit(draw, firsts[idx + 1])
                vals = np.atleast_1d(np.asarray(observe(ctx), dtype=np.float64))
                count = min(S, trajectories - first)
                values[first:first + count] = vals[:count]
    finally:
        ctx.noise_model = saved
    return ref, values


def noise_ensemble_csv(values, reference: float) -> str:
    """The noise-ensemble report (cli.py:329-334): running mean per count."""
    values = np.asarray(values, dtype=np.float64)
    running = np.cumsum(values) / np.arange(1, values.size + 1)
    lines = ["trajectories,running_mean,reference"]
    lines.extend(f"{i + 1},{float(running[i])!r},{reference!r}" for i in range(values.size))
    return "\n".join(lines) + "\n"


def apply_gate_pool(ctx: RankContext, gate, param_table=None) -> None:
    """One gate on every pool state; state s binds param_table[s]
    (runtime.py:175-189).  A pool context sends the per-state values as one
    table; a single-state context binds its own entry (state_offset)."""
    if param_table is None:
        apply_gate(ctx, gate)
        return
    vals = np.asarray(param_table, dtype=np.float64)
    if ctx.is_idle:
        return
    if ctx.pool is None:
        from dataclasses import replace
        apply_gate(ctx, replace(gate, param=float(vals[ctx.state_offset])))
        return
    if vals.shape != (ctx.num_states,):
        raise ValueError(f"parameter table has {vals.size} entries for {ctx.num_states} states")
    q = ctx.queue
    if gate.kind == "diagcost":
        q.cut_phase(gate.graph, vals)
    elif gate.kind in gates_mod.ROTATION_GATES:
        q.one_qubit(gate.qubits[0], gates_mod.rotation_batch(gate.kind, vals))
    elif gate.kind == "cphase":
        q.controlled(gate.qubits[0], gate.qubits[1],
                     np.stack([gates_mod.cphase(float(v)) for v in vals]))
    else:
        raise ValueError(f"gate kind {gate.kind} takes no parameter")


def pool_sum(ctx: RankContext, value) -> float:
    """Incoherent sum over the pool's states in the reference's fixed tree
    order (runtime.py:230-232, pool.py:131-155); `value` is the per-state
    array a pool context's measurements return (or one state's scalar)."""
    return sv.tree_sum_values(np.atleast_1d(np.asarray(value, dtype=np.float64)))


def pool_gather(ctx: RankContext, value, num_groups: int | None = None) -> np.ndarray:
    """Per-state values in state order (runtime.py:235-236)."""
    arr = np.atleast_1d(np.asarray(value, dtype=np.float64))
    return arr if num_groups is None else arr[:num_groups]


def _queue_fixed(q: GateQueue, gate) -> None:
    if gate.kind == "diagcost":
        q.cut_phase(gate.graph, _angle(gate))
    elif gate.kind in ("cx", "cz", "cphase", "cu"):
        q.controlled(gate.qubits[0], gate.qubits[1], _matrix_for(gate))
    else:
        q.one_qubit(gate.qubits[0], _matrix_for(gate))


def split_pool(num_states: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [first, first+count) of pool states owned by `rank`
    (the contiguous-group rule of pool.build_pool, pool.py:118-128)."""
    base, extra = divmod(num_states, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


# ---- SPMD driver and convenience entry -------------------------------------------------
def run_spmd(world_size: int, fn, timeout: float = 30.0, exchange_mode: str = "peer") -> list:
    """fn(comm) on one thread per rank (runtime.py:261-288)."""
    import threading

    fabric = dist.ThreadFabric(world_size, timeout=timeout, exchange_mode=exchange_mode)
    if world_size == 1:
        return [fn(fabric.endpoint(0))]
    results: list = [None] * world_size
    failures: list = []
    lock = threading.Lock()

    def worker(rank: int) -> None:
        try:
            results[rank] = fn(fabric.endpoint(rank))
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            with lock:
                failures.append((rank, exc))

    threads = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world_size)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if failures:
        failures.sort(key=lambda p: p[0])
        rank, exc = failures[0]
        raise RuntimeError(f"rank {rank} failed: {exc!r}") from exc
    return results


def simulate_circuit(circuit, num_ranks: int = 1, bindings: dict | None = None,
                     device: int = 0, fuse: bool = True, timeout: float = 30.0,
                     exchange_mode: str = "peer", remap: bool = False) -> np.ndarray:
    """Run a circuit over `num_ranks` emulated ranks and return the full state
    (runtime.py:291-302).  All emulated ranks share `device`."""

    def rank_fn(comm):
        ctx = make_context(comm, circuit.num_qubits, 1, device, fuse, remap)
        run_circuit(ctx, circuit, bindings)
        return gather_group_state(ctx)

    return run_spmd(num_ranks, rank_fn, timeout=timeout, exchange_mode=exchange_mode)[0]
