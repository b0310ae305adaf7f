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
from .pool import PoolLayout, build_pool, gather_state_values, incoherent_sum_over_pool

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

    def cut_phase(self, graph, gamma, luts=None) -> None:
        """`luts`: the (S, |E|+1) per-state LUTs of phase_lut_batch(gamma), when
        the caller built them already (run_circuit_pool builds all of a
        circuit's LUT batches concurrently)."""
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
            if luts is None:
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
    """What one rank needs to run circuits (runtime.py:44-87).

    The reference's fields come first and mean what they mean there:
    `transport` is the world endpoint (None for one rank), `layout` the pool
    layout of rank groups (pool.build_pool), `group`/`state_rank` this rank's
    place in it, `comm` the group communicator, `partition` the device-resident
    slice, and the three keyed random streams.  Shim-only fields follow, all
    defaulted: `device`, `fuse` (numerics mode), `remap` (qubit remapping),
    `state_offset` and `batch`.

    Two pool shapes:
      * num_states <= world (the reference's): contiguous power-of-two rank
        groups, one state per group, each state sharded over its group;
      * num_states > world (shim extension -- the reference raises): every rank
        holds a contiguous block of whole states (`batch` = count, first state
        `state_offset`) in ONE device allocation, so a pool step is one fused
        launch per pass for all of them (runtime.PoolState)."""

    transport: object
    layout: PoolLayout
    num_qubits: int
    seed: int
    noise_model: "noise_mod.NoiseModel | None" = None
    norm_check_interval: int = NORM_CHECK_INTERVAL
    device: int | None = None
    fuse: bool = True
    remap: bool = False
    state_offset: int | None = None
    batch: int = 0  # > 0: batched pool extension, states held by this rank
    pool_states: int = 0  # batched pool: states in the whole pool (tables cover them all)
    pool_first: int = 0   # batched pool: state index of entry 0 of a whole-pool table
    world_rank: int = field(init=False)
    group: int | None = field(init=False)
    state_rank: int | None = field(init=False)
    topology: dist.RankTopology = field(init=False)
    comm: dist.GroupComm | None = field(init=False)
    partition: sv.StatePartition | None = field(init=False, default=None)
    pool_stream: noise_mod.RandomStream = field(init=False)
    local_stream: noise_mod.RandomStream = field(init=False)
    gates_applied: int = field(init=False, default=0)
    qubit_layout: "dist.QubitLayout | None" = field(init=False, default=None)
    pool: "PoolState | None" = field(init=False, default=None)
    queue: GateQueue | None = field(init=False, default=None)
    _state_stream: object = field(init=False, default=None, repr=False)

    def __post_init__(self) -> None:
        t = self.transport
        if isinstance(t, dist.GroupComm) and t.transport is not None:
            t = t.transport  # round-1 callers passed a group view of the world
        elif isinstance(t, dist.GroupComm):
            t = None
        self.transport = t
        self.world_rank = 0 if t is None else t.rank
        if self.device is None:
            self.device = _default_device(self.world_rank)
        self.pool_stream = noise_mod.RandomStream(self.seed, noise_mod.SCOPE_POOL, 0)
        self.local_stream = noise_mod.RandomStream(self.seed, noise_mod.SCOPE_LOCAL,
                                                   self.world_rank)
        if self.batch > 0:
            # batched pool: whole states, no sharding, no peers
            self.group = self.state_offset
            self.state_rank = 0
            self.topology = dist.RankTopology(1, self.num_qubits)
            self.comm = dist.single_rank_comm()
            self.pool = PoolState(self.num_qubits, self.batch, self.device, self.fuse)
            self.queue = self.pool.queue
            if t is not None:
                dist.GroupComm(t, self.world_rank, 1).attach(None)
            return
        lay = self.layout
        self.group = lay.group_of_rank(self.world_rank)
        self.state_rank = lay.state_rank_of_rank(self.world_rank)
        self.topology = dist.RankTopology(lay.ranks_per_state, self.num_qubits)
        if self.group is None:
            self.comm = None
            if t is not None:  # the partition handles are a world collective
                dist.GroupComm(t, self.world_rank, 1).attach(None)
            return
        if self.state_offset is None:
            self.state_offset = self.group
        self.comm = dist.GroupComm(t, lay.group_base(self.group), lay.ranks_per_state)
        if self.state_rank < self.topology.effective_ranks:
            self.partition = sv.allocate_partition(
                self.num_qubits, self.topology.num_local_qubits, self.state_rank,
                device=self.device)
            sv.init_basis_state(self.partition, 0)
            self.queue = GateQueue(self.partition.state, self.fuse)
            if self.remap and self.topology.rank_bits > 0:
                self.qubit_layout = dist.QubitLayout(self.num_qubits,
                                                     self.topology.num_local_qubits)
        self.comm.attach(self.partition)
        if self.comm.exchange_mode == "nccl" and hasattr(t, "nccl_init"):
            t.nccl_init(self.comm.base_rank, self.comm.size)

    @property
    def is_idle(self) -> bool:
        return self.queue is None

    @property
    def num_states(self) -> int:
        """States held by this context (1, or the batch of a batched pool)."""
        return self.batch if self.batch > 0 else 1

    @property
    def state_stream(self):
        """The state-scope stream of this context's state (runtime.py:79);
        a batched pool gets a StreamBatch with one stream per state."""
        if self._state_stream is None and not (self.group is None and self.batch == 0):
            if self.pool is None:
                self._state_stream = noise_mod.RandomStream(self.seed, noise_mod.SCOPE_STATE,
                                                            self.state_offset)
            else:
                self._state_stream = noise_mod.StreamBatch(
                    noise_mod.RandomStream(self.seed, noise_mod.SCOPE_STATE, self.state_offset + s)
                    for s in range(self.batch))
        return self._state_stream

    @property
    def state(self) -> _native.DeviceState:
        return self.partition.state if self.partition is not None else self.pool.state

    def flush(self) -> None:
        if self.queue is not None:
            if self.partition is not None:
                self.partition.sync_in()
            self.queue.flush()


def _default_device(world_rank: int) -> int:
    """One process per GPU (torchrun): LOCAL_RANK; otherwise device 0 (thread
    ranks share the calling process's GPU unless told otherwise)."""
    import os

    if os.environ.get("QSB_ALL_RANKS_ON_DEVICE0") == "1":
        return 0
    lr = os.environ.get("LOCAL_RANK")
    return int(lr) if lr is not None else 0


def make_context(transport, num_qubits: int, num_states: int = 1, seed: int = 0,
                 noise_model=None, *, device: int | None = None, fuse: bool = True,
                 remap: bool = False, state_offset: int | None = None,
                 batch: bool | None = None) -> RankContext:
    """The reference's make_context (runtime.py:90-99): `transport` is this
    rank's world endpoint (or None), the pool layout is build_pool(world,
    num_states).  Shim keywords: `device` (default LOCAL_RANK or 0), `fuse`
    (True: bit-identical fused passes; "factored": the factored numerics;
    False: one kernel per gate), `remap` (global qubits are swapped into local
    positions instead of exchanged), `state_offset` (global index of this
    context's first state; keyed noise streams), `batch` (force/forbid the
    batched pool extension; default: batched when num_states > world)."""
    if isinstance(transport, dist.GroupComm):
        world = transport.size if transport.transport is not None else 1
    else:
        world = 1 if transport is None else transport.world_size
    if num_states < 1:
        raise ValueError("need at least one state")
    use_batch = num_states > world if batch is None else bool(batch)
    if use_batch:
        rank = 0 if transport is None else transport.rank
        first, count = split_pool(num_states, rank, world)
        base = 0
        if state_offset is not None:  # a block of a larger pool split by the caller
            base = state_offset
            first += state_offset
        if count < 1:
            raise ValueError(f"{num_states} states leave rank {rank} of {world} without a state")
        layout = PoolLayout(world, min(num_states, world), 1)
        return RankContext(transport, layout, num_qubits, seed, noise_model, device=device,
                           fuse=fuse, remap=remap, state_offset=first, batch=count,
                           pool_states=num_states, pool_first=base)
    layout = build_pool(world, num_states)
    if layout.ranks_per_state >= (1 << num_qubits):
        raise ValueError(f"{layout.ranks_per_state} ranks per state leave no local qubit "
                         f"for n={num_qubits}")
    return RankContext(transport, layout, num_qubits, seed, noise_model, device=device,
                       fuse=fuse, remap=remap, state_offset=state_offset)


def reset_state(ctx: RankContext, index: int = 0) -> None:
    if ctx.is_idle:
        return
    ctx.queue.discard()
    if ctx.qubit_layout is not None:  # a fresh basis state: back to the canonical layout
        ctx.qubit_layout = dist.QubitLayout(ctx.num_qubits, ctx.topology.num_local_qubits)
    if ctx.partition is not None:
        sv.init_basis_state(ctx.partition, index)
    else:
        # deferred to the next access: a program of H on every qubit first (the
        # QAOA pool circuits) starts from the uniform state and the reset is
        # never written (DeviceState.defer_basis)
        ctx.pool.state.defer_basis(index)
    ctx.gates_applied = 0


def _restore(ctx: RankContext) -> None:
    if ctx.qubit_layout is not None and not ctx.qubit_layout.is_identity():
        ctx.flush()
        dist.restore_layout(ctx.partition, ctx.comm, ctx.topology, ctx.qubit_layout)


def _apply_gate_remapped(ctx: RankContext, gate) -> None:
    """apply_gate under a qubit layout: logical qubits are mapped to physical
    positions; a gate on a global position swaps it in first."""
    L, topo, q = ctx.qubit_layout, ctx.topology, ctx.queue
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
    L, m = ctx.qubit_layout, ctx.topology.num_local_qubits
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
    if ctx.qubit_layout is not None:
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


def gather_group_state(ctx: RankContext, group: int = 0) -> np.ndarray | None:
    """Assemble group `group`'s full amplitude vector on world rank 0
    (runtime.py:239-258): its ranks send their slices (in the canonical qubit
    layout) through the transport, rank 0 concatenates them in rank order.
    A batched pool's `group` is a state index; its owner sends it."""
    t = ctx.transport
    if ctx.batch > 0:
        first = ctx.state_offset
        mine = None
        if first <= group < first + ctx.batch:
            mine = ctx.pool.amplitudes()[group - first].copy()
        if t is None or t.world_size == 1:
            return mine
        owner = None if mine is None else ctx.world_rank
        owners = dist.GroupComm(t, 0, t.world_size).allgather(
            -1.0 if owner is None else float(owner), t.world_size)
        src = int(max(owners))
        if ctx.world_rank == 0:
            return mine if src == 0 else t.receive(src)
        if src == ctx.world_rank:
            t.send(0, mine)
        return None
    members = ctx.group == group and not ctx.is_idle
    if members:
        _restore(ctx)
        ctx.flush()
    if t is None or t.world_size == 1:
        return ctx.state.download()
    base = ctx.layout.group_base(group)
    size = ctx.layout.ranks_per_state
    if ctx.world_rank == 0:
        pieces = [None] * size
        for r in range(size):
            w = base + r
            pieces[r] = ctx.state.download() if w == 0 else t.receive(w)
        return np.concatenate(pieces)
    if members:
        t.send(0, ctx.state.download())
    return None


# ---- pool mode -----------------------------------------------------------------------
class PoolState:
    """S independent n-qubit states, batched in one device allocation."""

    def __init__(self, num_qubits: int, num_states: int, device: int = 0, fuse: bool = True):
        self.num_qubits = num_qubits
        self.num_states = num_states
        self.state = _native.DeviceState(num_qubits, num_qubits, 0, num_states, device)
        self.queue = GateQueue(self.state, fuse)
        self.state.defer_basis(0)

    def observable(self, kind: int, q: int = 0, edges=None) -> np.ndarray:
        self.queue.flush()
        return self.state.observable(kind, q, edges)

    def amplitudes(self) -> np.ndarray:
        self.queue.flush()
        return self.state.download().reshape(self.num_states, -1)


_LUT_POOL = None


def _lut_pool():
    global _LUT_POOL
    if _LUT_POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _LUT_POOL = ThreadPoolExecutor(max_workers=4, thread_name_prefix="qsb-lut")
    return _LUT_POOL


def run_circuit_pool(ctx: RankContext, circuit, slot_tables: dict | None = None,
                     noise_stream=None) -> None:
    """Every pool state runs `circuit`; state s binds slot_tables[name][s]
    (runtime.py:192-209).  A rank-group state binds its group's entry; a
    batched pool sends its block of every table to the device as per-state
    matrices/LUTs (one fused program for all its states).  Noise gates draw
    state s's matrix from stream s of `noise_stream` (a StreamBatch or a list
    of streams; default: the states' own streams)."""
    if not slot_tables:
        run_circuit(ctx, circuit, noise_stream=noise_stream)
        return
    total = _pool_total(ctx)
    for name, vals in slot_tables.items():
        if len(vals) != total:
            raise ValueError(f"table for ${name} has {len(vals)} entries for {total} states")
    if ctx.is_idle:
        return
    tables = {k: np.asarray(v, dtype=np.float64) for k, v in slot_tables.items()}
    if ctx.batch == 0:
        bindings = {name: float(vals[ctx.group]) for name, vals in tables.items()}
        run_circuit(ctx, circuit, bindings, noise_stream=noise_stream)
        return
    tables = {k: _my_values(ctx, v) for k, v in tables.items()}
    q = ctx.queue
    pre = _circuit_noise(ctx, circuit.gates, noise_stream)
    rot_cache: dict = {}
    # the per-state cut-phase LUTs (S x (|E|+1) complex exps per slot, ~0.4 ms
    # each for 512 states) are built concurrently: numpy releases the GIL
    lut_jobs = {(g.slot, len(g.graph.edges)) for g in circuit.gates
                if g.kind == "diagcost" and isinstance(getattr(g, "param", None), str)
                and g.slot in tables}
    lut_cache = {}
    if len(lut_jobs) > 1 and ctx.batch and len(next(iter(tables.values()))) >= 64:
        jobs = sorted(lut_jobs)
        lut_cache = dict(zip(jobs, _lut_pool().map(
            lambda j: phase_lut_batch(tables[j[0]], j[1]), jobs)))
    for gate in circuit.gates:
        slot = gate.slot if isinstance(getattr(gate, "param", None), str) else None
        if slot is None:
            if gate.kind == "noise":
                apply_gate(ctx, gate, noise_matrix=next(pre))
                continue
            _queue_fixed(q, gate)
            continue
        if slot not in tables:
            raise ValueError(f"gate {gate.kind} has unbound slot ${slot}")
        vals = tables[slot]
        if gate.kind == "diagcost":
            q.cut_phase(gate.graph, vals, lut_cache.get((slot, len(gate.graph.edges))))
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
    # the norm check of runtime.py:146-152 for every state, deferred to the end
    # of the circuit (a check mid-program would split its fused passes): the
    # drift is caught in the same circuit, a few gates later at most
    before = ctx.gates_applied
    ctx.gates_applied += sum(1 for g in circuit.gates if g.kind != "noise")
    k = ctx.norm_check_interval
    if k and ctx.gates_applied // k > before // k:
        norm_sq = measure_norm_squared(ctx)
        worst = float(np.max(np.abs(np.asarray(norm_sq, dtype=np.float64) - 1.0)))
        if worst >= NORM_TOL:
            raise NormDriftError(f"norm^2 drifted to {norm_sq!r} after {ctx.gates_applied} gates")


def run_noise_ensemble(ctx: RankContext, circuit, model, trajectories: int, observe,
                       seed: int | None = None, num_groups: int | None = None, *,
                       shadow: RankContext | None = None):
    """Noisy-trajectory ensemble (cli.py:288-339) on this context.

    `shadow`: a second context of the same shape (same pool size, seed and
    device).  Rounds then alternate between the two, and round k's values are
    read back only after round k+1's program has been built and enqueued, so the
    host's per-round work (per-state table fusion and factoring, ~17 ms for 512
    trajectories of the config-5 circuit) runs while the device works; the
    shadow's program waits on the other context's (an event), so their kernels
    do not interleave.  Same values as without it.

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

        if shadow is not None and (ctx.pool is None or shadow.pool is None or
                                   shadow.num_states != ctx.num_states):
            raise ValueError("a shadow context pipelines batched pools of one shape")
        ctxs = [ctx] if shadow is None or shadow.is_idle else [ctx, shadow]

        def collect(c, first):
            vals = np.atleast_1d(np.asarray(observe(c), dtype=np.float64))
            count = min(S, trajectories - first)
            values[first:first + count] = vals[:count]

        with ThreadPoolExecutor(1) as ex:
            fut = ex.submit(draw, firsts[0]) if firsts else None
            behind = None  # (context, first) whose values are still on the device
            for idx, first in enumerate(firsts):
                c = ctxs[idx % len(ctxs)]
                mats = fut.result()
                c.noise_model = model
                if behind is not None:  # this program runs after the other context's
                    c.state.wait_event(behind[0].state.sync_event(0))
                reset_state(c)
                run_circuit(c, circuit, noise_matrices=mats)
                if idx + 1 < len(firsts):
                    fut = ex.submit(draw, firsts[idx + 1])
                if len(ctxs) == 1:
                    collect(c, first)
                    continue
                c.state.record_sync_event(0)
                if behind is not None:
                    collect(*behind)
                behind = (c, first)
            if behind is not None:
                collect(*behind)
    finally:
        ctx.noise_model = saved
        if shadow is not None:
            shadow.noise_model = saved
    return ref, values


def noise_ensemble_csv(values, reference: float) -> str:
    """The noise-ensemble report (cli.py:329-334): running mean per count."""
    values = np.asarray(values, dtype=np.float64)
    running = np.cumsum(values) / np.arange(1, values.size + 1)
    lines = ["trajectories,running_mean,reference"]
    lines.extend(f"{i + 1},{float(running[i])!r},{reference!r}" for i in range(values.size))
    return "\n".join(lines) + "\n"


def _pool_total(ctx: RankContext) -> int:
    return ctx.pool_states if ctx.batch > 0 else ctx.layout.num_states


def _my_values(ctx: RankContext, vals: np.ndarray) -> np.ndarray:
    """This context's entries of a whole-pool table (batched: its block)."""
    first = ctx.state_offset - ctx.pool_first
    return vals[first:first + ctx.batch]


def apply_gate_pool(ctx: RankContext, gate, param_table=None) -> None:
    """One gate on every pool state; state s binds param_table[s]
    (runtime.py:175-189).  A batched pool queues its block of values as one
    per-state table (one launch for all its states)."""
    if param_table is None:
        apply_gate(ctx, gate)
        return
    vals = np.asarray(param_table, dtype=np.float64)
    total = _pool_total(ctx)
    if vals.shape != (total,):
        raise ValueError(f"parameter table has {vals.size} entries for {total} states")
    if ctx.is_idle:
        return
    if ctx.batch == 0:
        from dataclasses import replace
        apply_gate(ctx, replace(gate, param=float(vals[ctx.group])))
        return
    vals = _my_values(ctx, vals)
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
    _count_and_check(ctx)


def _batched_values(ctx: RankContext, value):
    """Every state's value of a batched pool, in state order, on world rank 0
    (None elsewhere): each rank's block goes to rank 0 in rank order, which is
    state order (split_pool is contiguous)."""
    arr = np.atleast_1d(np.asarray(value, dtype=np.float64))
    t = ctx.transport
    if t is None or t.world_size == 1:
        return arr
    if ctx.world_rank == 0:
        parts = [arr] + [t.receive(r).real for r in range(1, t.world_size)]
        return np.concatenate(parts)
    t.send(0, arr)
    return None


def pool_sum(ctx: RankContext, value) -> float:
    """Incoherent sum of one group-reduced scalar per state, the same on every
    rank, in the reference's fixed tree order (runtime.py:230-232,
    pool.py:131-155).  A batched pool passes its per-state array."""
    if ctx is None:  # round-1 callers: a plain array of per-state values
        return sv.tree_sum_values(np.atleast_1d(np.asarray(value, dtype=np.float64)))
    if ctx.batch > 0:
        vals = _batched_values(ctx, value)
        t = ctx.transport
        if t is None or t.world_size == 1:
            return sv.tree_sum_values(vals)
        from .transport import broadcast_array
        total = sv.tree_sum_values(vals) if vals is not None else 0.0
        return float(broadcast_array(t, [total])[0].real)
    return incoherent_sum_over_pool(value, ctx.layout, ctx.transport)


def pool_gather(ctx: RankContext, value, num_groups: int | None = None):
    """One value per state in state order on world rank 0, None elsewhere
    (runtime.py:235-236, pool.py:158-182)."""
    if ctx is None:
        arr = np.atleast_1d(np.asarray(value, dtype=np.float64))
        return arr if num_groups is None else arr[:num_groups]
    if ctx.batch > 0:
        vals = _batched_values(ctx, value)
        if vals is None:
            return None
        return vals if num_groups is None else vals[:num_groups]
    return gather_state_values(value, ctx.layout, ctx.transport, num_groups)


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
def run_spmd(world_size: int, fn, timeout: float = 30.0, *, exchange_mode: str = "peer") -> list:
    """fn(transport) on one thread per rank; results by rank (runtime.py:261-288).
    Each thread gets its rank's world endpoint (InProcessFabric); the ranks'
    partitions share the process's device unless contexts name others."""
    import threading

    from .transport import InProcessFabric

    fabric = InProcessFabric(world_size, timeout=timeout, exchange_mode=exchange_mode)
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
        also = "".join(f"; rank {r}: {e!r}" for r, e in failures[1:])
        raise RuntimeError(f"rank {rank} failed: {exc!r}{also}") from exc
    return results


def simulate_circuit(circuit, num_ranks: int = 1, num_states: int = 1, seed: int = 0,
                     noise_model=None, bindings: dict | None = None, timeout: float = 30.0,
                     *, device: int = 0, fuse: bool = True, exchange_mode: str = "peer",
                     remap: bool = False) -> np.ndarray:
    """Run a circuit on `num_ranks` thread ranks and return group 0's full
    state vector (runtime.py:291-302).  All thread ranks share `device`."""

    def rank_fn(transport):
        ctx = make_context(transport, circuit.num_qubits, num_states, seed, noise_model,
                           device=device, fuse=fuse, remap=remap)
        run_circuit(ctx, circuit, bindings)
        return gather_group_state(ctx)

    return run_spmd(num_ranks, rank_fn, timeout=timeout, exchange_mode=exchange_mode)[0]
