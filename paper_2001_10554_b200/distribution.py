"""Rank/offset index math, the global-qubit exchange and controlled-gate
routing -- the drop-in for qpool.distribution (reference
pkg/src/qpool/distribution.py).

The routing decisions are the reference's (distribution.py:181-230); what
changes is the data movement.  A gate on a global qubit is ONE fused CUDA
kernel per partner rank (k_exchange_peer in csrc/exchange_kernels.cu): each
rank reads its partner's half of the shared pairs over NVLink peer memory,
applies the 2x2 and writes both members back, so transfer and arithmetic
overlap load by load.  The reference's own three-step half-buffer scheme
(Fig. 3, distribution.py:121-178) is kept as ``exchange_mode="nccl"``:
chunked, double-buffered NCCL send/recv with the step-2 update pipelined
against the transfers.

Communicators (all collective calls in the same order on every rank, as the
reference requires): ``GroupComm(transport, base_rank, size)`` is the
reference's group-relative view of a world endpoint (transport.py):
  * ``single_rank_comm()``           one rank, no peers
  * ``InProcessFabric(P)`` endpoints P ranks as threads of one process (the
                                     reference's run_spmd model); partitions
                                     may live on one device (emulated ranks)
                                     or on several
  * ``TorchTransport()``             one process per GPU over
                                     torch.distributed (control plane) + CUDA
                                     IPC peer mappings and events
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from . import statevector as sv
from .transport import (InProcessFabric, TorchTransport, TransportError,  # noqa: F401
                        TransportTimeout)

DEFAULT_CHUNK_AMPLITUDES = 1 << 26


@dataclass(frozen=True)
class RankTopology:
    """Group-level rank structure for one distributed state (distribution.py:27-57)."""

    total_ranks: int
    num_qubits: int

    def __post_init__(self) -> None:
        if self.total_ranks < 1:
            raise ValueError("need at least one rank")
        if self.num_local_qubits < 1:
            raise ValueError(
                f"{self.total_ranks} ranks leave no local qubit for n={self.num_qubits}")

    @property
    def rank_bits(self) -> int:
        return self.total_ranks.bit_length() - 1

    @property
    def effective_ranks(self) -> int:
        return 1 << self.rank_bits

    @property
    def num_local_qubits(self) -> int:
        return self.num_qubits - self.rank_bits

    def is_local(self, q: int) -> bool:
        if not (0 <= q < self.num_qubits):
            raise ValueError(f"qubit {q} out of range for n={self.num_qubits}")
        return q < self.num_local_qubits


def rank_and_offset(index: int, topology: RankTopology) -> tuple[int, int]:
    if not (0 <= index < (1 << topology.num_qubits)):
        raise ValueError(f"index {index} out of range")
    m = topology.num_local_qubits
    return index >> m, index & ((1 << m) - 1)


def exchange_partner(rank: int, q: int, topology: RankTopology) -> int:
    if topology.is_local(q):
        raise ValueError(f"qubit {q} is local; no exchange partner")
    return rank ^ (1 << (q - topology.num_local_qubits))


# ---- routing (pure functions, tested on CPU) --------------------------------------
def route_one_qubit(rank: int, topology: RankTopology, q: int):
    """('idle',) | ('local',) | ('exchange', partner, is_lower) -- distribution.py:181-192."""
    if not (0 <= q < topology.num_qubits):
        raise ValueError(f"qubit {q} out of range for n={topology.num_qubits}")
    if rank >= topology.effective_ranks:
        return ("idle",)
    if topology.is_local(q):
        return ("local",)
    d = 1 << (q - topology.num_local_qubits)
    return ("exchange", rank ^ d, (rank & d) == 0)


def route_controlled(rank: int, topology: RankTopology, control: int, target: int):
    """Four-case routing of distribution.py:195-230:
    ('idle',) | ('skip',) | ('local_controlled',) | ('local_one_qubit',) |
    ('exchange', partner, is_lower, control_local_or_None)."""
    n, m = topology.num_qubits, topology.num_local_qubits
    if control == target:
        raise ValueError("control and target must differ")
    for q in (control, target):
        if not (0 <= q < n):
            raise ValueError(f"qubit {q} out of range for n={n}")
    if rank >= topology.effective_ranks:
        return ("idle",)
    c_local, t_local = control < m, target < m
    if c_local and t_local:
        return ("local_controlled",)
    if not c_local:
        if not (rank >> (control - m)) & 1:
            return ("skip",)
        if t_local:
            return ("local_one_qubit",)
        d = 1 << (target - m)
        return ("exchange", rank ^ d, (rank & d) == 0, None)
    d = 1 << (target - m)
    return ("exchange", rank ^ d, (rank & d) == 0, control)


# ---- communicators ----------------------------------------------------------------
class GroupComm:
    """Group-relative view of a world endpoint for one state group
    (distribution.py:75-98): group ranks are the world ranks
    [base_rank, base_rank + size) and every peer is addressed group-relative.

    Beyond the reference's send/receive it carries the device plane of the
    exchange: pairwise handshakes that order one rank's exchange kernel after
    its partner's earlier work through CUDA events (no host stream sync),
    rank-ordered scalar gathers, and the partner's peer-memory pointer."""

    def __init__(self, transport, base_rank: int, size: int):
        if size > 1 and transport is None:
            raise ValueError("multi-rank group needs a transport")
        self.transport = transport
        self.base_rank = base_rank
        self.size = size
        self.rank = 0 if transport is None else transport.rank - base_rank
        if not (0 <= self.rank < size):
            raise ValueError(
                f"world rank {transport.rank} outside group [{base_rank}, {base_rank + size})")
        self.exchange_mode = getattr(transport, "exchange_mode", "peer")

    # the reference's point-to-point calls
    def send(self, dest: int, payload, tag: int = 0) -> None:
        self.transport.send(self.base_rank + dest, payload, tag=tag)

    def receive(self, src: int):
        return self.transport.receive(self.base_rank + src)

    # device plane
    def _need_peers(self) -> None:
        if self.transport is None or self.size == 1:
            raise TransportError("single-rank communicator has no peers")

    def pair_barrier(self, partner: int) -> None:
        self._need_peers()
        self.transport._dp_pair_barrier(self.base_rank + self.rank, self.base_rank + partner)

    def allgather(self, value: float, participants: int) -> list:
        """Values of group ranks [0, participants) in rank order (the caller is one)."""
        if self.transport is None or participants == 1:
            return [float(value)]
        return self.transport._dp_allgather(value, self.base_rank, participants)

    def attach(self, partition) -> None:
        """Collective over the world endpoint: make this rank's partition reachable."""
        if self.transport is not None:
            self.transport._dp_attach(partition)

    def peer_pointer(self, partner: int) -> int:
        self._need_peers()
        return self.transport._dp_peer_pointer(self.base_rank + partner)

    def peer_events(self, partner: int) -> tuple:
        self._need_peers()
        return self.transport._dp_peer_events(self.base_rank + partner)

    def nccl_peer(self, partner: int) -> int:
        return partner

    def account_exchange(self, messages: int, amplitudes: int) -> None:
        """Count an exchange in the reference's TransportCounters terms."""
        if self.transport is not None:
            self.transport.counters.messages_sent += messages
            self.transport.counters.amplitudes_sent += amplitudes


def single_rank_comm() -> GroupComm:
    return GroupComm(None, 0, 1)


def world_comm(transport) -> GroupComm:
    """The whole world as one group (a transport, a GroupComm, or None)."""
    if isinstance(transport, GroupComm):
        return transport
    if transport is None:
        return single_rank_comm()
    return GroupComm(transport, 0, transport.world_size)


# Names of round 1, kept for callers: the thread fabric is the transport's
# InProcessFabric; TorchComm is the torch.distributed world endpoint.
ThreadFabric = InProcessFabric
TorchComm = TorchTransport


# ---- gates --------------------------------------------------------------------------
def _ordered_peer_op(partition, comm: GroupComm, partner: int, launch) -> None:
    """Run `launch(state, peer_pointer)` -- a kernel that reads and writes the partner's
    slice -- ordered against the partner's work without a host stream sync:
    each side records its `pre` event, the pair meets on the host (so both
    records are enqueued), each stream waits on the partner's `pre`, launches,
    records `post`, meets again, and waits on the partner's `post` before its
    own next kernel.  The host never blocks on the GPU; the exchange queues
    behind the local passes and the next passes queue behind it."""
    comm.transport._dp_ensure(partition)
    st = partition.sync_in()
    st.record_sync_event(0)
    comm.pair_barrier(partner)
    # after the first meeting: the partner has attached and recorded `pre`
    pre, post = comm.peer_events(partner)
    st.wait_event(pre)
    launch(st, comm.peer_pointer(partner))
    st.record_sync_event(1)
    comm.pair_barrier(partner)
    st.wait_event(post)


def _exchange_pairs(partition: sv.StatePartition, comm: GroupComm, q: int, u,
                    topology: RankTopology, control_local: int | None = None,
                    chunk: int = DEFAULT_CHUNK_AMPLITUDES) -> None:
    """Gate on global qubit q with the partner at rank distance 2^(q-m)
    (distribution.py:121-178).  Accounted like the reference's Fig. 3 scheme:
    the half out and the updated half back, in chunks of `chunk` amplitudes."""
    m = topology.num_local_qubits
    d = 1 << (q - m)
    partner = comm.rank ^ d
    is_lower = (comm.rank & d) == 0
    mat = np.ascontiguousarray(np.asarray(u, dtype=np.complex128))
    ctrl = -1 if control_local is None else int(control_local)
    half = 1 << (m - 1)
    if chunk < 1:
        raise ValueError("chunk must be positive")
    comm.account_exchange(2 * (-(-half // chunk)), 2 * half)
    if comm.exchange_mode == "nccl":
        # NCCL orders the pair's grouped send/recv on the streams itself
        st = partition.sync_in()
        _native.call("qs_exchange_gate_nccl", st.handle, comm.nccl_peer(partner),
                     1 if is_lower else 0, _native.dptr(mat), ctrl, int(chunk))
        return
    _ordered_peer_op(partition, comm, partner, lambda st, peer: _native.call(
        "qs_exchange_gate_peer", st.handle, peer, 1 if is_lower else 0, _native.dptr(mat), ctrl))


# ---- qubit remapping -------------------------------------------
class QubitLayout:
    """Logical -> physical qubit positions of a distributed state.  Physical
    positions below m are local bits of the slice, the rest are rank bits.
    Every rank keeps an identical copy (all updates are collective)."""

    def __init__(self, num_qubits: int, num_local_qubits: int):
        self.n, self.m = num_qubits, num_local_qubits
        self.phys = list(range(num_qubits))
        self.log = list(range(num_qubits))
        self._next = 0
        self.recent: list = []  # physical positions in order of last use (most recent last)

    def use(self, phys: int) -> None:
        if self.recent and self.recent[-1] == phys:
            return
        if phys in self.recent:
            self.recent.remove(phys)
        self.recent.append(phys)

    def is_identity(self) -> bool:
        return self.phys == list(range(self.n))

    def swap(self, p1: int, p2: int) -> None:
        a, b = self.log[p1], self.log[p2]
        self.log[p1], self.log[p2] = b, a
        self.phys[a], self.phys[b] = p2, p1
        # recency follows the logical qubit: the positions trade places
        self.recent = [p2 if x == p1 else p1 if x == p2 else x for x in self.recent]

    def choose_slot(self, protected=()) -> int:
        """A local physical slot to trade for a global qubit: round-robin over
        the top local positions, skipping the ones the current gate uses."""
        for _ in range(self.m):
            slot = self.m - 1 - (self._next % self.m)
            self._next += 1
            if slot not in protected:
                return slot
        raise ValueError("no local slot available for the swap")


def swap_global_local(partition, comm: GroupComm, topology: RankTopology, layout: QubitLayout,
                      p: int, l: int) -> None:
    """Collective SWAP of physical global position p with local position l
    (half the slice crosses to the partner, k_swap_peer)."""
    m = topology.num_local_qubits
    if not (p >= m > l >= 0):
        raise ValueError(f"swap needs a global and a local position, got {p}, {l}")
    d = 1 << (p - m)
    partner = comm.rank ^ d
    bit = 1 if comm.rank & d else 0
    _ordered_peer_op(partition, comm, partner, lambda st, peer: _native.call(
        "qs_swap_qubits_peer", st.handle, peer, l, bit))
    comm.account_exchange(2, 1 << (m - 1))
    layout.swap(p, l)


def make_local(partition, comm: GroupComm, topology: RankTopology, layout: QubitLayout,
               q: int, protected=()) -> int:
    """Physical local position of logical qubit q, swapping it in if global."""
    p = layout.phys[q]
    if p < topology.num_local_qubits:
        return p
    slot = layout.choose_slot(protected)
    swap_global_local(partition, comm, topology, layout, p, slot)
    return slot


def restore_layout(partition, comm: GroupComm, topology: RankTopology,
                   layout: QubitLayout) -> None:
    """Bring every logical qubit back to its own physical position (collective)."""
    m, n = topology.num_local_qubits, topology.num_qubits
    for p in range(m, n):
        if layout.log[p] == p:
            continue
        lp = layout.phys[p]
        if lp >= m:  # logical p sits on another rank bit: bring it local first
            slot = layout.choose_slot(protected=())
            swap_global_local(partition, comm, topology, layout, lp, slot)
            lp = slot
        swap_global_local(partition, comm, topology, layout, p, lp)
    st = partition.sync_in()
    for l in range(m):
        if layout.log[l] == l:
            continue
        lp = layout.phys[l]
        _native.call("qs_swap_qubits_local", st.handle, l, lp)
        layout.swap(l, lp)


def apply_one_qubit_gate(partition, topology: RankTopology, comm: GroupComm, q: int, u,
                         chunk: int = DEFAULT_CHUNK_AMPLITUDES):
    """Collective one-qubit gate (distribution.py:181-192)."""
    comm = world_comm(comm)
    route = route_one_qubit(comm.rank, topology, q)
    if route[0] == "idle":
        return partition
    if route[0] == "local":
        return sv.apply_local_one_qubit_gate(partition, q, u)
    _exchange_pairs(partition, comm, q, u, topology, chunk=chunk)
    return partition


def apply_controlled_gate(partition, topology: RankTopology, comm: GroupComm, control: int,
                          target: int, u, chunk: int = DEFAULT_CHUNK_AMPLITUDES):
    """Controlled gate with the reference's four locality cases (distribution.py:195-230)."""
    comm = world_comm(comm)
    route = route_controlled(comm.rank, topology, control, target)
    kind = route[0]
    if kind in ("idle", "skip"):
        return partition
    if kind == "local_controlled":
        return sv.apply_local_controlled_gate(partition, control, target, u)
    if kind == "local_one_qubit":
        return sv.apply_local_one_qubit_gate(partition, target, u)
    _exchange_pairs(partition, comm, target, u, topology, control_local=route[3], chunk=chunk)
    return partition


def group_reduce_sum(partial: float, topology: RankTopology, comm: GroupComm) -> float:
    """Sum one scalar per rank with the association of sv.tree_sum over rank
    partials (the reference's recursive doubling, distribution.py:233-252)."""
    comm = world_comm(comm)
    if comm.rank >= topology.effective_ranks:
        return partial
    if topology.effective_ranks == 1:
        return float(partial)
    vals = comm.allgather(float(partial), topology.effective_ranks)
    return sv.tree_sum(np.asarray(vals, dtype=np.float64))


def measure_probability(partition, topology, comm, q: int) -> float:
    return group_reduce_sum(sv.get_probability(partition, q), topology, comm)


def measure_norm_squared(partition, topology, comm) -> float:
    return group_reduce_sum(sv.norm_squared(partition), topology, comm)


def measure_maxcut(partition, topology, comm, graph) -> float:
    return group_reduce_sum(sv.maxcut_expectation(partition, graph), topology, comm)


def measure_z(partition, topology, comm, q: int) -> float:
    return group_reduce_sum(sv.z_expectation(partition, q), topology, comm)
