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
reference requires):
  * ``single_rank_comm()``      one rank, no peers
  * ``ThreadFabric(P)``          P ranks as threads of one process (the
                                 reference's run_spmd model); partitions may
                                 live on one device (emulated ranks) or on
                                 several
  * ``TorchComm(...)``           one process per GPU over torch.distributed
                                 (control plane) + CUDA IPC peer mappings
"""
from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import _native
from . import statevector as sv

DEFAULT_CHUNK_AMPLITUDES = 1 << 26


class TransportTimeout(TimeoutError):
    """A collective partner never showed up (reference transport.py:41-42)."""


TransportError = _native.TransportError


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
    """Group-relative communicator for one distributed state."""

    rank: int = 0
    size: int = 1
    exchange_mode: str = "peer"

    def pair_barrier(self, partner: int) -> None:
        raise NotImplementedError

    def allgather(self, value: float, participants: int) -> list:
        """Values of ranks [0, participants) in rank order (caller is one of them)."""
        raise NotImplementedError

    def attach(self, partition) -> None:
        """Collective: make this rank's partition reachable by its peers."""

    def peer_pointer(self, partner: int) -> int:
        raise NotImplementedError

    def nccl_peer(self, partner: int) -> int:
        return partner


class _SingleComm(GroupComm):
    def pair_barrier(self, partner: int) -> None:
        raise TransportError("single-rank communicator has no peers")

    def allgather(self, value: float, participants: int) -> list:
        return [float(value)]


def single_rank_comm() -> GroupComm:
    return _SingleComm()


class ThreadFabric:
    """P ranks as threads of one process, like the reference's InProcessFabric
    + run_spmd (transport.py:118-154, runtime.py:261-288).  Partitions may sit
    on one GPU (emulated ranks: the exchange kernel of each rank touches a
    disjoint pair set, so no kernel ever waits on another) or on several."""

    def __init__(self, size: int, timeout: float = 30.0, exchange_mode: str = "peer"):
        self.size = size
        self.timeout = timeout
        self.exchange_mode = exchange_mode
        self._lock = threading.Lock()
        self._pair: dict = {}
        self._gather: dict = {}
        self._parts: dict = {}

    def endpoint(self, rank: int) -> "ThreadComm":
        return ThreadComm(self, rank)

    def _barrier(self, key, parties: int) -> threading.Barrier:
        with self._lock:
            b = self._pair.get(key)
            if b is None:
                b = self._pair[key] = threading.Barrier(parties)
            return b


class ThreadComm(GroupComm):
    def __init__(self, fabric: ThreadFabric, rank: int):
        self.fabric = fabric
        self.rank = rank
        self.size = fabric.size
        self.exchange_mode = fabric.exchange_mode

    def _wait(self, barrier: threading.Barrier) -> None:
        try:
            barrier.wait(timeout=self.fabric.timeout)
        except threading.BrokenBarrierError:
            raise TransportTimeout(f"rank {self.rank}: partner never arrived") from None

    def pair_barrier(self, partner: int) -> None:
        key = ("pair", min(self.rank, partner), max(self.rank, partner))
        self._wait(self.fabric._barrier(key, 2))

    def allgather(self, value: float, participants: int) -> list:
        f = self.fabric
        b = f._barrier(("gather", participants), participants)
        with f._lock:
            f._gather.setdefault(participants, {})[self.rank] = float(value)
        self._wait(b)
        with f._lock:
            vals = [f._gather[participants][r] for r in range(participants)]
        self._wait(b)
        return vals

    def attach(self, partition) -> None:
        with self.fabric._lock:
            self.fabric._parts[self.rank] = partition

    def peer_pointer(self, partner: int) -> int:
        with self.fabric._lock:
            part = self.fabric._parts.get(partner)
        if part is None:
            raise TransportError(f"rank {partner} has no attached partition")
        return part.state.device_ptr()


class TorchComm(GroupComm):
    """One process per GPU.  torch.distributed carries the control plane
    (barriers, scalar gathers, IPC handles; any backend -- gloo works on
    CPU); the data plane is the peer kernel over CUDA IPC mappings or NCCL
    inside libqsb200."""

    def __init__(self, group=None, exchange_mode: str = "peer"):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.exchange_mode = exchange_mode
        self._handles: list | None = None
        self._peers: dict = {}
        self._state = None

    def _global(self, r: int) -> int:
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def pair_barrier(self, partner: int) -> None:
        import torch

        t = torch.zeros(1)
        g = self._global(partner)
        if self.rank < partner:
            self.dist.send(t, g, group=self.group)
            self.dist.recv(t, g, group=self.group)
        else:
            self.dist.recv(t, g, group=self.group)
            self.dist.send(t, g, group=self.group)

    def allgather(self, value: float, participants: int) -> list:
        import torch

        # every group member joins the gather; ranks beyond `participants`
        # contribute nothing and the caller ignores them
        t = torch.tensor([float(value)], dtype=torch.float64)
        out = [torch.zeros(1, dtype=torch.float64) for _ in range(self.size)]
        self.dist.all_gather(out, t, group=self.group)
        return [float(x.item()) for x in out[:participants]]

    def attach(self, partition) -> None:
        import ctypes

        self._state = partition.state if partition is not None else None
        mine = b""
        if self._state is not None:
            buf = (ctypes.c_ubyte * 64)()
            _native.call("qs_state_ipc_handle", self._state.handle, buf)
            mine = bytes(buf)
        handles = [None] * self.size
        self.dist.all_gather_object(handles, mine, group=self.group)
        self._handles = handles
        if self.exchange_mode == "nccl" and self._state is not None:
            ident = [None]
            if self.rank == 0:
                buf = (ctypes.c_ubyte * 128)()
                _native.call("qs_nccl_unique_id", buf)
                ident = [bytes(buf)]
            self.dist.broadcast_object_list(ident, src=self._global(0), group=self.group)
            idb = (ctypes.c_ubyte * 128).from_buffer_copy(ident[0])
            _native.call("qs_comm_init", self._state.handle, idb, self.size, self.rank)

    def peer_pointer(self, partner: int) -> int:
        import ctypes

        if partner not in self._peers:
            if not self._handles or not self._handles[partner]:
                raise TransportError(f"rank {partner} has no attached partition")
            buf = (ctypes.c_ubyte * 64).from_buffer_copy(self._handles[partner])
            p = ctypes.c_void_p()
            _native.call("qs_peer_open", self._state.handle, buf, ctypes.byref(p))
            self._peers[partner] = p.value
        return self._peers[partner]


# ---- gates --------------------------------------------------------------------------
def _exchange_pairs(partition: sv.StatePartition, comm: GroupComm, q: int, u,
                    topology: RankTopology, control_local: int | None = None,
                    chunk: int = DEFAULT_CHUNK_AMPLITUDES) -> None:
    """Gate on global qubit q with the partner at rank distance 2^(q-m)
    (distribution.py:121-178).  The barriers order the partner's previous
    kernels before ours and ours before its next ones."""
    m = topology.num_local_qubits
    d = 1 << (q - m)
    partner = comm.rank ^ d
    is_lower = (comm.rank & d) == 0
    mat = np.ascontiguousarray(np.asarray(u, dtype=np.complex128))
    st = partition.sync_in()
    ctrl = -1 if control_local is None else int(control_local)
    st.synchronize()
    comm.pair_barrier(partner)
    if comm.exchange_mode == "nccl":
        _native.call("qs_exchange_gate_nccl", st.handle, comm.nccl_peer(partner),
                     1 if is_lower else 0, _native.dptr(mat), ctrl, int(chunk))
    else:
        _native.call("qs_exchange_gate_peer", st.handle, comm.peer_pointer(partner),
                     1 if is_lower else 0, _native.dptr(mat), ctrl)
    comm.pair_barrier(partner)


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
    st = partition.sync_in()
    st.synchronize()
    comm.pair_barrier(partner)
    _native.call("qs_swap_qubits_peer", st.handle, comm.peer_pointer(partner), l, bit)
    comm.pair_barrier(partner)
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
