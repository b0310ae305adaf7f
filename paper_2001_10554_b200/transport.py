"""Rank endpoints of the B200 core -- the drop-in for qpool.transport
(reference pkg/src/qpool/transport.py).

What a reference caller sees is kept: a world-level endpoint per rank with
``rank``, ``world_size``, ``counters`` (TransportCounters: messages and
amplitudes sent), point-to-point ``send``/``receive`` of complex128 payloads,
``barrier``, and ``TransportTimeout`` when a collective partner never shows
up.  What moves the amplitudes is not this module: a global-qubit gate is a
peer-memory kernel (or NCCL) inside libqsb200, and the endpoint only orders it
(pairwise handshakes) and accounts it in the reference's terms.

Two endpoint families:
  * ``InProcessFabric(P).endpoint(r)``  P ranks as threads of one process,
    the reference's run_spmd model (transport.py:118-154, runtime.py:261-288);
  * ``TorchTransport()``                one process per GPU over
    torch.distributed (gloo or NCCL) -- torchrun replaces the reference's TCP
    socket mesh, which is out of scope.

The device-plane hooks (``_dp_*``) are what distribution.GroupComm calls to
order exchange kernels across ranks: every rank's stream waits on its
partner's CUDA event instead of the host synchronising the stream.
"""
from __future__ import annotations

import queue
import threading
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import TransportError

DEFAULT_TIMEOUT = 30.0
TAG_DATA, TAG_EXCHANGE, TAG_RETURN, TAG_GATHER, TAG_BARRIER = 0, 1, 2, 3, 4


class TransportTimeout(TimeoutError):
    """A collective partner never showed up (reference transport.py:41-42)."""


@dataclass
class TransportCounters:
    """Messages and complex128 amplitudes this rank sent (transport.py:49-65).
    Exchange gates are accounted as the reference's Fig. 3 scheme would send
    them, whatever path moved the data."""

    messages_sent: int = 0
    amplitudes_sent: int = 0

    @property
    def bytes_sent(self) -> int:
        return 16 * self.amplitudes_sent

    def snapshot(self) -> "TransportCounters":
        return TransportCounters(self.messages_sent, self.amplitudes_sent)

    def delta(self, earlier: "TransportCounters") -> "TransportCounters":
        return TransportCounters(self.messages_sent - earlier.messages_sent,
                                 self.amplitudes_sent - earlier.amplitudes_sent)


def as_payload(values) -> np.ndarray:
    """Flat contiguous complex128 (the reference's wire type)."""
    return np.ascontiguousarray(np.asarray(values, dtype=np.complex128)).ravel()


class Transport:
    """World-level endpoint of one rank (transport.py:68-109)."""

    exchange_mode = "peer"

    def __init__(self, rank: int, world_size: int, timeout: float = DEFAULT_TIMEOUT):
        self.rank = rank
        self.world_size = world_size
        self.timeout = timeout
        self.counters = TransportCounters()

    def send(self, dest: int, payload, tag: int = 0) -> None:
        raise NotImplementedError

    def receive(self, src: int, timeout: float | None = None) -> np.ndarray:
        raise NotImplementedError

    def close(self) -> None:
        pass

    def _account(self, payload: np.ndarray) -> None:
        self.counters.messages_sent += 1
        self.counters.amplitudes_sent += int(payload.size)

    def barrier(self, ranks=None) -> None:
        """All of `ranks` (default: every rank) meet: gather at the lowest, release."""
        members = sorted(range(self.world_size) if ranks is None else ranks)
        if len(members) <= 1:
            return
        root = members[0]
        token = np.zeros(0, dtype=np.complex128)
        if self.rank == root:
            for r in members[1:]:
                self.receive(r)
            for r in members[1:]:
                self.send(r, token, tag=TAG_BARRIER)
        else:
            self.send(root, token, tag=TAG_BARRIER)
            self.receive(root)

    # whole-world group view: round-1 callers used the endpoint as a GroupComm
    def allgather(self, value: float, participants: int) -> list:
        return self._dp_allgather(value, 0, participants)

    def attach(self, partition) -> None:
        self._dp_attach(partition)

    def pair_barrier(self, partner: int) -> None:
        self._dp_pair_barrier(self.rank, partner)

    # ---- device plane (world-rank addressing; used by distribution.GroupComm) ----
    def _dp_pair_barrier(self, me: int, partner: int) -> None:
        raise NotImplementedError

    def _dp_ensure(self, partition) -> None:
        """Before an exchange: this rank's partition must be reachable."""
        raise NotImplementedError

    def _dp_allgather(self, value: float, base: int, participants: int) -> list:
        raise NotImplementedError

    def _dp_attach(self, partition) -> None:
        raise NotImplementedError

    def _dp_peer_pointer(self, world_rank: int) -> int:
        raise NotImplementedError

    def _dp_peer_events(self, world_rank: int) -> tuple:
        """(pre, post) exchange events of a rank's state, openable here."""
        raise NotImplementedError


# ---- threads of one process --------------------------------------------------------
class InProcessFabric:
    """Mailboxes and device-plane registries shared by P rank threads."""

    def __init__(self, world_size: int, timeout: float = DEFAULT_TIMEOUT,
                 exchange_mode: str = "peer"):
        self.world_size = world_size
        self.size = world_size
        self.timeout = timeout
        self.exchange_mode = exchange_mode
        self._queues = {(s, d): queue.Queue() for s in range(world_size)
                        for d in range(world_size)}
        self._lock = threading.Lock()
        self._barriers: dict = {}
        self._gather: dict = {}
        self._parts: dict = {}

    def queue(self, src: int, dest: int) -> queue.Queue:
        return self._queues[(src, dest)]

    def endpoint(self, rank: int) -> "InProcessTransport":
        return InProcessTransport(self, rank)

    def _barrier(self, key, parties: int) -> threading.Barrier:
        with self._lock:
            b = self._barriers.get(key)
            if b is None:
                b = self._barriers[key] = threading.Barrier(parties)
            return b


class InProcessTransport(Transport):
    def __init__(self, fabric: InProcessFabric, rank: int):
        super().__init__(rank, fabric.world_size, fabric.timeout)
        self.fabric = fabric
        self.exchange_mode = fabric.exchange_mode

    def send(self, dest: int, payload, tag: int = 0) -> None:
        payload = as_payload(payload)
        self._account(payload)
        self.fabric.queue(self.rank, dest).put(payload.copy())

    def receive(self, src: int, timeout: float | None = None) -> np.ndarray:
        try:
            return self.fabric.queue(src, self.rank).get(
                timeout=self.timeout if timeout is None else timeout)
        except queue.Empty:
            raise TransportTimeout(f"rank {self.rank}: no message from rank {src} "
                                   "(non-collective call or dead peer?)") from None

    def _wait(self, barrier: threading.Barrier) -> None:
        try:
            barrier.wait(timeout=self.fabric.timeout)
        except threading.BrokenBarrierError:
            raise TransportTimeout(f"rank {self.rank}: partner never arrived") from None

    def _dp_pair_barrier(self, me: int, partner: int) -> None:
        key = ("pair", min(me, partner), max(me, partner))
        self._wait(self.fabric._barrier(key, 2))

    def _dp_allgather(self, value: float, base: int, participants: int) -> list:
        f = self.fabric
        key = ("gather", base, participants)
        b = f._barrier(key, participants)
        with f._lock:
            f._gather.setdefault(key, {})[self.rank] = float(value)
        self._wait(b)
        with f._lock:
            vals = [f._gather[key][base + r] for r in range(participants)]
        self._wait(b)
        return vals

    def _dp_attach(self, partition) -> None:
        with self.fabric._lock:
            self.fabric._parts[self.rank] = partition

    def _dp_ensure(self, partition) -> None:
        # thread ranks share the process: registering is local (the reference's
        # callers never attach; their partitions join on first exchange)
        with self.fabric._lock:
            if self.fabric._parts.get(self.rank) is not partition:
                self.fabric._parts[self.rank] = partition

    def _part(self, world_rank: int):
        with self.fabric._lock:
            part = self.fabric._parts.get(world_rank)
        if part is None:
            raise TransportError(f"rank {world_rank} has no attached partition")
        return part

    def _dp_peer_pointer(self, world_rank: int) -> int:
        return self._part(world_rank).state.device_ptr()

    def _dp_peer_events(self, world_rank: int) -> tuple:
        st = self._part(world_rank).state
        return st.sync_event(0), st.sync_event(1)


# ---- one process per GPU (torchrun) ------------------------------------------------
class TorchTransport(Transport):
    """World endpoint over torch.distributed.  Payloads and the control plane
    go through the process group (gloo on CPU works); amplitudes of exchange
    gates go over CUDA-IPC peer mappings (or NCCL) inside libqsb200."""

    def __init__(self, exchange_mode: str = "peer", timeout: float = DEFAULT_TIMEOUT):
        import torch.distributed as dist

        self.dist = dist
        super().__init__(dist.get_rank(), dist.get_world_size(), timeout)
        self.exchange_mode = exchange_mode
        self._handles: list | None = None
        self._events: list | None = None
        self._peers: dict = {}
        self._peer_events: dict = {}
        self._state = None

    def send(self, dest: int, payload, tag: int = 0) -> None:
        payload = as_payload(payload)
        self._account(payload)
        self.dist.send_object_list([payload], dst=dest)

    def receive(self, src: int, timeout: float | None = None) -> np.ndarray:
        box = [None]
        self.dist.recv_object_list(box, src=src)
        return box[0]

    def _dp_pair_barrier(self, me: int, partner: int) -> None:
        import torch

        t = torch.zeros(1)
        if me < partner:
            self.dist.send(t, partner)
            self.dist.recv(t, partner)
        else:
            self.dist.recv(t, partner)
            self.dist.send(t, partner)

    def _dp_allgather(self, value: float, base: int, participants: int) -> list:
        """Group-local: members send to the group's first rank, which sends the
        rank-ordered values back (no collective over the whole world)."""
        import torch

        if participants == 1:
            return [float(value)]
        if self.rank == base:
            vals = [float(value)]
            for r in range(base + 1, base + participants):
                t = torch.zeros(1, dtype=torch.float64)
                self.dist.recv(t, r)
                vals.append(float(t.item()))
            out = torch.tensor(vals, dtype=torch.float64)
            for r in range(base + 1, base + participants):
                self.dist.send(out, r)
            return vals
        self.dist.send(torch.tensor([float(value)], dtype=torch.float64), base)
        out = torch.zeros(participants, dtype=torch.float64)
        self.dist.recv(out, base)
        return [float(x) for x in out.tolist()]

    def _dp_attach(self, partition) -> None:
        """World collective: every rank publishes its partition's IPC handles
        (memory and the two exchange events); idle ranks publish nothing."""
        import ctypes

        self._state = partition.state if partition is not None else None
        mine = (b"", b"", b"")
        if self._state is not None:
            buf = (ctypes.c_ubyte * 64)()
            _native.call("qs_state_ipc_handle", self._state.handle, buf)
            mine = (bytes(buf), self._state.sync_event_ipc(0), self._state.sync_event_ipc(1))
        table = [None] * self.world_size
        self.dist.all_gather_object(table, mine)
        self._handles = [t[0] for t in table]
        self._events = [(t[1], t[2]) for t in table]
        self._peers, self._peer_events = {}, {}

    def _dp_ensure(self, partition) -> None:
        if partition is None or self._state is not partition.state:
            raise TransportError("the partition was not attached collectively (make_context "
                                 "attaches it; across processes attach is a world collective)")

    def _dp_peer_pointer(self, world_rank: int) -> int:
        import ctypes

        if world_rank not in self._peers:
            if not self._handles or not self._handles[world_rank]:
                raise TransportError(f"rank {world_rank} has no attached partition")
            buf = (ctypes.c_ubyte * 64).from_buffer_copy(self._handles[world_rank])
            p = ctypes.c_void_p()
            _native.call("qs_peer_open", self._state.handle, buf, ctypes.byref(p))
            self._peers[world_rank] = p.value
        return self._peers[world_rank]

    def _dp_peer_events(self, world_rank: int) -> tuple:
        if world_rank not in self._peer_events:
            if not self._events or not self._events[world_rank][0]:
                raise TransportError(f"rank {world_rank} has no attached partition")
            self._peer_events[world_rank] = tuple(
                self._state.open_sync_event(h) for h in self._events[world_rank])
        return self._peer_events[world_rank]

    def nccl_init(self, base: int, size: int) -> None:
        """Collective over the world: one NCCL communicator per rank group
        [base, base + size) (its first rank makes the unique id)."""
        import ctypes

        ident = b""
        if self._state is not None and self.rank == base:
            buf = (ctypes.c_ubyte * 128)()
            _native.call("qs_nccl_unique_id", buf)
            ident = bytes(buf)
        table = [None] * self.world_size
        self.dist.all_gather_object(table, ident)
        if self._state is not None:
            idb = (ctypes.c_ubyte * 128).from_buffer_copy(table[base])
            _native.call("qs_comm_init", self._state.handle, idb, size, self.rank - base)


class SocketTransport(Transport):
    """The reference's TCP socket mesh (transport.py:207-340) is out of scope
    for the B200 core: one process per GPU runs under torchrun with
    TorchTransport instead (NVLink moves the amplitudes, not sockets)."""

    def __init__(self, rank: int, addresses, timeout: float = DEFAULT_TIMEOUT):
        raise TransportError("SocketTransport is not part of the B200 core; launch one "
                             "process per GPU with torchrun and use TorchTransport")


def parse_rendezvous(text: str) -> list:
    """`host:port` lines, one per rank (transport.py:157-169); kept for the
    reference's file format, the B200 core itself rendezvouses via torchrun."""
    out = []
    for raw in text.splitlines():
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        host, _, port = line.rpartition(":")
        if not host:
            raise TransportError(f"bad rendezvous line {line!r}")
        out.append((host, int(port)))
    if not out:
        raise TransportError("empty rendezvous file")
    return out


def write_rendezvous(path, num_ranks: int, host: str = "127.0.0.1") -> list:
    """Per-rank `host:port` file with free local ports (transport.py:177-192)."""
    import socket

    held, addrs = [], []
    for _ in range(num_ranks):
        s = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
        s.bind((host, 0))
        held.append(s)
        addrs.append((host, s.getsockname()[1]))
    for s in held:
        s.close()
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(f"{h}:{p}\n" for h, p in addrs)
    return addrs


def broadcast_array(transport: Transport, values, root: int = 0, ranks=None) -> np.ndarray:
    """Root fan-out of a complex128 payload to `ranks` (transport.py:343-353)."""
    if transport is None or transport.world_size == 1:
        return as_payload(values)
    members = sorted(range(transport.world_size) if ranks is None else ranks)
    if transport.rank == root:
        arr = as_payload(values)
        for r in members:
            if r != root:
                transport.send(r, arr, tag=TAG_DATA)
        return arr
    return transport.receive(root)
