"""Multi-process host path of the distributed core on CPU: world_size 2 (and
4) over torch.distributed gloo.  The GPU data plane cannot run here; the
control plane -- pair handshakes, group-local rank-ordered gathers, the tree
reduction, IPC handle exchange, the reference's point-to-point payloads and
pool reductions -- is exactly what runs between GPUs."""
import os
import socket
import threading

import numpy as np
import pytest
import torch.distributed as tdist
import torch.multiprocessing as mp

from paper_2001_10554_b200 import distribution as dist
from paper_2001_10554_b200 import pool as pl
from paper_2001_10554_b200 import statevector as sv
from paper_2001_10554_b200 import transport as tp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = tp.TorchTransport()
        comm = dist.GroupComm(t, 0, world)
        topo = dist.RankTopology(world, 4)
        out = {}
        comm.pair_barrier(rank ^ 1)
        out["gather"] = comm.allgather(float(rank) + 0.25, world)
        partials = np.random.default_rng(3).standard_normal(world)
        out["reduced"] = dist.group_reduce_sum(partials[rank], topo, comm)
        # two groups of world/2 ranks: group-local gathers only
        half = world // 2
        g = dist.GroupComm(t, (rank // half) * half, half)
        out["group_gather"] = g.allgather(10.0 * rank, half)
        comm.attach(None)  # no device here: empty handles travel
        out["handles"] = t._handles
        try:
            comm.peer_pointer(rank ^ 1)
            out["peer"] = "opened"
        except dist.TransportError:
            out["peer"] = "TransportError"
        out["route"] = dist.route_controlled(rank, topo, 0, 3)
        # the reference's payload path: send/receive, barrier, counters
        if rank == 0:
            t.send(1, np.arange(3) + 1j)
        elif rank == 1:
            out["payload"] = t.receive(0)
        t.barrier()
        out["counters"] = (t.counters.messages_sent, t.counters.amplitudes_sent)
        # pool reductions over a build_pool layout (pool.py:131-182)
        layout = pl.build_pool(world, world // 2 if world > 2 else 2)
        mine = float(layout.group_of_rank(rank) + 1)
        out["pool_sum"] = pl.incoherent_sum_over_pool(mine, layout, t)
        out["pool_gather"] = pl.gather_state_values(mine, layout, t)
        q.put((rank, out))
    finally:
        tdist.destroy_process_group()


def run_world(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    return res


@pytest.mark.timeout(200)
@pytest.mark.parametrize("world", [2, 4])
def test_gloo_control_plane(world):
    res = run_world(world)
    partials = np.random.default_rng(3).standard_normal(world)
    half = world // 2
    S = world // 2 if world > 2 else 2
    for r in range(world):
        assert res[r]["gather"] == [float(k) + 0.25 for k in range(world)]
        assert res[r]["reduced"] == sv.tree_sum(partials)
        base = (r // half) * half
        assert res[r]["group_gather"] == [10.0 * (base + k) for k in range(half)]
        assert res[r]["handles"] == [b""] * world
        assert res[r]["peer"] == "TransportError"
        assert res[r]["pool_sum"] == sv.tree_sum_values([float(s + 1) for s in range(S)])
    assert np.array_equal(res[0]["pool_gather"], np.arange(1, S + 1, dtype=float))
    assert all(res[r]["pool_gather"] is None for r in range(1, world))
    assert np.array_equal(res[1]["payload"], np.arange(3) + 1j)
    if world == 2:
        assert res[0]["route"] == ("exchange", 1, True, 0)
        assert res[1]["route"] == ("exchange", 0, False, 0)
    else:  # n=4 over 4 ranks: qubit 3 is rank bit 1
        assert res[0]["route"] == ("exchange", 2, True, 0)
        assert res[3]["route"] == ("exchange", 1, False, 0)


def test_inprocess_fabric_barriers_payloads_and_timeout():
    fab = tp.InProcessFabric(2, timeout=0.3)
    out = [None, None]

    def run(r):
        t = fab.endpoint(r)
        c = dist.GroupComm(t, 0, 2)
        c.pair_barrier(1 - r)
        got = c.allgather(r * 2.0, 2)
        c.send(1 - r, np.full(4, r + 1.0))
        out[r] = (got, c.receive(1 - r), t.counters.snapshot())

    ts = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert out[0][0] == out[1][0] == [0.0, 2.0]
    assert np.array_equal(out[0][1], np.full(4, 2.0 + 0j))
    assert out[0][2] == tp.TransportCounters(1, 4)
    lonely = dist.GroupComm(tp.InProcessFabric(2, timeout=0.2).endpoint(0), 0, 2)
    with pytest.raises(tp.TransportTimeout):
        lonely.pair_barrier(1)
    with pytest.raises(tp.TransportTimeout):
        tp.InProcessFabric(2, timeout=0.1).endpoint(0).receive(1)


def test_group_comm_rejects_rank_outside_group():
    t = tp.InProcessFabric(4).endpoint(3)
    with pytest.raises(ValueError):
        dist.GroupComm(t, 0, 2)
    with pytest.raises(ValueError):
        dist.GroupComm(None, 0, 2)
    assert dist.GroupComm(t, 2, 2).rank == 1
