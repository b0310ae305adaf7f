"""Multi-process host path of the distributed core on CPU: world_size 2 over
torch.distributed gloo (the GPU data plane cannot run here; the control
plane -- pair barriers, rank-ordered gathers, the tree reduction, IPC handle
exchange -- is exactly what runs between GPUs)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as tdist
import torch.multiprocessing as mp

from paper_2001_10554_b200 import distribution as dist
from paper_2001_10554_b200 import statevector as sv


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
        comm = dist.TorchComm()
        topo = dist.RankTopology(world, 4)
        out = {}
        comm.pair_barrier(rank ^ 1)
        out["gather"] = comm.allgather(float(rank) + 0.25, world)
        partials = np.random.default_rng(3).standard_normal(world)
        out["reduced"] = dist.group_reduce_sum(partials[rank], topo, comm)
        comm.attach(None)  # no device here: empty handles travel
        out["handles"] = comm._handles
        try:
            comm.peer_pointer(rank ^ 1)
            out["peer"] = "opened"
        except dist.TransportError as e:
            out["peer"] = "TransportError"
        out["route"] = dist.route_controlled(rank, topo, 0, 3)
        q.put((rank, out))
    finally:
        tdist.destroy_process_group()


@pytest.mark.timeout(120)
def test_world2_gloo_control_plane():
    world = 2
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
    partials = np.random.default_rng(3).standard_normal(world)
    for r in range(world):
        assert res[r]["gather"] == [0.25, 1.25]
        assert res[r]["reduced"] == sv.tree_sum(partials)
        assert res[r]["handles"] == [b"", b""]
        assert res[r]["peer"] == "TransportError"
    assert res[0]["route"] == ("exchange", 1, True, 0)
    assert res[1]["route"] == ("exchange", 0, False, 0)


def test_thread_fabric_barriers_and_timeout():
    fab = dist.ThreadFabric(2, timeout=0.3)
    import threading

    out = [None, None]

    def run(r):
        c = fab.endpoint(r)
        c.pair_barrier(1 - r)
        out[r] = c.allgather(r * 2.0, 2)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert out == [[0.0, 2.0], [0.0, 2.0]]
    lonely = dist.ThreadFabric(2, timeout=0.2).endpoint(0)
    with pytest.raises(dist.TransportTimeout):
        lonely.pair_barrier(1)
