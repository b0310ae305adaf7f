"""The real multi-process path (one process per rank, torch.distributed gloo
control plane, CUDA-IPC peer mappings, k_exchange_peer) run with every rank
on cuda:0.  The exchange kernels of partner ranks touch disjoint pair sets and
never wait on each other (the pairwise barriers are host-side), so this is a
faithful single-GPU run of the multi-GPU code path.  Compared bit for bit with
the reference's own run_spmd output (golden_cfg4_m10.npz)."""
import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN, bits_equal

pytestmark = pytest.mark.gpu


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, p, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as tdist

    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2001_10554_b200 import distribution as dist, runtime
        from paper_2001_10554_b200.circuit import Circuit, GateSpec

        g = np.load(os.path.join(GOLDEN, "golden_cfg4_m10.npz"))
        n = 10 + p
        psi0, us = g[f"psi0_p{p}"], g[f"us_p{p}"]
        seq, k = [], 0
        for layer in range(4):
            for qb in range(n):
                seq.append(GateSpec("custom", (qb,), matrix=us[k]))
                k += 1
            for qb in range(n // 2):
                seq.append(GateSpec("cx", (qb, n - 1 - qb)))
        comm = dist.TorchComm(exchange_mode="peer")
        ctx = runtime.make_context(comm, n, 1, device=0)
        m = ctx.topology.num_local_qubits
        ctx.partition.amplitudes = psi0[rank << m:(rank + 1) << m]
        ctx.norm_check_interval = 0
        runtime.run_circuit(ctx, Circuit(n, tuple(seq)))
        full = runtime.gather_group_state(ctx)
        norm = runtime.measure_norm_squared(ctx)
        q.put((rank, full, norm, ctx.state.counters()))
    except BaseException as exc:  # surface the failure to the parent
        q.put((rank, repr(exc), None, None))
        raise
    finally:
        tdist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("p", [1, 2])
def test_multiprocess_peer_exchange_matches_reference(p):
    import torch.multiprocessing as mp

    world = 1 << p
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r, full, norm, counters = q.get(timeout=280)
        res[r] = (full, norm, counters)
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r][0], str), res[r][0]
    ref = np.load(os.path.join(GOLDEN, "golden_cfg4_m10.npz"))[f"out_p{p}"]
    assert bits_equal(res[0][0], ref)
    for r in range(world):
        assert abs(res[r][1] - 1.0) < 1e-10
        assert res[r][2][0] > 0  # exchanges happened
