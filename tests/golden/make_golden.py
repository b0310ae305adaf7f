"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports qpool from /root/reference/pkg/src (read-only) and the reference
test recipes from /root/reference/pkg/tests/oracles.py, runs the reference's
own functions on seeded inputs and writes small .npz fixtures next to this
file.  The fixtures travel with the repo; nothing at test time reads
/root/reference.  Large outputs (2^20-amplitude states) are stored as a
SHA-256 of the complex128 bytes plus seeded samples.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import oracles  # noqa: E402  (reference test recipes)
from qpool import distribution as dist  # noqa: E402
from qpool import gates, runtime  # noqa: E402
from qpool import statevector as sv  # noqa: E402
from qpool.circuit import Circuit, GateSpec, build_qaoa_circuit, qaoa_bindings  # noqa: E402
from qpool.graphs import cut_counts, make_graph  # noqa: E402
from qpool.optimize import exact_maxcut, random_3regular_graph  # noqa: E402
from qpool.pool import RandomStream  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SEED = 20260809  # the reference's test seed (tests/conftest.py:31-33)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.complex128).tobytes()).hexdigest()


def save(name, **arrays):
    np.savez_compressed(os.path.join(OUT, name), **arrays)
    print("wrote", name, {k: getattr(v, "shape", None) for k, v in arrays.items()})


def part(psi, m=None, r=0):
    n = int(np.log2(psi.size)) if m is None else m
    return sv.StatePartition(n if m is None else m, n if m is None else m, r, psi.copy())


def gen_1q():
    rng = np.random.default_rng(SEED)
    n = 10
    psi0 = oracles.random_state(n, rng)
    us, outs = [], []
    for q in range(n):
        u = oracles.random_unitary_2x2(rng)
        p = sv.StatePartition(n, n, 0, psi0.copy())
        sv.apply_local_one_qubit_gate(p, q, gates.gate_matrix(u))
        us.append(u)
        outs.append(p.amplitudes.copy())
    # named gates on a basis state (known answers) and a chained sequence
    chain_q = rng.integers(0, n, size=40)
    chain_u = np.stack([oracles.random_unitary_2x2(rng) for _ in chain_q])
    p = sv.StatePartition(n, n, 0, psi0.copy())
    for q, u in zip(chain_q, chain_u):
        sv.apply_local_one_qubit_gate(p, int(q), u)
    save("golden_1q.npz", psi0=psi0, us=np.stack(us), outs=np.stack(outs),
         chain_q=chain_q, chain_u=chain_u, chain_out=p.amplitudes.copy())


def gen_ctrl():
    rng = np.random.default_rng(SEED + 1)
    n = 10
    psi0 = oracles.random_state(n, rng)
    pairs, kinds, mats, outs = [], [], [], []
    for k in range(36):
        c = int(rng.integers(n))
        t = int(rng.integers(n - 1))
        t = t if t < c else t + 1
        kind = k % 3
        if kind == 0:
            u = gates.PAULI_X
        elif kind == 1:
            phi = float(rng.uniform(0, 2 * np.pi))
            u = np.array([[1, 0], [0, np.exp(1j * phi)]], dtype=np.complex128)
        else:
            u = oracles.random_unitary_2x2(rng)
        p = sv.StatePartition(n, n, 0, psi0.copy())
        sv.apply_local_controlled_gate(p, c, t, u)
        pairs.append((c, t))
        kinds.append(kind)
        mats.append(u)
        outs.append(p.amplitudes.copy())
    save("golden_ctrl.npz", psi0=psi0, pairs=np.array(pairs), kinds=np.array(kinds),
         mats=np.stack(mats), outs=np.stack(outs))


def gen_phase_obs():
    rng = np.random.default_rng(SEED + 2)
    n = 10
    graph = random_3regular_graph(n, RandomStream(SEED, "pool", 0))
    edges = np.array(graph.edges, dtype=np.int32)
    psi0 = oracles.random_state(n, rng)
    gammas = rng.uniform(0, 2 * np.pi, size=6)
    outs = []
    for g in gammas:
        p = sv.StatePartition(n, n, 0, psi0.copy())
        sv.apply_diagonal_phase(p, lambda idx, g=g: g * cut_counts(graph, idx))
        outs.append(p.amplitudes.copy())
    # observables on several random states, full and split into 4 ranks
    states = np.stack([oracles.random_state(n, rng) for _ in range(4)])
    norm, prob, z, cut = [], [], [], []
    for s in states:
        p = sv.StatePartition(n, n, 0, s.copy())
        norm.append(sv.norm_squared(p))
        prob.append([sv.get_probability(p, q) for q in range(n)])
        z.append([sv.z_expectation(p, q) for q in range(n)])
        cut.append(sv.maxcut_expectation(p, graph))
    # rank partials of state 0 over 4 ranks (m = 8)
    m = n - 2
    partials = {"norm": [], "prob": [], "z": [], "cut": []}
    for r in range(4):
        p = sv.StatePartition(n, m, r, states[0][r << m:(r + 1) << m].copy())
        partials["norm"].append(sv.norm_squared(p))
        partials["prob"].append([sv.get_probability(p, q) for q in range(n)])
        partials["z"].append([sv.z_expectation(p, q) for q in range(n)])
        partials["cut"].append(sv.maxcut_expectation(p, graph))
    save("golden_phase_obs.npz", edges=edges, psi0=psi0, gammas=gammas, outs=np.stack(outs),
         states=states, norm=np.array(norm), prob=np.array(prob), z=np.array(z),
         cut=np.array(cut), part_norm=np.array(partials["norm"]),
         part_prob=np.array(partials["prob"]), part_z=np.array(partials["z"]),
         part_cut=np.array(partials["cut"]),
         tree_in=rng.standard_normal(64), tree_out=np.array(sv.tree_sum(np.arange(64) * 0.1)))


def cfg1_gates(n: int, layers: int, seed: int):
    """BASELINE config 1 recipe: per layer, per qubit, kind ~ U{H,RX,RZ},
    theta ~ U[0,2pi) for rotations, one default_rng stream; then CX(q,q+1) from
    q = layer%2 in steps of 2."""
    rng = np.random.default_rng(seed)
    out = []
    for layer in range(layers):
        for q in range(n):
            k = ("h", "rx", "rz")[int(rng.integers(3))]
            if k == "h":
                out.append({"kind": "h", "qubits": (q,)})
            else:
                out.append({"kind": k, "qubits": (q,), "param": float(rng.uniform(0, 2 * np.pi))})
        for q in range(layer % 2, n - 1, 2):
            out.append({"kind": "cx", "qubits": (q, q + 1)})
    return out


def to_circuit(n, glist):
    specs = []
    for g in glist:
        specs.append(GateSpec(g["kind"], tuple(g["qubits"]), g.get("param")))
    return Circuit(n, tuple(specs))


def encode(glist):
    kinds = {"h": 0, "rx": 1, "rz": 2, "cx": 3}
    arr = np.zeros((len(glist), 4))
    for i, g in enumerate(glist):
        q = g["qubits"]
        arr[i] = (kinds[g["kind"]], q[0], q[1] if len(q) > 1 else -1, g.get("param", 0.0))
    return arr


def gen_cfg1():
    for n, layers, name in ((12, 10, "golden_cfg1_n12.npz"), (20, 10, "golden_cfg1_n20.npz")):
        glist = cfg1_gates(n, layers, SEED)
        circ = to_circuit(n, glist)
        t0 = time.perf_counter()
        psi = runtime.simulate_circuit(circ, num_ranks=1)
        dt = time.perf_counter() - t0
        probs = []
        ctx = runtime.make_context(None, n, 1, 0)
        ctx.partition.amplitudes[:] = psi
        for q in range(n):
            probs.append(runtime.measure_probability(ctx, q))
        rng = np.random.default_rng(1)
        idx = np.sort(rng.choice(psi.size, size=min(psi.size, 4096), replace=False))
        extra = {"state": psi} if n <= 12 else {}
        save(name, gates=encode(glist), probs=np.array(probs), sha=np.array(sha(psi)),
             sample_idx=idx, sample=psi[idx], ref_seconds=np.array(dt), **extra)


def gen_cfg3_small():
    rng = np.random.default_rng(SEED + 3)
    n = 12
    psi0 = oracles.random_state(n, rng)
    pairs, mats = [], []
    p = sv.StatePartition(n, n, 0, psi0.copy())
    for _ in range(64):
        c = int(rng.integers(n))
        t = int(rng.integers(n - 1))
        t = t if t < c else t + 1
        phi = float(rng.uniform(0, 2 * np.pi))
        for u in (gates.PAULI_X, np.array([[1, 0], [0, np.exp(1j * phi)]], dtype=np.complex128),
                  oracles.random_unitary_2x2(rng)):
            sv.apply_local_controlled_gate(p, c, t, u)
            pairs.append((c, t))
            mats.append(u)
    save("golden_cfg3_n12.npz", psi0=psi0, pairs=np.array(pairs), mats=np.stack(mats),
         out=p.amplitudes.copy())


def gen_cfg4_small():
    """Config 4 recipe at m=10: n = 10 + p over P = 2^p ranks, 4 layers of Haar 1q on
    every qubit then CX(q, n-1-q) for q < n//2, via the reference's distributed path."""
    out = {}
    for p in range(4):
        P = 1 << p
        n = 10 + p
        rng = np.random.default_rng(SEED + 10 + p)
        psi0 = oracles.random_state(n, rng)
        us = []
        seq = []
        for layer in range(4):
            for q in range(n):
                u = oracles.random_unitary_2x2(rng)
                us.append(u)
                seq.append(("u", q, len(us) - 1))
            for q in range(n // 2):
                seq.append(("cx", q, n - 1 - q))
        us = np.stack(us)

        def rank_fn(transport, n=n, psi0=psi0, seq=seq, us=us):
            ctx = runtime.make_context(transport, n, 1, 0)
            m = ctx.topology.num_local_qubits
            r = ctx.state_rank
            ctx.partition.amplitudes[:] = psi0[r << m:(r + 1) << m]
            before = transport.counters.snapshot()
            for op in seq:
                if op[0] == "u":
                    dist.apply_one_qubit_gate(ctx.partition, ctx.topology, ctx.comm, op[1],
                                              us[op[2]])
                else:
                    dist.apply_controlled_gate(ctx.partition, ctx.topology, ctx.comm, op[1], op[2],
                                               gates.PAULI_X)
            delta = transport.counters.delta(before)
            return ctx.partition.amplitudes.copy(), delta.messages_sent, delta.amplitudes_sent

        res = runtime.run_spmd(P, rank_fn, timeout=60.0)
        out[f"psi0_p{p}"] = psi0
        out[f"us_p{p}"] = us
        out[f"out_p{p}"] = np.concatenate([r[0] for r in res])
        out[f"msgs_p{p}"] = np.array([r[1] for r in res])
        out[f"amps_p{p}"] = np.array([r[2] for r in res])
    save("golden_cfg4_m10.npz", **out)


def gen_cfg5():
    """QAOA MaxCut (config 5 recipe): graph = random_3regular_graph(20, RandomStream(seed,
    'pool', 0)), p=4, params ~ U[0,pi)^8; reference run_circuit + measure_maxcut."""
    n, depth = 20, 4
    graph = random_3regular_graph(n, RandomStream(SEED, "pool", 0))
    exact = exact_maxcut(graph)
    circ = build_qaoa_circuit(graph, depth)
    rng = np.random.default_rng(SEED + 5)
    params = rng.uniform(0, np.pi, size=(8, 2 * depth))
    values, shas, samples = [], [], []
    sidx = np.sort(np.random.default_rng(2).choice(1 << n, size=2048, replace=False))
    for pos in params:
        ctx = runtime.make_context(None, n, 1, 0)
        runtime.run_circuit(ctx, circ, qaoa_bindings(depth, pos))
        values.append(runtime.measure_maxcut(ctx, graph))
        psi = ctx.partition.amplitudes
        shas.append(sha(psi))
        samples.append(psi[sidx])
    # small full-state QAOA (n=10, p=2) for exact amplitude checks
    g10 = random_3regular_graph(10, RandomStream(SEED, "pool", 1))
    c10 = build_qaoa_circuit(g10, 2)
    p10 = rng.uniform(0, np.pi, size=(4, 4))
    st10, v10 = [], []
    for pos in p10:
        ctx = runtime.make_context(None, 10, 1, 0)
        runtime.run_circuit(ctx, c10, qaoa_bindings(2, pos))
        st10.append(ctx.partition.amplitudes.copy())
        v10.append(runtime.measure_maxcut(ctx, g10))
    save("golden_cfg5.npz", edges=np.array(graph.edges, dtype=np.int32), exact=np.array(exact),
         params=params, values=np.array(values), shas=np.array(shas), sample_idx=sidx,
         samples=np.stack(samples), edges10=np.array(g10.edges, dtype=np.int32), params10=p10,
         states10=np.stack(st10), values10=np.array(v10))


def gen_accounting():
    """Exchange accounting of the reference's criterion 2 (test_acceptance.py:67-89)."""
    n, world = 12, 4
    u = oracles.random_unitary_2x2(np.random.default_rng(7))

    def rank_fn(transport):
        ctx = runtime.make_context(transport, n, 1, seed=0)
        sv.init_uniform(ctx.partition)
        obs = {}
        for q in range(n):
            before = transport.counters.snapshot()
            dist.apply_one_qubit_gate(ctx.partition, ctx.topology, ctx.comm, q,
                                      np.asarray(u, dtype=np.complex128))
            d = transport.counters.delta(before)
            obs[q] = (d.messages_sent, d.bytes_sent)
        return obs, ctx.partition.amplitudes.copy()

    res = runtime.run_spmd(world, rank_fn, timeout=20.0)
    with open(os.path.join(OUT, "golden_accounting.json"), "w") as fh:
        json.dump({"n": n, "world": world, "u": [[x.real, x.imag] for x in u.ravel()],
                   "per_rank": [{str(q): v for q, v in r[0].items()} for r in res]}, fh, indent=1)
    save("golden_accounting_state.npz", u=u, out=np.concatenate([r[1] for r in res]))


def gen_noise():
    """Noise trajectories (noise.py): a 12-qubit circuit with scheduled T1/T2
    noise, trajectories 0..3 of the reference's trajectory streams."""
    from qpool.noise import NoiseModel, schedule_noise, trajectory_stream
    n = 12
    rng = np.random.default_rng(SEED + 7)
    specs = []
    for layer in range(3):
        for q in range(n):
            k = ("h", "rx", "ry")[int(rng.integers(3))]
            specs.append(GateSpec(k, (q,)) if k == "h" else
                         GateSpec(k, (q,), float(rng.uniform(0, 2 * np.pi))))
        for q in range(layer % 2, n - 1, 2):
            specs.append(GateSpec("cx", (q, q + 1)))
    circ = schedule_noise(Circuit(n, tuple(specs)))
    model = NoiseModel(20.0, 15.0)
    states = []
    for t in range(4):
        ctx = runtime.make_context(None, n, 1, 0, model)
        runtime.run_circuit(ctx, circ, noise_stream=trajectory_stream(SEED, t))
        states.append(ctx.partition.amplitudes.copy())
    enc = []
    kinds = {"h": 0, "rx": 1, "ry": 2, "cx": 3, "noise": 4}
    for g in circ.gates:
        q = g.qubits
        enc.append((kinds[g.kind], q[0], q[1] if len(q) > 1 else -1,
                    g.param if g.param is not None else 0.0, g.duration))
    save("golden_noise.npz", gates=np.array(enc), states=np.stack(states),
         t1=np.array(20.0), t2=np.array(15.0), seed=np.array(SEED))


def gen_cli():
    """Reports of the reference CLI (cli.py) on small circuit/graph files,
    for the format-compatibility tests (tests/test_gpu_cli.py).  The input
    files are written next to the reports in tests/golden/cli/."""
    import contextlib
    import io

    from qpool import cli
    from qpool.circuit import serialize_circuit
    from qpool.graphs import serialize_graph

    d = os.path.join(OUT, "cli")
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(SEED + 11)
    with open(os.path.join(d, "ring.graph"), "w") as fh:
        fh.write(serialize_graph(make_graph(4, [(0, 1), (1, 2), (2, 3), (3, 0)])))
    g6 = random_3regular_graph(6, RandomStream(SEED, "pool", 3))
    with open(os.path.join(d, "cubic6.graph"), "w") as fh:
        fh.write(serialize_graph(g6))
    # mixed gates, noise and a cut phase on 4 qubits
    mix = ("qubits 4\nh 0\nh 1\nh 2\nh 3\nnoise 2 1.5\ndiagcost ring.graph 0.61\n"
           "cx 3 1\nrz 0 0.9\nnoise 0 0.5\nry 2 -1.25\ncz 0 3\n")
    with open(os.path.join(d, "mix.qc"), "w") as fh:
        fh.write(mix)
    # QAOA with slots on the 6-vertex cubic graph
    lines = ["qubits 6"] + [f"h {q}" for q in range(6)]
    for k in (1, 2):
        lines.append(f"diagcost cubic6.graph $gamma{k}")
        lines += [f"rx {q} $beta{k}" for q in range(6)]
    with open(os.path.join(d, "qaoa6.qc"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    # 12 qubits: random layers (no amplitude lines in the report)
    lines = ["qubits 12"]
    for layer in range(3):
        for q in range(12):
            k = ("h", "rx", "ry", "rz")[int(rng.integers(4))]
            lines.append(f"{k} {q}" if k == "h" else f"{k} {q} {float(rng.uniform(0, 6.2))!r}")
        lines += [f"cx {q} {q + 1}" for q in range(layer % 2, 11, 2)]
    with open(os.path.join(d, "layers12.qc"), "w") as fh:
        fh.write("\n".join(lines) + "\n")

    cases = {
        "run_mix": ["run", "mix.qc", "--seed", "777777", "--t1", "30", "--t2", "15"],
        "run_mix_r4": ["run", "mix.qc", "--seed", "777777", "--t1", "30", "--t2", "15",
                       "--ranks", "4"],
        "run_mix_s2": ["run", "mix.qc", "--seed", "5", "--t1", "30", "--t2", "15",
                       "--ranks", "4", "--states", "2"],
        "run_qaoa6": ["run", "qaoa6.qc", "--bind", "gamma1=0.3", "--bind", "beta1=1.1",
                      "--bind", "$gamma2=2.2", "--bind", "beta2=0.4", "--maxcut", "cubic6.graph",
                      "--ranks", "2"],
        "run_layers12": ["run", "layers12.qc", "--ranks", "8"],
        "noise_mix": ["noise-ensemble", "mix.qc", "--t1", "30", "--t2", "15",
                      "--trajectories", "8", "--seed", "9", "--states", "2", "--ranks", "2"],
        "noise_qaoa6": ["noise-ensemble", "qaoa6.qc", "--t1", "40", "--t2", "20",
                        "--trajectories", "11", "--seed", "3", "--states", "3", "--ranks", "6",
                        "--observable", "maxcut:cubic6.graph", "--bind", "gamma1=0.3",
                        "--bind", "beta1=1.1", "--bind", "gamma2=2.2", "--bind", "beta2=0.4"],
        "bench_gate": ["bench-gate", "--n", "7", "--ranks", "4", "--repetitions", "2"],
        "pso_v8": ["qaoa-pso", "--vertices", "8", "--graphs", "2", "--depth", "2",
                   "--particles", "6", "--budget", "24", "--seed", "11", "--states", "4",
                   "--ranks", "4"],
        "pso_v12_paper": ["qaoa-pso", "--vertices", "12", "--depth", "1", "--particles", "5",
                          "--budget", "15", "--seed", "3", "--pso-sign", "paper",
                          "--states", "2", "--ranks", "4"],
        "pso_v14": ["qaoa-pso", "--vertices", "14", "--depth", "3", "--particles", "3",
                    "--budget", "9", "--seed", "5"],
    }
    meta = {}
    cwd = os.getcwd()
    os.chdir(d)
    try:
        for name, argv in cases.items():
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                rc = cli.main(argv)
            assert rc == 0, (name, rc)
            text = buf.getvalue()
            if name == "bench_gate":  # timings vary: keep qubit,messages,bytes,ranks,n
                rows = [r.split(",") for r in text.splitlines()]
                text = "\n".join(",".join(r[i] for i in (0, 2, 3, 4, 5)) for r in rows) + "\n"
            with open(name + ".txt", "w") as fh:
                fh.write(text)
            meta[name] = argv
    finally:
        os.chdir(cwd)
    with open(os.path.join(d, "cases.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("wrote", len(cases), "CLI reports")


def gen_optimize():
    """Swarm and graph pins for optimize.py: random_3regular_graph edges from
    keyed streams, exact_maxcut, and a swarm driven by fixed values."""
    from qpool import optimize as opt

    graphs = {}
    for n, key in ((4, 0), (8, 1), (12, 2), (20, 3)):
        g = opt.random_3regular_graph(n, RandomStream(SEED, "pool", key))
        graphs[f"edges_{n}"] = np.array(g.edges)
        graphs[f"exact_{n}"] = np.array(opt.exact_maxcut(g))
    rng = np.random.default_rng(SEED + 21)
    out = {}
    for sign in ("standard", "paper"):
        sw = opt.init_swarm(5, 4, opt.PsoHyperparams(sign=sign), RandomStream(SEED, "pool", 9))
        pos, vel, gb = [], [], []
        vals = rng.uniform(0, 1, size=(6, 5))
        for v in vals:
            opt.step_swarm(sw, v)
            pos.append(np.stack([p.position for p in sw.particles]))
            vel.append(np.stack([p.velocity for p in sw.particles]))
            gb.append(sw.global_best_value)
        out[f"{sign}_values"] = vals
        out[f"{sign}_pos"] = np.stack(pos)
        out[f"{sign}_vel"] = np.stack(vel)
        out[f"{sign}_gbest"] = np.array(gb)
    save("golden_optimize.npz", **graphs, **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["1q", "ctrl", "phase_obs", "cfg1", "cfg3", "cfg4", "cfg5", "acct"]
    table = {"1q": gen_1q, "ctrl": gen_ctrl, "phase_obs": gen_phase_obs, "cfg1": gen_cfg1,
             "cfg3": gen_cfg3_small, "cfg4": gen_cfg4_small, "cfg5": gen_cfg5,
             "acct": gen_accounting, "noise": lambda: gen_noise(), "cli": lambda: gen_cli(),
             "optimize": lambda: gen_optimize()}
    for w in which:
        t0 = time.perf_counter()
        table[w]()
        print(f"  {w}: {time.perf_counter() - t0:.1f}s")
