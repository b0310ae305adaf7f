"""Command-line front end with the reference's report formats (qpool/cli.py).

SURVEY 8f row 4: scripts and bindings that drive the reference through its
CLI (scripts/scaling_study.py reads the ``bench-gate`` CSV; the TypeScript
QubitRegister parses the ``run`` report) can drive this core unchanged:

  run             circuit file -> "qubits/ranks/states/seed", "prob q p",
                  "amp i re im" (n <= 10) and "maxcut c" lines (cli.py:151-185)
  bench-gate      one random 2x2 per target qubit, CSV
                  qubit,mean_seconds,messages,bytes,ranks,n,min_seconds
                  (cli.py:193-238); each timing brackets the kernel with a
                  device synchronize, messages/bytes are rank 0's exchange
                  counters per repetition
  noise-ensemble  running mean of a noisy circuit's observable, CSV
                  trajectories,running_mean,reference (cli.py:288-339)
  qaoa-pso        PSO over QAOA/MaxCut on random 3-regular graphs, CSV
                  evaluations,mean_ratio,step (cli.py:240-274); each chunk of
                  particles is one pool program on the device

Ranks are emulated on one GPU as threads (``--ranks``), exactly the
reference's in-process transport; multi-GPU runs use torchrun + TorchComm
(runtime.make_context) instead of the reference's socket transport, which is
not part of this core (--transport socket exits with a usage error).  Values
are bit-identical to the reference's for any rank/state layout.  Exit codes:
0 ok, 2 usage/parse errors, 3 transport failures.
"""
from __future__ import annotations

import argparse
import math
import sys
import time

import numpy as np

from . import distribution as dist
from . import gates as G
from . import runtime
from . import statevector as sv
from ._native import TransportError
from .circuit import CircuitParseError, UnboundParameterError, load_circuit
from .graphs import load_graph
from .noise import NoiseModel, RandomStream, SCOPE_POOL
from .pool import build_pool

EXIT_OK, EXIT_USAGE, EXIT_TRANSPORT = 0, 2, 3


class UsageError(ValueError):
    pass


def _common(p: argparse.ArgumentParser) -> None:
    p.add_argument("--ranks", type=int, default=1, help="emulated ranks (threads, one GPU)")
    p.add_argument("--states", type=int, default=1, help="pool states (rank groups)")
    p.add_argument("--transport", choices=("inproc", "socket"), default="inproc")
    p.add_argument("--rendezvous", help="(socket transport: not supported by this core)")
    p.add_argument("--seed", type=int, default=0, help="master seed (decimal)")
    p.add_argument("--out", help="also write the report/CSV to this path")
    p.add_argument("--device", type=int, default=0, help="CUDA device")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="qsb200")
    sub = ap.add_subparsers(dest="command", required=True)
    r = sub.add_parser("run", help="run a circuit file")
    r.add_argument("circuit")
    r.add_argument("--t1", type=float, default=math.inf)
    r.add_argument("--t2", type=float, default=math.inf)
    r.add_argument("--bind", action="append", default=[], metavar="NAME=VALUE")
    r.add_argument("--maxcut", metavar="GRAPHFILE")
    _common(r)
    b = sub.add_parser("bench-gate", help="one-qubit gate timing per qubit")
    b.add_argument("--n", type=int, required=True)
    b.add_argument("--repetitions", type=int, default=3)
    _common(b)
    e = sub.add_parser("noise-ensemble", help="running incoherent average of a noisy circuit")
    e.add_argument("circuit")
    e.add_argument("--t1", type=float, required=True)
    e.add_argument("--t2", type=float, required=True)
    e.add_argument("--trajectories", type=int, default=100)
    e.add_argument("--observable", default="prob:0", help="prob:<qubit> or maxcut:<graphfile>")
    e.add_argument("--bind", action="append", default=[], metavar="NAME=VALUE")
    _common(e)
    o = sub.add_parser("qaoa-pso", help="PSO/QAOA study on random 3-regular graphs")
    o.add_argument("--vertices", type=int, required=True)
    o.add_argument("--graphs", type=int, default=1)
    o.add_argument("--depth", type=int, default=1)
    o.add_argument("--particles", type=int, default=4)
    o.add_argument("--budget", type=int, required=True)
    o.add_argument("--pso-sign", choices=("standard", "paper"), default="standard")
    _common(o)
    return ap


def _bindings(pairs) -> dict:
    out = {}
    for pair in pairs:
        name, eq, value = pair.partition("=")
        if not eq or not name:
            raise UsageError(f"--bind expects NAME=VALUE, got {pair!r}")
        out[name.lstrip("$")] = float(value)
    return out


def _layout(args, n: int):
    if args.transport == "socket":
        raise UsageError("the socket transport is not part of the B200 core; "
                         "run one process per GPU under torchrun instead")
    if args.ranks < 1:
        raise UsageError("--ranks must be >= 1")
    layout = build_pool(args.ranks, args.states)
    if layout.ranks_per_state >= (1 << n):
        raise ValueError(f"{layout.ranks_per_state} ranks per state leave no local qubit "
                         f"for n={n}")
    return layout


def _emit(text: str, args) -> None:
    sys.stdout.write(text)
    if args.out:
        with open(args.out, "w", encoding="utf-8") as fh:
            fh.write(text)


def cmd_run(args) -> int:
    circuit = load_circuit(args.circuit)
    bindings = _bindings(args.bind)
    model = NoiseModel(args.t1, args.t2)
    cut_graph = load_graph(args.maxcut) if args.maxcut else None
    n = circuit.num_qubits
    layout = _layout(args, n)

    # the report is group 0's state (world rank 0); any other group only
    # differs in its noise stream, so only group 0 is simulated
    def rank_fn(comm):
        ctx = runtime.make_context(comm, n, 1, device=args.device, seed=args.seed,
                                   noise_model=model)
        runtime.run_circuit(ctx, circuit, bindings)
        probs = [runtime.measure_probability(ctx, q) for q in range(n)]
        cut = runtime.measure_maxcut(ctx, cut_graph) if cut_graph is not None else None
        full = runtime.gather_group_state(ctx) if n <= 10 else None
        return probs, cut, full

    probs, cut, full = runtime.run_spmd(layout.ranks_per_state, rank_fn)[0]
    lines = [f"qubits {n}", f"ranks {args.ranks}", f"states {layout.num_states}",
             f"seed {args.seed}"]
    lines += [f"prob {q} {probs[q]!r}" for q in range(n)]
    if full is not None:
        lines += [f"amp {i} {float(a.real)!r} {float(a.imag)!r}" for i, a in enumerate(full)]
    if cut is not None:
        lines.append(f"maxcut {cut!r}")
    _emit("\n".join(lines) + "\n", args)
    return EXIT_OK


def _bench_unitary(stream: RandomStream) -> np.ndarray:
    """rz(a) @ ry(b) @ rz(c), (a, b, c) ~ U[0, 2pi) from the pool stream (cli.py:188-190)."""
    a, b, c = stream.uniform(3, 0.0, 2.0 * math.pi)
    return G.rz(a) @ G.ry(b) @ G.rz(c)


def cmd_bench_gate(args) -> int:
    n = args.n
    if args.repetitions < 1:
        raise UsageError("--repetitions must be >= 1")
    if args.transport == "socket":
        raise UsageError("the socket transport is not part of the B200 core")
    if args.ranks < 1:
        raise UsageError("--ranks must be >= 1")
    reps = args.repetitions

    def rank_fn(comm):
        ctx = runtime.make_context(comm, n, 1, device=args.device, seed=args.seed)
        ctx.norm_check_interval = 0
        stream = RandomStream(args.seed, SCOPE_POOL, 0)
        if ctx.is_idle:
            return None
        active = ctx.topology.effective_ranks
        sv.init_uniform(ctx.partition)
        st = ctx.state
        # one untimed warm-up gate (cli.py:201-203)
        comm = ctx.comm
        dist.apply_one_qubit_gate(ctx.partition, ctx.topology, comm, 0,
                                  np.eye(2, dtype=np.complex128))
        st.synchronize()
        rows = []
        for q in range(n):
            u = _bench_unitary(stream)
            comm.allgather(0.0, active)  # barrier
            m0, a0 = st.counters()
            times = []
            for _ in range(reps):
                t0 = time.perf_counter()
                dist.apply_one_qubit_gate(ctx.partition, ctx.topology, comm, q, u)
                st.synchronize()
                times.append(time.perf_counter() - t0)
            m1, a1 = st.counters()
            comm.allgather(0.0, active)
            rows.append((q, sum(times) / len(times), (m1 - m0) // reps,
                         16 * (a1 - a0) // reps, min(times)))
        return rows

    rows = runtime.run_spmd(args.ranks, rank_fn)[0]
    lines = ["qubit,mean_seconds,messages,bytes,ranks,n,min_seconds"]
    lines += [f"{q},{mean!r},{msgs},{nbytes},{args.ranks},{n},{tmin!r}"
              for q, mean, msgs, nbytes, tmin in rows]
    _emit("\n".join(lines) + "\n", args)
    return EXIT_OK


def _observable(spec: str):
    kind, _, arg = spec.partition(":")
    if kind == "prob":
        q = int(arg)
        return lambda ctx: runtime.measure_probability(ctx, q)
    if kind == "maxcut":
        graph = load_graph(arg)
        return lambda ctx: runtime.measure_maxcut(ctx, graph)
    raise UsageError(f"unknown observable {spec!r}")


def cmd_noise_ensemble(args) -> int:
    model = NoiseModel(args.t1, args.t2)
    circuit = load_circuit(args.circuit).bind(_bindings(args.bind))
    circuit.require_bound()
    observe = _observable(args.observable)
    total = args.trajectories
    if total < 1:
        raise UsageError("--trajectories must be >= 1")
    n = circuit.num_qubits
    layout = _layout(args, n)
    S, rps = layout.num_states, layout.ranks_per_state
    if rps == 1:  # whole states: one batched pool on the device, S states per round
        ctx = runtime.make_context(None, n, S, device=args.device, seed=args.seed)
        reference, values = runtime.run_noise_ensemble(ctx, circuit, model, total, observe,
                                                       num_groups=S)
    else:  # groups of rps emulated ranks, one group at a time
        values = np.full(total, np.nan)
        reference = None
        for g in range(S):
            def rank_fn(comm, g=g):
                ctx = runtime.make_context(comm, n, 1, device=args.device, seed=args.seed,
                                           state_offset=g)
                return runtime.run_noise_ensemble(ctx, circuit, model, total, observe,
                                                  num_groups=S)

            ref_g, vals = runtime.run_spmd(rps, rank_fn)[0]
            reference = ref_g if reference is None else reference
            values = np.where(np.isnan(values), vals, values)
    _emit(runtime.noise_ensemble_csv(values, reference), args)
    return EXIT_OK


def cmd_qaoa_pso(args) -> int:
    import os

    from .optimize import PsoHyperparams, random_3regular_graph, run_pso_qaoa, trace_csv_lines

    if args.vertices % 2 or args.vertices > 20:
        raise UsageError("--vertices must be even and <= 20 at desk scale")
    hyper = PsoHyperparams(sign=args.pso_sign)
    n = args.vertices
    layout = _layout(args, n)
    # every particle's value is layout-independent (tree-ordered reductions),
    # so the states of the pool hold whole circuits on one device
    S = layout.num_states
    ctx = runtime.make_context(None, n, S, device=args.device, seed=args.seed)
    pool_stream = RandomStream(args.seed, SCOPE_POOL, 0)
    traces = []
    for k in range(args.graphs):
        graph = random_3regular_graph(n, pool_stream.split(2 * k))
        traces.append(run_pso_qaoa(ctx, graph, args.depth, args.particles, args.budget,
                                   pool_stream.split(2 * k + 1), hyper))
    lines = ["evaluations,mean_ratio,step"]
    for i, row in enumerate(traces[0]):
        mean = sum(t[i].global_best_ratio for t in traces) / len(traces)
        lines.append(f"{row.evaluations},{mean!r},{row.step}")
    _emit("\n".join(lines) + "\n", args)
    if args.out:
        stem, ext = os.path.splitext(args.out)
        for k, trace in enumerate(traces):
            with open(f"{stem}_instance{k}{ext or '.csv'}", "w", encoding="utf-8") as fh:
                fh.write("\n".join(trace_csv_lines(trace)) + "\n")
    return EXIT_OK


COMMANDS = {"run": cmd_run, "bench-gate": cmd_bench_gate, "noise-ensemble": cmd_noise_ensemble,
            "qaoa-pso": cmd_qaoa_pso}


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return COMMANDS[args.command](args)
    except TransportError as exc:
        print(f"transport error: {exc}", file=sys.stderr)
        return EXIT_TRANSPORT
    except (CircuitParseError, UnboundParameterError, UsageError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except RuntimeError as exc:
        cause = exc.__cause__
        if isinstance(cause, TransportError):
            print(f"transport error: {exc}", file=sys.stderr)
            return EXIT_TRANSPORT
        if isinstance(cause, ValueError):
            print(f"error: {exc}", file=sys.stderr)
            return EXIT_USAGE
        raise


if __name__ == "__main__":
    sys.exit(main())
