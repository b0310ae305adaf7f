"""Minimal circuit IR for driving the core (host side).

The reference's IR lives in qpool/circuit.py (GateSpec 44-84, Circuit 87-129,
build_qaoa_circuit 248-264, qaoa_bindings 267-279).  The runtime here accepts
any object with the same attribute names (kind, qubits, param, matrix, graph),
so reference Circuit objects run unchanged; this module provides an
equivalent for callers that do not import qpool.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

ONE_QUBIT_KINDS = frozenset({"h", "x", "y", "z", "rx", "ry", "rz", "custom"})
ROTATION_KINDS = frozenset({"rx", "ry", "rz"})
TWO_QUBIT_KINDS = frozenset({"cx", "cz", "cphase", "cu"})
ALL_KINDS = ONE_QUBIT_KINDS | TWO_QUBIT_KINDS | {"diagcost", "noise"}
DEFAULT_GATE_DURATION = 1.0  # circuit.py:31 (noise scheduling, noise.py:92-139)


class UnboundParameterError(ValueError):
    pass


class CircuitParseError(ValueError):
    """A malformed circuit file line (circuit.py:34-37): message "line N: ..."."""

    def __init__(self, lineno: int, message: str):
        super().__init__(f"line {lineno}: {message}")
        self.lineno = lineno


@dataclass(frozen=True)
class GateSpec:
    kind: str
    qubits: tuple = ()
    param: float | str | None = None
    matrix: np.ndarray | None = field(default=None, repr=False, compare=False)
    graph: object | None = None
    graph_path: str | None = None
    duration: float = DEFAULT_GATE_DURATION

    def __post_init__(self) -> None:
        if self.kind not in ALL_KINDS:
            raise ValueError(f"unknown gate kind {self.kind!r}")
        if self.kind in TWO_QUBIT_KINDS:
            if len(self.qubits) != 2 or self.qubits[0] == self.qubits[1]:
                raise ValueError(f"{self.kind} needs two distinct qubits")
        elif self.kind != "diagcost" and len(self.qubits) != 1:
            raise ValueError(f"{self.kind} needs exactly one qubit")
        if self.kind == "diagcost" and self.graph is None:
            raise ValueError("diagcost needs a graph")
        if self.kind in ("custom", "cu") and self.matrix is None:
            raise ValueError(f"{self.kind} gate needs a matrix")

    @property
    def slot(self) -> str | None:
        return self.param[1:] if isinstance(self.param, str) else None


@dataclass(frozen=True)
class Circuit:
    num_qubits: int
    gates: tuple = ()

    def __post_init__(self) -> None:
        if self.num_qubits < 1:
            raise ValueError("need at least one qubit")
        for g in self.gates:
            for q in g.qubits:
                if not (0 <= q < self.num_qubits):
                    raise ValueError(f"{g.kind} on qubit {q} out of range")

    @property
    def slots(self) -> tuple:
        seen: list = []
        for g in self.gates:
            s = getattr(g, "slot", None)
            if s is not None and s not in seen:
                seen.append(s)
        return tuple(seen)

    def bind(self, bindings: dict) -> "Circuit":
        out = []
        for g in self.gates:
            s = g.slot
            out.append(replace(g, param=float(bindings[s])) if s is not None and s in bindings
                       else g)
        return Circuit(self.num_qubits, tuple(out))

    def require_bound(self) -> None:
        if self.slots:
            raise UnboundParameterError(
                "unbound parameter slot(s): " + ", ".join("$" + s for s in self.slots))


def gamma_slot(k: int) -> str:
    """Slot name of layer k's cost angle (circuit.py:240-241)."""
    return f"gamma{k}"


def beta_slot(k: int) -> str:
    """Slot name of layer k's mixer angle (circuit.py:244-245)."""
    return f"beta{k}"


def build_qaoa_circuit(graph, depth: int, graph_path: str | None = None) -> Circuit:
    """H on every qubit, then per layer k: cut phase with slot gamma_k and RX
    mixers with slot beta_k on every qubit (circuit.py:248-264, same gate
    sequence); `graph_path` is kept on the cost gates for serialisation."""
    if depth < 1:
        raise ValueError("depth must be >= 1")
    n = graph.num_vertices
    gates = [GateSpec("h", (q,)) for q in range(n)]
    for k in range(1, depth + 1):
        gates.append(GateSpec("diagcost", (), "$" + gamma_slot(k), graph=graph,
                              graph_path=graph_path))
        gates.extend(GateSpec("rx", (q,), "$" + beta_slot(k)) for q in range(n))
    return Circuit(n, tuple(gates))


def qaoa_bindings(depth: int, position) -> dict:
    """(gamma_1..gamma_p, beta_1..beta_p) -> slot values; betas doubled so the
    RX mixer realises RX(2 beta) (circuit.py:267-279)."""
    position = np.asarray(position, dtype=np.float64)
    if position.shape != (2 * depth,):
        raise ValueError(f"expected {2 * depth} parameters, got shape {position.shape}")
    out = {}
    for k in range(1, depth + 1):
        out[gamma_slot(k)] = float(position[k - 1])
        out[beta_slot(k)] = 2.0 * float(position[depth + k - 1])
    return out


# ---- text format (circuit.py:1-12, 130-237) -------------------------------------------
#   qubits <n> | h|x|y|z <q> | rx|ry|rz <q> <angle|$slot> | cx|cz <c> <t>
#   noise <q> <duration> | diagcost <graphfile> <gamma|$slot>      ('#' comments)
_TEXT_ARITY = {"h": 1, "x": 1, "y": 1, "z": 1, "rx": 2, "ry": 2, "rz": 2, "cx": 2, "cz": 2,
               "noise": 2, "diagcost": 2}
_TEXT_USAGE = {"h": "'h <q>'", "x": "'x <q>'", "y": "'y <q>'", "z": "'z <q>'",
               "rx": "'rx <q> <angle|$slot>'", "ry": "'ry <q> <angle|$slot>'",
               "rz": "'rz <q> <angle|$slot>'", "cx": "'cx <c> <t>'", "cz": "'cz <c> <t>'",
               "noise": "'noise <q> <duration>'",
               "diagcost": "'diagcost <graphfile> <gamma|$slot>'"}


def _param_token(tok: str, lineno: int):
    if tok.startswith("$"):
        if tok == "$":
            raise CircuitParseError(lineno, "empty slot name")
        return tok
    try:
        return float(tok)
    except ValueError:
        raise CircuitParseError(lineno, f"bad number {tok!r}") from None


def _gate_from_tokens(op: str, args: list, lineno: int, graph_dir):
    import os

    from .graphs import load_graph

    if len(args) != _TEXT_ARITY[op]:
        raise CircuitParseError(lineno, f"expected {_TEXT_USAGE[op]}")
    if op in ("h", "x", "y", "z"):
        return GateSpec(op, (int(args[0]),))
    if op in ROTATION_KINDS:
        return GateSpec(op, (int(args[0]),), _param_token(args[1], lineno))
    if op in ("cx", "cz"):
        return GateSpec(op, (int(args[0]), int(args[1])))
    if op == "noise":
        duration = float(args[1])
        if duration < 0:
            raise CircuitParseError(lineno, "negative noise duration")
        return GateSpec("noise", (int(args[0]),), duration=duration)
    path = args[0]  # diagcost: relative graph paths are anchored at graph_dir
    where = path if graph_dir is None or os.path.isabs(path) else os.path.join(graph_dir, path)
    try:
        graph = load_graph(where)
    except (OSError, ValueError) as exc:
        raise CircuitParseError(lineno, f"cannot load graph {path!r}: {exc}") from None
    return GateSpec("diagcost", (), _param_token(args[1], lineno), graph=graph, graph_path=path)


def parse_circuit(text: str, graph_dir: str | None = None) -> Circuit:
    """Circuit file text -> Circuit (same grammar and errors as the reference)."""
    n = None
    specs = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        tokens = raw.split("#", 1)[0].split()
        if not tokens:
            continue
        op, args = tokens[0], tokens[1:]
        if op == "qubits":
            if n is not None:
                raise CircuitParseError(lineno, "repeated qubits header")
            if len(args) != 1:
                raise CircuitParseError(lineno, "expected 'qubits <n>'")
            n = int(args[0])
            if n < 1:
                raise CircuitParseError(lineno, "need at least one qubit")
            continue
        if n is None:
            raise CircuitParseError(lineno, "gate before qubits header")
        if op not in _TEXT_ARITY:
            raise CircuitParseError(lineno, f"unknown mnemonic {op!r}")
        try:
            specs.append(_gate_from_tokens(op, args, lineno, graph_dir))
        except CircuitParseError:
            raise
        except ValueError as exc:
            raise CircuitParseError(lineno, str(exc)) from None
    if n is None:
        raise CircuitParseError(0, "missing 'qubits <n>' header")
    try:
        return Circuit(n, tuple(specs))
    except ValueError as exc:
        raise CircuitParseError(0, str(exc)) from None


def load_circuit(path) -> Circuit:
    import os

    with open(path, "r", encoding="utf-8") as fh:
        return parse_circuit(fh.read(), graph_dir=os.path.dirname(os.path.abspath(path)))


def serialize_circuit(circuit) -> str:
    """Circuit -> text; floats via repr so the text round-trips exactly."""
    def par(p):
        return p if isinstance(p, str) else repr(float(p))

    out = [f"qubits {circuit.num_qubits}"]
    for g in circuit.gates:
        k, q = g.kind, g.qubits
        if k in ("h", "x", "y", "z"):
            out.append(f"{k} {q[0]}")
        elif k in ROTATION_KINDS:
            out.append(f"{k} {q[0]} {par(g.param)}")
        elif k in ("cx", "cz"):
            out.append(f"{k} {q[0]} {q[1]}")
        elif k == "noise":
            out.append(f"noise {q[0]} {float(g.duration)!r}")
        elif k == "diagcost":
            if g.graph_path is None:
                raise ValueError("cannot serialize a diagcost gate without a graph file path")
            out.append(f"diagcost {g.graph_path} {par(g.param)}")
        else:
            raise ValueError(f"kind {k!r} has no text form")
    return "\n".join(out) + "\n"
