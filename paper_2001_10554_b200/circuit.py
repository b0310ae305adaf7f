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


@dataclass(frozen=True)
class GateSpec:
    kind: str
    qubits: tuple = ()
    param: float | str | None = None
    matrix: np.ndarray | None = field(default=None, repr=False, compare=False)
    graph: object | None = None
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


def build_qaoa_circuit(graph, depth: int) -> Circuit:
    """H on every qubit, then per layer k: cut phase with slot gamma_k and RX
    mixers with slot beta_k on every qubit (same sequence as the reference)."""
    if depth < 1:
        raise ValueError("depth must be >= 1")
    n = graph.num_vertices
    gates = [GateSpec("h", (q,)) for q in range(n)]
    for k in range(1, depth + 1):
        gates.append(GateSpec("diagcost", (), f"$gamma{k}", graph=graph))
        gates.extend(GateSpec("rx", (q,), f"$beta{k}") for q in range(n))
    return Circuit(n, tuple(gates))


def qaoa_bindings(depth: int, position) -> dict:
    """(gamma_1..gamma_p, beta_1..beta_p) -> slot values; betas doubled so the
    RX mixer realises RX(2 beta)."""
    position = np.asarray(position, dtype=np.float64)
    if position.shape != (2 * depth,):
        raise ValueError(f"expected {2 * depth} parameters, got shape {position.shape}")
    out = {}
    for k in range(1, depth + 1):
        out[f"gamma{k}"] = float(position[k - 1])
        out[f"beta{k}"] = 2.0 * float(position[depth + k - 1])
    return out
