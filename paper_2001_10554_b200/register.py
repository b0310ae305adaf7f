"""Paper-style register API (IQS ``QubitRegister``; the
reference's TypeScript wrapper bindings/src/register.ts:56-129 uses the same
method names).

Gates are queued and flushed as one fused program when a value is read, so a
Python loop of ApplyX calls costs one HBM pass per tile-sized run of gates
instead of one per call.  With ``num_states > 1`` the register is a pool:
every Apply* acts on each state, and per-state angles may be passed as arrays
(PAPER.md:206-210).
"""
from __future__ import annotations

import numpy as np

from . import _native
from . import gates as G
from .graphs import edge_array, make_graph
from .runtime import GateQueue


class QubitRegister:
    def __init__(self, num_qubits: int, kind: str = "base", index: int = 0,
                 num_states: int = 1, device: int = 0, fuse: bool = True):
        self.num_qubits = num_qubits
        self.num_states = num_states
        self.state = _native.DeviceState(num_qubits, num_qubits, 0, num_states, device)
        self.queue = GateQueue(self.state, fuse)
        self.Initialize(kind, index)

    # ---- initialisation ----------------------------------------------------------
    def Initialize(self, kind: str, index: int = 0) -> "QubitRegister":
        self.queue.discard()
        if kind == "base":
            if not (0 <= index < (1 << self.num_qubits)):
                raise ValueError(f"basis index {index} out of range")
            self.state.defer_basis(index)
        elif kind == "uniform":
            _native.call("qs_init_constant", self.state.handle,
                         2.0 ** (-self.num_qubits / 2.0), 0.0)
        else:
            raise ValueError(f"unknown initialization {kind!r}")
        return self

    def _q(self, q: int) -> int:
        if not (0 <= q < self.num_qubits):
            raise ValueError(f"qubit {q} out of range")
        return q

    def _rot(self, fn, angle):
        a = np.asarray(angle, dtype=np.float64)
        if a.ndim == 0:
            return fn(float(a))
        if a.shape != (self.num_states,):
            raise ValueError(f"expected {self.num_states} angles")
        kind = {G.rx: "rx", G.ry: "ry", G.rz: "rz"}.get(fn)
        if kind is not None:
            return G.rotation_batch(kind, a)
        return np.stack([fn(float(x)) for x in a])

    # ---- one-qubit gates -----------------------------------------------------------
    def Apply1QubitGate(self, q: int, u) -> "QubitRegister":
        self.queue.one_qubit(self._q(q), np.asarray(u, dtype=np.complex128))
        return self

    def ApplyHadamard(self, q: int):
        return self.Apply1QubitGate(q, G.HADAMARD)

    def ApplyPauliX(self, q: int):
        return self.Apply1QubitGate(q, G.PAULI_X)

    def ApplyPauliY(self, q: int):
        return self.Apply1QubitGate(q, G.PAULI_Y)

    def ApplyPauliZ(self, q: int):
        return self.Apply1QubitGate(q, G.PAULI_Z)

    def ApplyRotationX(self, q: int, angle):
        return self.Apply1QubitGate(q, self._rot(G.rx, angle))

    def ApplyRotationY(self, q: int, angle):
        return self.Apply1QubitGate(q, self._rot(G.ry, angle))

    def ApplyRotationZ(self, q: int, angle):
        return self.Apply1QubitGate(q, self._rot(G.rz, angle))

    # ---- controlled gates ------------------------------------------------------------
    def ApplyControlled1QubitGate(self, control: int, target: int, u) -> "QubitRegister":
        if control == target:
            raise ValueError("control and target must differ")
        self.queue.controlled(self._q(control), self._q(target), np.asarray(u, np.complex128))
        return self

    def ApplyCPauliX(self, control: int, target: int):
        return self.ApplyControlled1QubitGate(control, target, G.PAULI_X)

    def ApplyCPauliZ(self, control: int, target: int):
        return self.ApplyControlled1QubitGate(control, target, G.PAULI_Z)

    def ApplyCPhaseRotation(self, control: int, target: int, phi):
        return self.ApplyControlled1QubitGate(control, target, self._rot(G.cphase, phi))

    # ---- QAOA cost layer ---------------------------------------------------------------
    def ApplyDiagonalCutPhase(self, graph_or_edges, gamma):
        graph = graph_or_edges if hasattr(graph_or_edges, "edges") else \
            make_graph(self.num_qubits, graph_or_edges)
        self.queue.cut_phase(graph, gamma)
        return self

    # ---- reads (flush first) -------------------------------------------------------------
    def _obs(self, kind, q=0, edges=None):
        self.queue.flush()
        v = self.state.observable(kind, q, edges)
        return float(v[0]) if self.num_states == 1 else v

    def GetProbability(self, q: int):
        return self._obs(_native.QS_OBS_PROB, self._q(q))

    def GetProbabilities(self):
        """P(q=1) for every qubit, one pass over the state."""
        self.queue.flush()
        v = self.state.marginals()
        return v[0] if self.num_states == 1 else v

    def ExpectationValueZ(self, q: int):
        return self._obs(_native.QS_OBS_Z, self._q(q))

    def ComputeNorm(self):
        v = self._obs(_native.QS_OBS_NORM)
        return np.sqrt(v)

    def MaxCutExpectation(self, graph_or_edges):
        graph = graph_or_edges if hasattr(graph_or_edges, "edges") else \
            make_graph(self.num_qubits, graph_or_edges)
        return self._obs(_native.QS_OBS_MAXCUT, 0, edge_array(graph))

    def GetAmplitudes(self) -> np.ndarray:
        self.queue.flush()
        a = self.state.download()
        return a if self.num_states == 1 else a.reshape(self.num_states, -1)

    def Flush(self) -> int:
        return self.queue.flush()
