"""Circuit runner over the oracle (TEST INFRASTRUCTURE ONLY); follows
qpool/runtime.py:115-162 gate by gate (no norm check)."""
from __future__ import annotations

import numpy as np

from . import distribution as dist
from . import gates
from . import statevector as sv


def matrix(kind, param=None, mat=None):
    if kind in gates.FIXED:
        return gates.FIXED[kind]
    if kind in gates.ROT:
        return gates.ROT[kind](float(param))
    if kind in ("custom", "cu"):
        return np.asarray(mat, dtype=np.complex128)
    if kind == "cx":
        return gates.X
    if kind == "cz":
        return gates.Z
    if kind == "cphase":
        return np.array([[1, 0], [0, np.exp(1j * float(param))]], dtype=np.complex128)
    raise ValueError(kind)


def run(n: int, gate_list, psi0=None, ranks: int = 1):
    """gate_list: dicts {kind, qubits, param?, matrix?, edges?}.  Returns the full state."""
    m = n - (ranks.bit_length() - 1)
    full = np.zeros(1 << n, dtype=np.complex128) if psi0 is None else \
        np.array(psi0, dtype=np.complex128)
    if psi0 is None:
        full[0] = 1.0
    parts = [full[r << m:(r + 1) << m].copy() for r in range(ranks)]
    for g in gate_list:
        kind = g["kind"]
        if kind == "diagcost":
            for r, p in enumerate(parts):
                sv.apply_cut_phase(p, g["edges"], float(g["param"]), rank=r)
        elif kind in ("cx", "cz", "cphase", "cu"):
            c, t = g["qubits"]
            dist.apply_controlled_gate(parts, n, c, t, matrix(kind, g.get("param"), g.get("matrix")))
        else:
            dist.apply_one_qubit_gate(parts, n, g["qubits"][0],
                                      matrix(kind, g.get("param"), g.get("matrix")))
    return np.concatenate(parts)
