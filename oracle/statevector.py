"""Restatement of qpool/statevector.py (TEST INFRASTRUCTURE ONLY).

Same numpy expressions in the same order as the reference, so results are
bit-identical to it on the same host (checked against tests/golden).
"""
from __future__ import annotations

import numpy as np


class LocalityError(ValueError):
    pass


def tree_sum(values) -> float:
    """statevector.py:29-45: pairwise halving over element order."""
    x = np.asarray(values, dtype=np.float64).ravel()
    if x.size == 0:
        return 0.0
    if x.size & (x.size - 1):
        raise ValueError("tree_sum requires power-of-two length")
    while x.size > 1:
        x = x.reshape(-1, 2).sum(axis=1)
    return float(x[0])


def tree_sum_values(values) -> float:
    """statevector.py:53-71."""
    vals = [float(v) for v in values]
    if not vals:
        return 0.0

    def red(seq):
        if len(seq) == 1:
            return seq[0]
        split = 1 << (len(seq) - 1).bit_length() - 1
        return red(seq[:split]) + red(seq[split:])

    return red(vals)


def pair_update(a, b, u):
    """statevector.py:144-150."""
    return u[0, 0] * a + u[0, 1] * b, u[1, 0] * a + u[1, 1] * b


def pair_indices(size: int, q: int):
    """statevector.py:153-159: lower indices ascending, partner lo + 2^q."""
    step = 1 << q
    base = np.arange(0, size, step << 1)
    lo = (base[:, None] + np.arange(step)[None, :]).ravel()
    return lo, lo + step


def apply_1q(psi: np.ndarray, q: int, u: np.ndarray, m: int | None = None) -> np.ndarray:
    """statevector.py:162-177 (in place on psi)."""
    m = int(np.log2(psi.size)) if m is None else m
    if q >= m:
        raise LocalityError(f"qubit {q} is global for m={m}")
    if q < 0:
        raise ValueError("negative qubit index")
    lo, hi = pair_indices(psi.size, q)
    a, b = pair_update(psi[lo], psi[hi], u)
    psi[lo] = a
    psi[hi] = b
    return psi


def apply_controlled(psi: np.ndarray, control: int, target: int, u: np.ndarray) -> np.ndarray:
    """statevector.py:180-195 (in place)."""
    if control == target:
        raise ValueError("control and target must differ")
    idx = np.arange(psi.size)
    lo = idx[((idx >> control) & 1 == 1) & ((idx >> target) & 1 == 0)]
    hi = lo | (1 << target)
    a, b = pair_update(psi[lo], psi[hi], u)
    psi[lo] = a
    psi[hi] = b
    return psi


def cut_counts(edges, indices) -> np.ndarray:
    """graphs.py:35-42."""
    idx = np.asarray(indices, dtype=np.uint64)
    cuts = np.zeros(idx.shape, dtype=np.float64)
    one = np.uint64(1)
    for u, v in edges:
        cuts += ((idx >> np.uint64(u)) ^ (idx >> np.uint64(v))) & one
    return cuts


def owned_indices(m: int, rank: int) -> np.ndarray:
    """statevector.py:105-108."""
    base = rank << m
    return np.arange(base, base + (1 << m), dtype=np.uint64)


def apply_cut_phase(psi: np.ndarray, edges, gamma: float, rank: int = 0) -> np.ndarray:
    """statevector.py:198-206 with the phase function of runtime.py:131-133."""
    m = int(np.log2(psi.size))
    angles = np.asarray(gamma * cut_counts(edges, owned_indices(m, rank)), dtype=np.float64)
    psi *= np.exp(-1j * angles)
    return psi


def norm_squared(psi) -> float:
    """statevector.py:209-212."""
    return tree_sum(psi.real * psi.real + psi.imag * psi.imag)


def get_probability(psi, q: int, n: int | None = None, rank: int = 0) -> float:
    """statevector.py:215-231."""
    m = int(np.log2(psi.size))
    n = m if n is None else n
    if not (0 <= q < n):
        raise ValueError(f"qubit {q} out of range")
    if q >= m:
        return norm_squared(psi) if (rank >> (q - m)) & 1 else 0.0
    idx = np.arange(psi.size)
    sel = psi[(idx >> q) & 1 == 1]
    return tree_sum(sel.real * sel.real + sel.imag * sel.imag)


def z_expectation(psi, q: int, rank: int = 0) -> float:
    """statevector.py:234-242."""
    m = int(np.log2(psi.size))
    w = np.where((owned_indices(m, rank) >> np.uint64(q)) & np.uint64(1), -1.0, 1.0)
    return tree_sum(w * (psi.real * psi.real + psi.imag * psi.imag))


def maxcut_expectation(psi, edges, rank: int = 0) -> float:
    """statevector.py:245-251."""
    m = int(np.log2(psi.size))
    cuts = cut_counts(edges, owned_indices(m, rank))
    return tree_sum(cuts * (psi.real * psi.real + psi.imag * psi.imag))
