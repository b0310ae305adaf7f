"""Restatement of qpool/distribution.py (TEST INFRASTRUCTURE ONLY).

The SPMD ranks are emulated sequentially over a list of host partitions;
each pair of partner ranks performs the reference's three-step exchange
(distribution.py:121-178): the lower rank updates the pairs at offsets
[0, half) (its psi[:half] with the partner's psi[:half]), the upper rank
those at [half, 2 half), masked by the local control bit in case (c).
"""
from __future__ import annotations

import numpy as np

from . import statevector as sv


def exchange_pairs(parts, m: int, q: int, u, control_local=None) -> None:
    d = 1 << (q - m)
    half = 1 << (m - 1)
    for lower_rank in range(len(parts)):
        if lower_rank & d:
            continue
        lower, upper = parts[lower_rank], parts[lower_rank | d]
        for sl, offsets in ((slice(0, half), np.arange(0, half)),
                            (slice(half, 2 * half), np.arange(half, 2 * half))):
            a, b = lower[sl], upper[sl]
            if control_local is None:
                na, nb = sv.pair_update(a, b, u)
            else:
                sel = np.nonzero((offsets >> control_local) & 1)[0]
                na, nb = a.copy(), b.copy()
                xa, xb = sv.pair_update(a[sel], b[sel], u)
                na[sel], nb[sel] = xa, xb
            lower[sl] = na
            upper[sl] = nb


def apply_one_qubit_gate(parts, n: int, q: int, u) -> None:
    """distribution.py:181-192 over all ranks."""
    m = n - (len(parts).bit_length() - 1)
    if q < m:
        for p in parts:
            sv.apply_1q(p, q, u)
    else:
        exchange_pairs(parts, m, q, u)


def apply_controlled_gate(parts, n: int, control: int, target: int, u) -> None:
    """distribution.py:195-230, cases (a)-(d)."""
    m = n - (len(parts).bit_length() - 1)
    if control == target:
        raise ValueError("control and target must differ")
    if control < m and target < m:
        for p in parts:
            sv.apply_controlled(p, control, target, u)
        return
    if control >= m:
        selected = [r for r in range(len(parts)) if (r >> (control - m)) & 1]
        if target < m:
            for r in selected:
                sv.apply_1q(parts[r], target, u)
            return
        # (d): only control=1 ranks exchange; pairs never mix selected/unselected
        d = 1 << (target - m)
        sub = {r: parts[r] for r in selected}
        half = 1 << (m - 1)
        for lr in selected:
            if lr & d:
                continue
            lower, upper = sub[lr], sub[lr | d]
            for sl in (slice(0, half), slice(half, 2 * half)):
                na, nb = sv.pair_update(lower[sl], upper[sl], u)
                lower[sl], upper[sl] = na, nb
        return
    exchange_pairs(parts, m, target, u, control_local=control)


def group_reduce_sum(partials) -> float:
    """distribution.py:233-252: recursive doubling == tree over rank order."""
    return sv.tree_sum(np.asarray(partials, dtype=np.float64))
