"""Noise trajectories restated for the oracle (TEST INFRASTRUCTURE ONLY).

Follows qpool/noise.py:60-80 and the keyed stream of qpool/pool.py:27-78
literally -- numpy's own Philox generator constructed per draw, scipy's ndtri,
numpy's ``@`` -- so it is the scalar path the product's vectorised draws
(paper_2001_10554_b200/noise.py) are checked against.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import ndtri

from . import gates

_MASK64 = (1 << 64) - 1
_STATE_SCOPE_ID = 2  # pool.py:25


def _mix(x: int) -> int:
    """SplitMix64 (pool.py:27-31)."""
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


class TrajectoryStream:
    """RandomStream(seed, "state", scope_key=t) (noise.py:60-69, pool.py:34-78)."""

    def __init__(self, seed: int, trajectory: int):
        mix = _mix(_STATE_SCOPE_ID)
        mix = _mix(mix ^ (trajectory & _MASK64))
        mix = _mix(mix ^ 0)
        self.key = [seed & _MASK64, mix]
        self.counter = 0

    def normal(self, count: int) -> np.ndarray:
        gen = np.random.Generator(np.random.Philox(counter=[self.counter, 0, 0, 0], key=self.key))
        u = gen.random(count)
        self.counter += count
        return ndtri(np.clip(u, 1e-300, None))


def variances(duration: float, t1: float, t2: float):
    """noise.py:48-55."""
    return duration / t1, 2.0 * duration * (1.0 / t2 - 1.0 / (2.0 * t1))


def noise_matrix(duration: float, t1: float, t2: float, stream: TrajectoryStream) -> np.ndarray:
    """noise.py:70-80: draws (tx, ty, tz), then rz(tz) @ ry(ty) @ rx(tx)."""
    vxy, vz = variances(duration, t1, t2)
    d = stream.normal(3)
    tx, ty, tz = d[0] * math.sqrt(vxy), d[1] * math.sqrt(vxy), d[2] * math.sqrt(vz)
    return gates.rz(tz) @ gates.ry(ty) @ gates.rx(tx)


def bind_trajectory(gate_list, t1: float, t2: float, seed: int, trajectory: int) -> list:
    """Replace every {"kind": "noise", "qubits", "duration"} entry by the
    custom matrix trajectory `trajectory` draws for it, in circuit order."""
    stream = TrajectoryStream(seed, trajectory)
    out = []
    for g in gate_list:
        if g["kind"] == "noise":
            out.append({"kind": "custom", "qubits": g["qubits"],
                        "matrix": noise_matrix(g["duration"], t1, t2, stream)})
        else:
            out.append(g)
    return out
