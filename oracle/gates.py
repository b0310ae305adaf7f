"""Restatement of qpool/gates.py:12-32 and the test input recipes of
pkg/tests/oracles.py:92-101 (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

import numpy as np

H = np.array([[1, 1], [1, -1]], dtype=np.complex128) / np.sqrt(2.0)
X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
Y = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)


def rx(t):
    c, s = np.cos(t / 2.0), np.sin(t / 2.0)
    return np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)


def ry(t):
    c, s = np.cos(t / 2.0), np.sin(t / 2.0)
    return np.array([[c, -s], [s, c]], dtype=np.complex128)


def rz(t):
    return np.array([[np.exp(-0.5j * t), 0], [0, np.exp(0.5j * t)]], dtype=np.complex128)


FIXED = {"h": H, "x": X, "y": Y, "z": Z}
ROT = {"rx": rx, "ry": ry, "rz": rz}


def random_unitary_2x2(rng):
    """oracles.py:92-96: QR of a complex Ginibre matrix, phase-fixed."""
    raw = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
    q, r = np.linalg.qr(raw)
    return q @ np.diag(np.diag(r) / np.abs(np.diag(r)))


def random_state(n, rng):
    """oracles.py:99-101: i.i.d. normal re/im, normalised."""
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return (psi / np.linalg.norm(psi)).astype(np.complex128)
