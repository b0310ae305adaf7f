"""CPU checks of the QS_FUSE_FACTORED host side (csrc/factor.cu): the 2x2
factorisation u = k diag(1,za) [c*[[1,-t],[t,1]]] diag(1,zb) reconstructs u,
and the Python fuse-mode mapping.  The GPU parity of the factored path is in
test_gpu_factored.py."""
import numpy as np
import pytest

from paper_2001_10554_b200 import _native as N

from oracle import gates as ogates


def rebuild(u):
    k, za, zb, form, t, scale = N.decompose_2x2(u)
    assert form == 0
    assert abs(abs(k) - 1) < 1e-15 and abs(abs(za) - 1) < 1e-15 and abs(abs(zb) - 1) < 1e-15
    shear = scale * np.array([[1.0, -t], [t, 1.0]])
    return k * np.diag([1.0, za]) @ shear @ np.diag([1.0, zb]), t


def test_haar_and_named_gates_reconstruct():
    rng = np.random.default_rng(1)
    mats = [ogates.random_unitary_2x2(rng) for _ in range(3000)]
    mats += [ogates.rx(x) for x in np.linspace(0.01, 3.1, 9)]
    mats += [ogates.ry(x) for x in np.linspace(0.01, 3.1, 9)]
    mats += [np.array([[1, 1], [1, -1]]) / np.sqrt(2), np.array([[1, -1j], [-1j, 1]]) / np.sqrt(2)]
    worst = 0.0
    for u in mats:
        rec, t = rebuild(u)
        worst = max(worst, float(np.abs(rec - u).max()))
        assert 0 <= abs(t) <= 1e9
    assert worst < 1e-14


def test_unfactorable_matrices_are_refused():
    X = np.array([[0, 1], [1, 0]], dtype=complex)
    for u in (X, np.diag([1, 1j]), np.eye(2), 2 * np.eye(2)[[1, 0]],
              np.array([[1, 1], [0, 1]], dtype=complex),
              np.array([[1e-10, 1], [1, -1e-10]])):
        with pytest.raises(ValueError):
            N.decompose_2x2(u)


def test_fuse_modes():
    assert N.fuse_code(False) == N.FUSE_NONE
    assert N.fuse_code(True) == N.FUSE_EXACT
    assert N.fuse_code("exact") == N.FUSE_EXACT
    assert N.fuse_code("factored") == N.FUSE_FACTORED == 2
    with pytest.raises(ValueError):
        N.fuse_code("fast")
    with pytest.raises(ValueError):
        N.fuse_code(7)
