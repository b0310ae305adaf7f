"""Seeded synthetic inputs with the shapes and distributions BASELINE.json's
configs name (there is no dataset: every input is generated).

* Haar-random 2x2 unitaries: QR of a complex Ginibre matrix with the phases
  of diag(R) removed -- the recipe of the reference's test oracle
  (pkg/tests/oracles.py:92-96).
* Gaussian states: i.i.d. N(0,1) real and imaginary parts, normalised
  (oracles.py:99-101).  On the device they come from a counter-based
  generator keyed by the global amplitude index (qs_init_gaussian), so a state
  is identical for every rank split; host states use numpy for small n.
* Random 3-regular graphs: the pairing model with rejection.
"""
from __future__ import annotations

import numpy as np

from . import _native


def haar_2x2(rng: np.random.Generator) -> np.ndarray:
    raw = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
    q, r = np.linalg.qr(raw)
    d = np.diag(r)
    return q @ np.diag(d / np.abs(d))


def gaussian_state(n: int, rng: np.random.Generator) -> np.ndarray:
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return (psi / np.linalg.norm(psi)).astype(np.complex128)


def device_gaussian(state: _native.DeviceState, seed: int, group_norm=None) -> float:
    """Fill a device state with the keyed Gaussian and normalise it over the
    whole (possibly distributed) state; `group_norm(partial) -> total`."""
    _native.call("qs_init_gaussian", state.handle, seed)
    partial = float(state.observable(_native.QS_OBS_NORM)[0])
    total = group_norm(partial) if group_norm else partial
    _native.call("qs_scale", state.handle, 1.0 / np.sqrt(total))
    return total


def random_3regular_graph(num_vertices: int, rng: np.random.Generator):
    from .graphs import make_graph

    if num_vertices < 4 or num_vertices % 2:
        raise ValueError("3-regular graphs need an even vertex count >= 4")
    stubs0 = np.repeat(np.arange(num_vertices), 3)
    while True:
        stubs = rng.permutation(stubs0).reshape(-1, 2)
        edges = set()
        ok = True
        for a, b in stubs:
            a, b = int(a), int(b)
            key = (min(a, b), max(a, b))
            if a == b or key in edges:
                ok = False
                break
            edges.add(key)
        if ok:
            return make_graph(num_vertices, sorted(edges))


def config1_gates(n: int, layers: int, seed: int) -> list:
    """BASELINE config 1: per layer, each qubit gets H/RX/RZ drawn
    uniformly (theta ~ U[0,2pi) for rotations) from one default_rng stream,
    then CX(q, q+1) from q = layer % 2 in steps of 2."""
    from .circuit import GateSpec

    rng = np.random.default_rng(seed)
    out = []
    for layer in range(layers):
        for q in range(n):
            k = ("h", "rx", "rz")[int(rng.integers(3))]
            out.append(GateSpec(k, (q,)) if k == "h" else
                       GateSpec(k, (q,), float(rng.uniform(0, 2 * np.pi))))
        for q in range(layer % 2, n - 1, 2):
            out.append(GateSpec("cx", (q, q + 1)))
    return out
