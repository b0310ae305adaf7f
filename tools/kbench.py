"""Kernel-level timing of the B200 core (CUDA events on the library stream).

  python tools/kbench.py [--m 30] [--reps 5] [--what 1q,fused,ctrl,obs,phase]

Prints one JSON object per measurement: per-target GB/s for single 1q gates
(config 2 per-target table), fused sweep passes, controlled gates (config 3),
cut phase and observables.  Algorithmic bytes: 32 B/amp per 1q gate,
16 B/amp per controlled gate (control=1 half), 8 B/amp for a CPhase-like
diag(1,z) gate, 16 B/amp per reduction read.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2001_10554_b200 import _native as N  # noqa: E402
from paper_2001_10554_b200.workloads import haar_2x2, device_gaussian  # noqa: E402


def timed(st, fn, reps):
    fn()
    st.synchronize()
    out = []
    for _ in range(reps):
        st.event_record(0)
        fn()
        st.event_record(1)
        out.append(st.event_elapsed_ms(0, 1))
    return float(np.median(out)), float(np.min(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=30)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--what", default="1q,fused,ctrl,phase,obs")
    args = ap.parse_args()
    m = args.m
    amps = 1 << m
    st = N.DeviceState(m, m)
    device_gaussian(st, 11)
    rng = np.random.default_rng(0)
    what = args.what.split(",")
    if "1q" in what:
        for q in range(m):
            u = haar_2x2(rng).view(np.float64).ravel()
            g = [N.QsGate(0, q, -1, 0, 0, 0)]
            med, best = timed(st, lambda: st.apply_program(g, u, fuse=False), args.reps)
            print(json.dumps({"kernel": "k_gate1q", "q": q, "ms": med,
                              "gbs": 32 * amps / med / 1e6, "gbs_best": 32 * amps / best / 1e6}))
    if "fused" in what:
        us = np.stack([haar_2x2(rng) for _ in range(m)]).view(np.float64).reshape(-1)
        gates = [N.QsGate(0, q, -1, 0, 8 * q, 0) for q in range(m)]
        starts = N.plan_program(m, gates)
        st.launch_log(True)
        med, best = timed(st, lambda: st.apply_program(gates, us, fuse=True), args.reps)
        ms, kinds = st.read_launch_log()
        st.launch_log(False)
        passes = len(starts)
        per = ms.reshape(-1, passes) if ms.size % passes == 0 else ms[None, :]
        print(json.dumps({"kernel": "sweep_fused", "passes": passes, "starts": starts,
                          "ms_step": med, "gate_updates_per_s": m / (med / 1e3),
                          "pass_ms": np.median(per, axis=0).tolist(),
                          "pass_gbs": (32 * amps / np.median(per, axis=0) / 1e6).tolist()}))
    if "ctrl" in what:
        for kind, mat in (("cnot", np.array([[0, 1], [1, 0]], np.complex128)),
                          ("cphase", np.diag([1, np.exp(0.7j)]).astype(np.complex128)),
                          ("cu", haar_2x2(rng))):
            res = []
            for (c, t) in ((0, 1), (1, 0), (3, 20), (20, 3), (29, 0), (0, 29), (15, 16)):
                g = [N.QsGate(1, t, c, 0, 0, 0)]
                u = mat.view(np.float64).ravel()
                med, _ = timed(st, lambda: st.apply_program(g, u, fuse=False), args.reps)
                alg = (8 if kind == "cphase" else 16) * amps
                res.append({"c": c, "t": t, "ms": med, "gbs": alg / med / 1e6})
            print(json.dumps({"kernel": "k_controlled", "gate": kind, "cases": res}))
    if "phase" in what:
        edges = np.array([(i, (i + 1) % 20) for i in range(20)] + [(i, (i + 7) % 20)
                                                                   for i in range(10)], np.int32)
        lut = np.exp(-1j * 0.3 * np.arange(31)).view(np.float64)
        g = [N.QsGate(2, 0, -1, 0, 0, 0)]
        med, _ = timed(st, lambda: st.apply_program(g, lut, edges, fuse=False), args.reps)
        print(json.dumps({"kernel": "k_cut_phase", "ms": med, "gbs": 32 * amps / med / 1e6}))
    if "obs" in what:
        for kind in (0, 1, 3):
            edges = np.array([(i, (i + 1) % 20) for i in range(20)], np.int32)
            med, _ = timed(st, lambda: st.observable(kind, 5, edges), args.reps)
            rd = 16 * amps // (2 if kind == 1 else 1)
            print(json.dumps({"kernel": "k_tree", "obs": kind, "ms": med, "gbs": rd / med / 1e6}))


if __name__ == "__main__" and "--scan" not in sys.argv:
    main()


def pass_scan(m=30, reps=3):
    """Tile-pass time vs number of fused gates (low targets 0..k-1 / high targets)."""
    st = N.DeviceState(m, m)
    device_gaussian(st, 5)
    rng = np.random.default_rng(1)
    amps = 1 << m
    for base in (0, 18):
        for k in (2, 3, 6, 9, 12):
            if base + k > m or (base > 0 and k > 9):
                continue
            us = np.stack([haar_2x2(rng) for _ in range(k)]).view(np.float64).reshape(-1)
            gates = [N.QsGate(0, base + i, -1, 0, 8 * i, 0) for i in range(k)]
            med, _ = timed(st, lambda: st.apply_program(gates, us, fuse=True), reps)
            print(json.dumps({"scan": "tile", "first_target": base, "gates": k, "ms": med,
                              "gbs": 32 * amps / med / 1e6,
                              "ms_per_gate_fp64_floor": 10 * amps * k / 18e12 * 1e3}))


if __name__ == "__main__" and "--scan" in sys.argv:
    pass_scan()
