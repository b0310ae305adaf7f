"""Multi-threaded CPU restatement of apply_local_one_qubit_gate for the
benchmark's CPU baseline (TEST/BENCH INFRASTRUCTURE ONLY).

Same elementwise numpy expression as statevector.py:150 (u00*a + u01*b,
u10*a + u11*b, numpy complex128 ufuncs), evaluated on strided views instead
of the reference's int64 index arrays, and split over host threads (numpy
releases the GIL inside ufunc loops).  Results are bit-identical to the
faithful restatement (tests/test_oracle.py checks it); it is simply the
strongest honest CPU version of the reference's own algorithm.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_POOL: ThreadPoolExecutor | None = None


def threads() -> int:
    return int(os.environ.get("QSB_CPU_THREADS", os.cpu_count() or 1))


def _pool() -> ThreadPoolExecutor:
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(threads())
    return _POOL


def apply_1q_threaded(psi: np.ndarray, q: int, u: np.ndarray, block: int = 1 << 18) -> None:
    """In-place 2x2 on qubit q of psi, blocked over pair ranges and threads."""
    step = 1 << q
    v = psi.reshape(-1, 2, step)  # [blocks, side, offset]
    nb = v.shape[0]
    u00, u01, u10, u11 = u[0, 0], u[0, 1], u[1, 0], u[1, 1]

    def work(sl0, sl2):
        a = v[sl0, 0, sl2]
        b = v[sl0, 1, sl2]
        na = u00 * a + u01 * b
        nb_ = u10 * a + u11 * b
        v[sl0, 0, sl2] = na
        v[sl0, 1, sl2] = nb_

    tasks = []
    if nb * step // max(nb, 1) >= block or nb == 1:
        # few large blocks: split the offset axis
        per = max(1, block)
        for i in range(nb):
            for j in range(0, step, per):
                tasks.append((slice(i, i + 1), slice(j, min(step, j + per))))
    else:
        rows = max(1, block // step)
        for i in range(0, nb, rows):
            tasks.append((slice(i, min(nb, i + rows)), slice(0, step)))
    list(_pool().map(lambda t: work(*t), tasks))


def apply_controlled_threaded(psi: np.ndarray, control: int, target: int, u: np.ndarray,
                              block: int = 1 << 18) -> None:
    """In-place 2x2 on `target` over the amplitudes with `control` = 1
    (statevector.py:180-195: the same ufunc expression on the control=1
    pairs), on strided views split over host threads."""
    hi, lo = max(control, target), min(control, target)
    n = int(np.log2(psi.size))
    v = psi.reshape(1 << (n - hi - 1), 2, 1 << (hi - lo - 1), 2, 1 << lo)
    sub = v[:, 1] if control == hi else v[:, :, :, 1]  # control = 1
    # target axis: 2 (lo) of (A, M, L, B) or 1 (hi) of (A, H, M, B)
    tax = 2 if control == hi else 1
    u00, u01, u10, u11 = u[0, 0], u[0, 1], u[1, 0], u[1, 1]

    def work(sl):
        s = sub[sl]
        a = s.take(0, axis=tax)
        b = s.take(1, axis=tax)
        na = u00 * a + u01 * b
        nb = u10 * a + u11 * b
        idx0 = [slice(None)] * 4
        idx1 = [slice(None)] * 4
        idx0[tax], idx1[tax] = 0, 1
        s[tuple(idx0)] = na
        s[tuple(idx1)] = nb

    # split the outermost axis (or the middle one when it is short)
    A = sub.shape[0]
    if A >= threads():
        step = max(1, A // (4 * threads()))
        tasks = [slice(i, min(A, i + step)) for i in range(0, A, step)]
        list(_pool().map(work, tasks))
    else:
        for i in range(A):
            s = sub[i:i + 1]
            M = s.shape[1] if tax == 2 else s.shape[2]
            ax = 1 if tax == 2 else 2
            step = max(1, M // (4 * threads()))

            def work_m(j, s=s, ax=ax, step=step):
                sl = [slice(None)] * 4
                sl[ax] = slice(j, min(M, j + step))
                t = s[tuple(sl)]
                a = t.take(0, axis=tax)
                b = t.take(1, axis=tax)
                na = u00 * a + u01 * b
                nb = u10 * a + u11 * b
                i0 = [slice(None)] * 4
                i1 = [slice(None)] * 4
                i0[tax], i1[tax] = 0, 1
                t[tuple(i0)] = na
                t[tuple(i1)] = nb

            list(_pool().map(work_m, range(0, M, step)))
