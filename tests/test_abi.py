"""The C-ABI library loads, exports exactly what include/qsb200.h declares,
fails loudly without a device, and its native planner (CPU-only entry point)
fuses as designed.  No kernel runs here."""
import os
import re
import subprocess

import pytest

from paper_2001_10554_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qsb200.h")


def header_functions():
    text = open(HEADER).read()
    return set(re.findall(r"^(?:int|const char\*|uint64_t)\s+(qs_\w+)\s*\(", text, flags=re.M))


def test_library_loads_and_version():
    lib = N.load()
    assert lib.qs_abi_version() == 2


def test_exports_match_header():
    declared = header_functions()
    assert declared == set(N.EXPORTS), declared ^ set(N.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (qs_\w+)", out))
    assert declared <= exported, declared - exported


def test_header_constants_match_binding():
    text = open(HEADER).read()
    consts = dict(re.findall(r"#define (QS_\w+)\s+(\d+)", text))
    assert int(consts["QS_ERR_VALUE"]) == N.QS_ERR_VALUE
    assert int(consts["QS_ERR_LOCALITY"]) == N.QS_ERR_LOCALITY
    assert int(consts["QS_ERR_CUDA"]) == N.QS_ERR_CUDA
    assert int(consts["QS_KIND_CUTPHASE"]) == N.QS_KIND_CUTPHASE
    assert int(consts["QS_OBS_MAXCUT"]) == N.QS_OBS_MAXCUT
    import ctypes
    assert N.QsGate.stride.offset == 24 and ctypes.sizeof(N.QsGate) == 32


@pytest.mark.skipif(N.device_count() > 0, reason="checks the no-device path")
def test_no_device_fails_loudly():
    with pytest.raises(N.NativeError, match="no CUDA device"):
        N.DeviceState(4, 4)
    import paper_2001_10554_b200 as qs
    with pytest.raises(N.NativeError):
        qs.allocate_partition(3)


def gates(*targets, kind=0):
    return [N.QsGate(kind, t, -1, 0, 0, 0) for t in targets]


def test_planner_sweep_passes():
    assert N.plan_program(30, gates(*range(30))) == [0, 12, 21]
    assert N.plan_program(30, gates(*range(30)), fuse=False) == list(range(30))
    # small states cannot hold a 2^12 tile: one launch per gate
    assert N.plan_program(10, gates(*range(10))) == list(range(10))


def test_planner_controls_and_phases_need_no_tile_bits():
    g = gates(20, 21, 22)
    g.append(N.QsGate(N.QS_KIND_CTRL, 23, 29, 0, 0, 0))   # control 29 stays outside the tile
    g.append(N.QsGate(N.QS_KIND_CUTPHASE, 0, -1, 0, 0, 0))
    g += gates(24, 25, 26, 27, 28)
    # targets 20..28 + qubits 0..2 = 12 tile bits: one pass
    assert N.plan_program(30, g) == [0]
    g += gates(19)
    assert N.plan_program(30, g) == [0, len(g) - 1]


def test_planner_rejects_nonlocal_target():
    with pytest.raises(ValueError):
        N.plan_program(12, gates(12))


def test_planner_round_limit_splits_long_passes():
    # alternating targets force a new register round per gate: passes split
    g = gates(*([3, 4, 5, 6, 7] * 30))
    starts = N.plan_program(20, g)
    assert starts[0] == 0 and len(starts) >= 2
    assert all(b > a for a, b in zip(starts, starts[1:]))
