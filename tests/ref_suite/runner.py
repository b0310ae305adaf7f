"""Run the fetched reference tests against the shim in a pytest subprocess
(their conftest.py and `import oracles` stay in their own directory; `qpool`
resolves to the alias package in tests/ref_suite/shim).  Test infrastructure."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
FETCHED = os.path.join(HERE, "_fetched")
SHIM = os.path.join(HERE, "shim")

# the reference modules that pin the hot path
MODULES = ["test_statevector.py", "test_distribution.py", "test_pool.py", "test_runtime.py",
           "test_circuit.py", "test_gates.py"]
# acceptance criteria 1-4: oracle equivalence on 1/2/4/8
# ranks, exchange accounting, allocation sizes, pool layouts
ACCEPTANCE = "test_acceptance.py"
ACCEPTANCE_K = "criterion_1 or criterion_2 or criterion_3 or criterion_4"
# host-only classes that need no CUDA device (run in the CPU suite too)
HOST_K = ("(TestGraphFile or TestParse or TestQaoaBuilder or TestRoundTrip or TestRankAndOffset "
          "or TestTopology or TestBuildPool or TestRandomStream or TestTreeSum or rotations "
          "or named_gates or custom_matrix or gate_matrix_rejects or full_state_bytes) and not "
          "(execution_before_binding or zero_angles_keep or single_edge_matches or "
          "sequential_noisy)")


def available() -> bool:
    return all(os.path.exists(os.path.join(FETCHED, f)) for f in MODULES + [ACCEPTANCE])


def run(args: list, timeout: float = 1500.0) -> subprocess.CompletedProcess:
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([SHIM, FETCHED, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir",
           FETCHED, "-rfE", *args]
    return subprocess.run(cmd, cwd=FETCHED, env=env, capture_output=True, text=True,
                          timeout=timeout)
