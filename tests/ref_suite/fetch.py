"""Fetch the reference's own hot-path test suite for the drop-in check.

Run in the build container (the only place /root/reference exists; build()
calls it):

    python tests/ref_suite/fetch.py

It copies, unchanged, the reference test modules that pin the hot path
(test_statevector, test_distribution, test_pool,
test_runtime, test_circuit, test_gates, test_acceptance, with their
oracles.py and conftest.py) into tests/ref_suite/_fetched/.  That directory is
git-ignored -- the reference's tests are not part of this repository's
history -- but it travels to the GPU box with the working tree, where
tests/test_gpu_ref_suite.py runs it against the shim through the `qpool`
alias package in tests/ref_suite/shim.  Test infrastructure only.
"""
from __future__ import annotations

import os
import shutil
import sys

SRC = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
DST = os.path.join(HERE, "_fetched")
FILES = ["conftest.py", "oracles.py", "test_statevector.py", "test_distribution.py",
         "test_pool.py", "test_runtime.py", "test_circuit.py", "test_gates.py",
         "test_acceptance.py"]


def fetch() -> bool:
    if not os.path.isdir(SRC):
        return False
    os.makedirs(DST, exist_ok=True)
    for name in FILES:
        shutil.copyfile(os.path.join(SRC, name), os.path.join(DST, name))
    with open(os.path.join(DST, "SOURCE"), "w") as fh:
        fh.write(f"copied from {SRC} by tests/ref_suite/fetch.py; not tracked by git\n")
    return True


if __name__ == "__main__":
    ok = fetch()
    print("fetched" if ok else f"{SRC} not present; nothing fetched", file=sys.stderr)
