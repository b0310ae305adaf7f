"""The reference's own tests of the host-side pieces (tree sums, rank/offset
math, pool layouts, keyed random streams, gate matrices, the circuit and
graph formats) pass against the shim with no device (tests/ref_suite)."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_suite"))
import runner  # noqa: E402


@pytest.mark.skipif(not runner.available(), reason="reference suite not fetched "
                    "(python tests/ref_suite/fetch.py in the build container)")
def test_reference_host_tests_pass_on_the_shim():
    res = runner.run([*runner.MODULES, "-k", runner.HOST_K], timeout=600)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    assert " passed" in res.stdout
