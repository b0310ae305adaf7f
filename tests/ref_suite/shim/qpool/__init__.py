"""`qpool` alias of the B200 shim, for running the reference's own tests
against it (tests/test_gpu_ref_suite.py).  `import qpool.X` resolves to
paper_2001_10554_b200.X; nothing of the reference is imported."""
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

import paper_2001_10554_b200 as _shim  # noqa: E402
from paper_2001_10554_b200 import *  # noqa: E402,F401,F403

for _name in ("statevector", "distribution", "runtime", "pool", "gates", "graphs", "circuit",
              "noise", "optimize", "transport", "cli"):
    _mod = __import__(f"paper_2001_10554_b200.{_name}", fromlist=["_"])
    sys.modules[f"qpool.{_name}"] = _mod
    globals()[_name] = _mod
