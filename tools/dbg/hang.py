"""Debug: criterion-1 style circuits on 2/4/8 emulated ranks with a stack dump on hang."""
import faulthandler
import sys
import os
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
faulthandler.dump_traceback_later(40, exit=True)
import numpy as np
from paper_2001_10554_b200 import runtime
from test_gpu_acceptance import random_circuit
from oracle import circuit as ocirc

rng = np.random.default_rng(20260401)
t0 = time.time()
for trial in range(100):
    circ, plain = random_circuit(8, 50, rng)
    expected = ocirc.run(8, plain)
    for ranks in (1, 2, 4, 8):
        got = runtime.simulate_circuit(circ, num_ranks=ranks, timeout=20)
        d = float(np.max(np.abs(got - expected)))
        if d > 1e-12:
            print("BAD", trial, ranks, d)
    faulthandler.cancel_dump_traceback_later()
    faulthandler.dump_traceback_later(40, exit=True)
print("ok", time.time() - t0)
