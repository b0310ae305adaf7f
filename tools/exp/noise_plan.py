"""Pass plan and per-pass times of the noise-ensemble pool program (512
trajectories of the noisy config-5 QAOA circuit, bench.py --workload noise)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2001_10554_b200 import noise, runtime  # noqa: E402

seed, S = 20260809, 512
graph, circ = bench.noise_instance(seed)
model = noise.NoiseModel(bench.NOISE_T1, bench.NOISE_T2)
ctx = runtime.make_context(None, 20, num_states=S, fuse="factored", seed=seed, noise_model=model)
ctx.norm_check_interval = 0
durations = [g.duration for g in circ.gates if g.kind == "noise"]
batch = noise.StreamBatch(noise.trajectory_stream(seed, s) for s in range(S))
mats = noise.circuit_noise_matrices(durations, model, batch)
for k in range(2):
    runtime.reset_state(ctx)
    if k:
        ctx.state.synchronize()
        ctx.state.launch_log(True)
    runtime.run_circuit(ctx, circ, noise_matrices=mats)
    ctx.state.synchronize()
ctx.state.launch_log(False)
ms, kinds = ctx.state.read_launch_log()
print("passes", list(zip(kinds.tolist(), np.round(ms, 3).tolist())), "total", round(float(ms.sum()), 2))
