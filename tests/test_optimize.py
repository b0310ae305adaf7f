"""PSO driver pieces (optimize.py) against the reference's own outputs
(tests/golden/golden_optimize.npz): keyed-stream 3-regular graphs, exact
MaxCut and swarm trajectories in both sign modes -- bit for bit, no GPU."""
import numpy as np
import pytest

from paper_2001_10554_b200 import optimize as opt
from paper_2001_10554_b200.noise import RandomStream

from conftest import golden

SEED = 20260809


@pytest.mark.parametrize("n,key", [(4, 0), (8, 1), (12, 2), (20, 3)])
def test_random_3regular_graph_and_exact_maxcut(n, key):
    g = golden("golden_optimize.npz")
    graph = opt.random_3regular_graph(n, RandomStream(SEED, "pool", key))
    assert np.array_equal(np.array(graph.edges), g[f"edges_{n}"])
    assert opt.exact_maxcut(graph) == int(g[f"exact_{n}"])
    assert all(d == 3 for d in np.bincount(np.array(graph.edges).ravel(), minlength=n))


@pytest.mark.parametrize("sign", ["standard", "paper"])
def test_swarm_trajectory_bit_exact(sign):
    g = golden("golden_optimize.npz")
    sw = opt.init_swarm(5, 4, opt.PsoHyperparams(sign=sign), RandomStream(SEED, "pool", 9))
    for step, vals in enumerate(g[f"{sign}_values"]):
        opt.step_swarm(sw, vals)
        pos = np.stack([p.position for p in sw.particles])
        vel = np.stack([p.velocity for p in sw.particles])
        assert np.array_equal(pos, g[f"{sign}_pos"][step]), step
        assert np.array_equal(vel, g[f"{sign}_vel"][step]), step
        assert sw.global_best_value == g[f"{sign}_gbest"][step]
    assert sw.steps_taken == len(g[f"{sign}_values"])


def test_validation_and_trace_format():
    with pytest.raises(ValueError):
        opt.PsoHyperparams(sign="odd")
    with pytest.raises(ValueError):
        opt.init_swarm(0, 2)
    with pytest.raises(ValueError):
        opt.random_3regular_graph(5, RandomStream(1, "pool"))
    sw = opt.init_swarm(3, 2, stream=RandomStream(1, "pool"))
    with pytest.raises(ValueError):
        opt.step_swarm(sw, [0.1, 0.2])
    lines = opt.trace_csv_lines([opt.TraceRow(4, 0.5, 0), opt.TraceRow(8, 0.75, 1)])
    assert lines == ["evaluations,global_best_ratio,step", "4,0.5,0", "8,0.75,1"]
    tabs = opt.qaoa_slot_tables(np.array([[0.1, 0.2, 0.3, 0.4]]), 2)
    assert tabs["gamma2"][0] == 0.2 and tabs["beta1"][0] == 2.0 * 0.3
