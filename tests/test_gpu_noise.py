"""GPU parity for noise trajectories (noise.py, cli.py:288-339): noisy states
through the CUDA path are bit-identical to the reference's own trajectories
(tests/golden/golden_noise.npz) on one state, on a pool of states (per-state
tables in one fused program) and across emulated ranks."""
import numpy as np
import pytest

from paper_2001_10554_b200 import noise as N
from paper_2001_10554_b200 import runtime

from conftest import bits_equal
from noise_fixture import load, to_circuit
from oracle import circuit as ocirc
from oracle import noise as onoise

pytestmark = pytest.mark.gpu


def test_single_state_trajectories_match_golden():
    glist, states, t1, t2, seed = load()
    circ = to_circuit(glist)
    ctx = runtime.make_context(None, 12, noise_model=N.NoiseModel(t1, t2))
    for t in range(states.shape[0]):
        runtime.reset_state(ctx)
        runtime.run_circuit(ctx, circ, noise_stream=N.trajectory_stream(seed, t))
        assert bits_equal(ctx.state.download(), states[t]), t


def test_pool_trajectories_match_golden_in_one_program():
    glist, states, t1, t2, seed = load()
    circ = to_circuit(glist)
    S = states.shape[0]
    ctx = runtime.make_context(None, 12, S, noise_model=N.NoiseModel(t1, t2))
    batch = N.StreamBatch(N.trajectory_stream(seed, t) for t in range(S))
    runtime.run_circuit_pool(ctx, circ, noise_stream=batch)
    assert bits_equal(ctx.pool.amplitudes(), states)
    # the context's default state streams are trajectories 0..S-1 (state scope)
    ctx2 = runtime.make_context(None, 12, S, seed=seed, noise_model=N.NoiseModel(t1, t2))
    runtime.run_circuit(ctx2, circ)
    assert bits_equal(ctx2.pool.amplitudes(), states)


@pytest.mark.parametrize("P", [2, 4])
def test_distributed_trajectory_matches_golden(P):
    """Global-qubit noise gates go through the exchange path; every rank
    draws the same angles from the shared state stream."""
    glist, states, t1, t2, seed = load()
    circ = to_circuit(glist)

    def rank_fn(comm):
        ctx = runtime.make_context(comm, 12, noise_model=N.NoiseModel(t1, t2))
        ctx.norm_check_interval = 0
        runtime.run_circuit(ctx, circ, noise_stream=N.trajectory_stream(seed, 2))
        return ctx.state.download()

    out = np.concatenate(runtime.run_spmd(P, rank_fn, timeout=120.0))
    assert bits_equal(out, states[2])


def test_ensemble_is_layout_independent():
    """Trajectory t is the same whether it runs alone or as state t mod S of
    a pool (noise.py:60-69); the ensemble values agree bit for bit."""
    glist, _, t1, t2, seed = load()
    circ = to_circuit(glist, with_noise=False)  # run_noise_ensemble schedules it
    model = N.NoiseModel(t1, t2)
    T = 7

    def z0(ctx):
        return runtime.measure_z(ctx, 0)

    single = runtime.make_context(None, 12, seed=seed)
    ref1, v1 = runtime.run_noise_ensemble(single, circ, model, T, z0)
    pool = runtime.make_context(None, 12, 3, seed=seed)
    ref3, v3 = runtime.run_noise_ensemble(pool, circ, model, T, z0)
    assert ref1 == ref3
    assert np.array_equal(v1, v3)
    # two pools in turns (round k's values read back after round k+1 is enqueued):
    # the same values, for pool sizes that do and do not divide the ensemble
    for S in (3, 2):
        a = runtime.make_context(None, 12, S, seed=seed)
        b = runtime.make_context(None, 12, S, seed=seed)
        refp, vp = runtime.run_noise_ensemble(a, circ, model, T, z0, shadow=b)
        assert refp == ref1 and np.array_equal(vp, v1)
    with pytest.raises(ValueError):
        runtime.run_noise_ensemble(single, circ, model, T, z0, shadow=pool)
    # against the oracle's scalar path for two trajectories
    sched = N.schedule_noise(circ)
    glist_s = [{"kind": g.kind, "qubits": g.qubits, "param": g.param, "duration": g.duration}
               for g in sched.gates]
    for t in (0, 6):
        psi = ocirc.run(12, onoise.bind_trajectory(glist_s, t1, t2, seed, t))
        p1 = np.sum(np.abs(psi[1::2]) ** 2)
        assert abs(v1[t] - (1.0 - 2.0 * p1)) < 1e-10
    # the noiseless reference is the ideal circuit's value
    ideal = ocirc.run(12, [g for g in glist_s if g["kind"] != "noise"])
    assert abs(ref1 - (1.0 - 2.0 * np.sum(np.abs(ideal[1::2]) ** 2))) < 1e-10


def test_split_pool_ensemble_equals_one_pool():
    """Two contexts holding pool groups [0,2) and [2,4) of a 4-group ensemble
    (split_pool over two ranks) produce the same values as one 4-state pool."""
    glist, _, t1, t2, seed = load()
    circ = to_circuit(glist)
    model = N.NoiseModel(t1, t2)
    T = 10
    obs = lambda ctx: runtime.measure_norm_squared(ctx)  # noqa: E731
    whole = runtime.make_context(None, 12, 4, seed=seed)
    _, vw = runtime.run_noise_ensemble(whole, circ, model, T, lambda c: runtime.measure_z(c, 3))
    parts = []
    for r in range(2):
        first, count = runtime.split_pool(4, r, 2)
        ctx = runtime.make_context(None, 12, count, seed=seed, state_offset=first)
        parts.append(runtime.run_noise_ensemble(ctx, circ, model, T,
                                                lambda c: runtime.measure_z(c, 3),
                                                num_groups=4)[1])
    merged = np.where(np.isnan(parts[0]), parts[1], parts[0])
    assert not np.isnan(merged).any()
    assert np.array_equal(merged, vw)
    ref, norms = runtime.run_noise_ensemble(whole, circ, model, 4, obs)
    assert np.all(np.abs(norms - 1.0) < 1e-12)
