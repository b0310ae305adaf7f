"""Noise trajectories, host side (no GPU): the vectorised Philox stream, the
noise matrices and schedule_noise against numpy's own generator, the oracle
and the reference's golden trajectories (tests/golden/golden_noise.npz)."""
import math

import numpy as np
import pytest

from paper_2001_10554_b200 import noise as N
from paper_2001_10554_b200.runtime import noise_ensemble_csv

from conftest import bits_equal
from noise_fixture import load, to_circuit
from oracle import circuit as ocirc
from oracle import noise as onoise


def test_philox_matches_numpy_word_for_word():
    rng = np.random.default_rng(11)
    keys = rng.integers(0, 2**63, size=(64, 2), dtype=np.uint64)
    keys[::3, 1] |= np.uint64(1 << 63)     # high words
    keys[1::3, 0] |= np.uint64(1 << 63)
    ctr = rng.integers(0, 2**40, size=64, dtype=np.uint64)
    ctr[:4] = [0, 1, 3, 4]
    for count in (1, 3, 4, 5, 11):
        got = N.philox4x64_uniform(keys, ctr, count)
        for i in range(64):
            bg = np.random.Philox(counter=np.array([ctr[i], 0, 0, 0], dtype=np.uint64),
                                  key=keys[i])
            assert np.array_equal(got[i], np.random.Generator(bg).random(count)), (i, count)


def test_random_stream_matches_oracle_scalar_path():
    for t in range(40):  # keys above and below 2^63 (float64 key quirk)
        mine, ref = N.trajectory_stream(20260809, t), onoise.TrajectoryStream(20260809, t)
        for _ in range(3):
            assert np.array_equal(mine.normal(3), ref.normal(3))
    assert mine.counter == 9


def test_stream_batch_equals_member_streams():
    streams = [N.trajectory_stream(5, t) for t in range(17)]
    twins = [N.trajectory_stream(5, t) for t in range(17)]
    batch = N.StreamBatch(streams)
    for _ in range(4):
        d = batch.normal(3)
        assert np.array_equal(d, np.stack([s.normal(3) for s in twins]))
    assert [s.counter for s in streams] == [12] * 17


@pytest.mark.parametrize("duration", [0.0, 0.5, 1.0, 7.25])
def test_noise_matrices_bit_equal_oracle(duration):
    model = N.NoiseModel(20.0, 15.0)
    S = 64
    got = N.noise_gate_matrices(duration, model, N.StreamBatch(
        N.trajectory_stream(3, t) for t in range(S)))
    for t in range(S):
        ref = onoise.noise_matrix(duration, 20.0, 15.0, onoise.TrajectoryStream(3, t))
        assert bits_equal(got[t], ref), t
    one = N.noise_gate_matrix(duration, model, N.trajectory_stream(3, 5))
    assert bits_equal(one, got[5])


def test_noiseless_model_gives_identity_rotations():
    u = N.noise_gate_matrix(3.0, N.NOISELESS, N.trajectory_stream(1, 0))
    assert np.array_equal(np.abs(u), np.eye(2))


def test_noise_model_validation():
    with pytest.raises(ValueError):
        N.NoiseModel(0.0, 1.0)
    with pytest.raises(ValueError):
        N.NoiseModel(1.0, 2.5)
    with pytest.raises(ValueError):
        N.NoiseModel(1.0, 1.0).variances(-1.0)
    vxy, vz = N.NoiseModel(20.0, 15.0).variances(2.0)
    assert vxy == 2.0 / 20.0 and vz == 2.0 * 2.0 * (1.0 / 15.0 - 1.0 / 40.0)
    assert N.NOISELESS.variances(1.0) == (0.0, 0.0)


def test_schedule_noise_matches_reference_schedule():
    glist, _, _, _, _ = load()
    base = to_circuit(glist, with_noise=False)
    sched = N.schedule_noise(base)
    assert len(sched.gates) == len(glist)
    for g, ref in zip(sched.gates, glist):
        assert g.kind == ref["kind"] and tuple(g.qubits) == tuple(ref["qubits"])
        if g.kind == "noise":
            assert g.duration == ref["duration"]
    with pytest.raises(ValueError):
        N.schedule_noise(sched)


def test_schedule_noise_covers_idle_qubits():
    from paper_2001_10554_b200.circuit import Circuit, GateSpec

    c = N.schedule_noise(Circuit(3, (GateSpec("h", (0,)), GateSpec("x", (0,)))))
    noise = [(g.qubits[0], g.duration) for g in c.gates if g.kind == "noise"]
    # per qubit, the noise durations sum to the covered time plus the tail
    assert noise == [(0, 1.0), (0, 1.0), (0, 1.0), (1, 2.0), (2, 2.0)]


def test_oracle_trajectories_pin_to_golden():
    glist, states, t1, t2, seed = load()
    for t in range(states.shape[0]):
        out = ocirc.run(12, onoise.bind_trajectory(glist, t1, t2, seed, t))
        assert bits_equal(out, states[t]), t


def test_noise_ensemble_csv_format():
    csv = noise_ensemble_csv([1.0, 0.0, 0.5], 0.25)
    assert csv.splitlines() == ["trajectories,running_mean,reference", "1,1.0,0.25",
                                "2,0.5,0.25", "3,0.5,0.25"]
    assert math.isclose(float(csv.splitlines()[-1].split(",")[1]), 0.5)


def test_native_philox_equals_numpy_restatement():
    rng = np.random.default_rng(4)
    k = rng.integers(0, 2**64 - 1, size=(300, 2), dtype=np.uint64)
    c = rng.integers(0, 2**64 - 1, size=(300, 2), dtype=np.uint64)
    a = N._philox_block(k[:, 0], k[:, 1], c[:, 0], c[:, 1])
    b = N.philox_block_numpy(k[:, 0], k[:, 1], c[:, 0], c[:, 1])
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_circuit_noise_matrices_equal_gate_by_gate_draws():
    model = N.NoiseModel(20.0, 15.0)
    durs = np.random.default_rng(0).uniform(0, 5, size=37)
    b1 = N.StreamBatch(N.trajectory_stream(1, t) for t in range(9))
    b2 = N.StreamBatch(N.trajectory_stream(1, t) for t in range(9))
    got = N.circuit_noise_matrices(durs, model, b1)
    ref = np.stack([N.noise_gate_matrices(d, model, b2) for d in durs])
    assert bits_equal(got, ref)
    assert [s.counter for s in b1.streams] == [3 * 37] * 9
    s1, s2 = N.trajectory_stream(1, 3), N.trajectory_stream(1, 3)
    one = N.circuit_noise_matrices(durs[:5], model, s1)
    assert bits_equal(one, np.stack([N.noise_gate_matrix(d, model, s2) for d in durs[:5]]))
