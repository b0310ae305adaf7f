"""B200-native state-vector core for the hot path of arXiv 2001.10554.

Drop-in for the reference package ``qpool`` on its hot path: the modules
``statevector``, ``distribution``, ``runtime``, ``gates``, ``graphs`` and
``pool`` keep the reference's names and semantics while the amplitudes live
in HBM and every update is a hand-written sm_100a kernel in libqsb200.so
(C ABI: include/qsb200.h).  No CPU fallback exists.
"""
from __future__ import annotations

from . import _native
from ._native import LocalityError, TransportError, device_count
from . import transport, gates, graphs, statevector, distribution, runtime, circuit, pool, noise, optimize  # noqa: E402
from .register import QubitRegister
from .statevector import (StatePartition, allocate_partition, full_state_bytes, init_basis_state,
                          init_uniform, apply_local_one_qubit_gate, apply_local_controlled_gate,
                          apply_diagonal_phase, apply_cut_phase, CutPhase, norm_squared,
                          get_probability, z_expectation, maxcut_expectation, tree_sum,
                          tree_sum_values)
from .distribution import (GroupComm, RankTopology, rank_and_offset, exchange_partner,
                           single_rank_comm, ThreadFabric, TorchComm, apply_one_qubit_gate,
                           apply_controlled_gate, group_reduce_sum)
from .transport import (InProcessFabric, SocketTransport, TorchTransport, Transport,
                        TransportCounters, TransportTimeout, write_rendezvous)
from .runtime import (NormDriftError, RankContext, make_context, reset_state, run_circuit,
                      run_circuit_pool, apply_gate, apply_gate_pool, measure_probability,
                      measure_probabilities, measure_maxcut, measure_z, measure_norm_squared,
                      gather_group_state, pool_sum, run_spmd, simulate_circuit, PoolState,
                      run_noise_ensemble, noise_ensemble_csv)
from .noise import (NoiseModel, NOISELESS, apply_noise_gate, noise_gate_matrix, schedule_noise,
                    trajectory_stream)
from .pool import (build_pool, PoolLayout, RandomStream, incoherent_sum_over_pool,
                   uniform_randoms)
from .graphs import Graph, cut_counts, load_graph, make_graph, parse_graph, serialize_graph
from .circuit import (Circuit, CircuitParseError, GateSpec, UnboundParameterError,
                      build_qaoa_circuit, load_circuit, parse_circuit, qaoa_bindings,
                      serialize_circuit)
from .optimize import (Particle, PsoHyperparams, Swarm, exact_maxcut, init_swarm,
                       random_3regular_graph, run_pso_qaoa, step_swarm, update_velocity)

__version__ = "0.1.0"


def load_library():
    """Load libqsb200.so (raises ImportError if it was not built)."""
    return _native.load()
