/*
 * qsb200.h -- C ABI of the B200-native state-vector core (libqsb200.so).
 *
 * This is the drop-in boundary for the hot path of arXiv 2001.10554 as
 * implemented by the `qpool` reference (pure Python/numpy).  The reference has
 * no FFI; its "operator API" is the Python module surface of
 * qpool.statevector / qpool.distribution.  Each entry point
 * below names the reference function whose arithmetic it replaces.  The
 * Python shim `paper_2001_10554_b200` binds these with ctypes and keeps the
 * reference names, argument meaning and exception types.
 *
 * Conventions
 *  - Amplitudes are complex128, interleaved (re, im) doubles: numpy's memory
 *    layout, so `array.view(np.float64)` crosses the ABI without a copy.
 *  - A 2x2 gate matrix is 8 doubles: u00.re u00.im u01.re u01.im u10.re
 *    u10.im u11.re u11.im (C order of a (2,2) complex128 array).
 *  - Qubit 0 is the least-significant index bit.  One handle holds
 *    `num_states` independent partitions ("pool" mode) of 2^m amplitudes
 *    each, contiguous, state-major.  Rank r of a 2^p-rank group owns global
 *    indices [r*2^m, (r+1)*2^m) (reference distribution.py:60-65).
 *  - Every function returns a status (QS_OK == 0).  On failure
 *    qs_last_error() returns a thread-local message.  Kernel launches are
 *    stream-ordered on the handle's own CUDA stream; downloads and
 *    observables synchronise.  There is no CPU fallback: without a CUDA
 *    device every compute entry point fails with QS_ERR_CUDA.
 */
#ifndef QSB200_H
#define QSB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSB200_ABI_VERSION 2  /* 2: QS_FUSE_FACTORED, qs_decompose_2x2 */

/* status codes -- the Python shim maps them to the reference exceptions */
#define QS_OK            0
#define QS_ERR_VALUE     1   /* ValueError      (statevector.py:129-130,170-171,184-187) */
#define QS_ERR_LOCALITY  2   /* LocalityError   (statevector.py:25-26,165-169,186-187)   */
#define QS_ERR_CUDA      3   /* RuntimeError    (no device / launch failure)             */
#define QS_ERR_COMM      4   /* TransportError  (transport.py:44-46)                      */
#define QS_ERR_NOMEM     5   /* MemoryError                                               */

/* gate kinds for qs_gate.kind */
#define QS_KIND_1Q        0  /* 2x2 on `target`            statevector.py:162-177        */
#define QS_KIND_CTRL      1  /* 2x2 on `target` if `control` statevector.py:180-195      */
#define QS_KIND_CUTPHASE  2  /* psi_i *= lut[cut(i)]        statevector.py:198-206 with
                                                            runtime.py:131-133, graphs.py:35-42 */

/* observable kinds for qs_observable */
#define QS_OBS_NORM    0     /* statevector.py:209-212 */
#define QS_OBS_PROB    1     /* statevector.py:215-231 */
#define QS_OBS_Z       2     /* statevector.py:234-242 */
#define QS_OBS_MAXCUT  3     /* statevector.py:245-251 */

typedef struct qs_state qs_state;

/* One gate of a program.  `offset` indexes `mats` (in doubles) for state 0;
 * state s uses offset + s*stride (stride 0 = same entry for every state).
 * For QS_KIND_1Q / QS_KIND_CTRL an entry is 8 doubles (2x2 matrix); for
 * QS_KIND_CUTPHASE it is the (num_edges+1)-entry complex LUT
 * lut[k] = exp(-1j * gamma * k) computed by the host with numpy. */
typedef struct qs_gate {
    int32_t  kind;
    int32_t  target;
    int32_t  control;   /* -1 when uncontrolled */
    int32_t  reserved;
    uint64_t offset;
    uint64_t stride;
} qs_gate;

/* ---- library ---------------------------------------------------------- */
int         qs_abi_version(void);
const char* qs_last_error(void);
int         qs_device_count(int32_t* out);
/* Per-thread byte/message counters of the global-qubit exchange, mirroring
 * TransportCounters (transport.py:49-65): amplitudes moved between ranks. */
int         qs_counters(const qs_state* st, uint64_t* messages, uint64_t* amplitudes);
/* Process-wide count of host-blocking CUDA calls the library has made
 * (stream/event/device synchronisations).  No reference counterpart: it makes
 * the asynchrony of the global-qubit path testable (distribution.py:121-178
 * blocks in MPI-style send/recv; the B200 path must not block the host). */
uint64_t    qs_host_sync_count(void);

/* ---- state lifetime: replaces StatePartition + allocate_partition
 *      (statevector.py:74-115) ------------------------------------------- */
int qs_state_create(int32_t num_qubits, int32_t num_local_qubits, int32_t rank_index,
                    int32_t num_states, int32_t device, qs_state** out);
int qs_state_destroy(qs_state* st);
int qs_state_info(const qs_state* st, int32_t* num_qubits, int32_t* num_local_qubits,
                  int32_t* rank_index, int32_t* num_states, uint64_t* amps_per_state);
/* raw device pointer of the amplitudes (for peer mapping / inspection) */
int qs_state_device_ptr(const qs_state* st, void** out);
int qs_synchronize(qs_state* st);

/* host <-> device, `count` complex amplitudes starting at flat amplitude
 * index `offset` (state-major).  Pinned or pageable host memory. */
int qs_state_upload(qs_state* st, const double* host, uint64_t offset, uint64_t count);
int qs_state_download(qs_state* st, double* host, uint64_t offset, uint64_t count);

/* Step boundary for streamed workloads: download the whole handle into
 * host_out while uploading host_in in its place, pipelined in `chunk`-
 * amplitude pieces on two streams (full-duplex PCIe).  Both host buffers
 * should be pinned and must not alias. */
int qs_state_exchange_host(qs_state* st, const double* host_in, double* host_out,
                           uint64_t chunk);

/* ---- initialisation: statevector.py:123-141 --------------------------- */
int qs_init_zero(qs_state* st);
int qs_init_basis(qs_state* st, uint64_t global_index);            /* init_basis_state */
int qs_init_constant(qs_state* st, double re, double im);           /* init_uniform: host passes 2**(-n/2) */
/* i.i.d. N(0,1) re/im from a counter-based generator keyed by (seed, global
 * index): identical for any rank split (not the numpy stream; unnormalised). */
int qs_init_gaussian(qs_state* st, uint64_t seed);
int qs_scale(qs_state* st, double factor);
/* apply_diagonal_phase with an arbitrary phase function (statevector.py:
 * 198-206): the caller evaluates exp(-1j * phases(owned_indices)) on the host
 * (the reference's own numpy expression) and passes the complex factors of
 * amplitudes [offset, offset + count); the device multiplies them in with
 * numpy's complex product.  Staged through device scratch in chunks. */
/* Numerics diagnostic (bench numerics_error, factored-vs-exact parity):
 * out[0] = max|a-b|, out[1] = sum|a-b|^2, out[2] = sum|b|^2, out[3] = max|b|
 * over all amplitudes of two same-shape states on one device. */
int qs_state_diff(qs_state* a, const qs_state* b, double* out);
int qs_apply_diagonal(qs_state* st, const double* factors, uint64_t offset, uint64_t count);

/* ---- gates ------------------------------------------------------------- */
/* apply_local_one_qubit_gate (statevector.py:162-177), one matrix per state
 * (`u_stride` doubles apart; 0 = one matrix for all states). */
int qs_apply_1q(qs_state* st, int32_t q, const double* u, uint64_t u_stride);
/* apply_local_controlled_gate (statevector.py:180-195): control-mask
 * compaction touches only the control=1 half; for CPhase-like matrices
 * diag(1, z) only the control=1, target=1 quarter is written (the target=0
 * amplitude is written back only if a signed zero changed it). */
int qs_apply_controlled(qs_state* st, int32_t control, int32_t target,
                        const double* u, uint64_t u_stride);
/* apply_diagonal_phase with gamma*cut_counts (statevector.py:198-206,
 * runtime.py:131-133): edges is 2*num_edges vertex ids, lut as in qs_gate. */
int qs_apply_cut_phase(qs_state* st, const int32_t* edges, int32_t num_edges,
                       const double* lut, uint64_t lut_stride);
/* A sequence of gates in program order (runtime.run_circuit, runtime.py:155-162).
 * fuse == QS_FUSE_NONE: one streaming kernel per gate.
 * fuse == QS_FUSE_EXACT: the native planner groups consecutive gates into
 *   shared-memory tile passes (one HBM read+write per pass); per-amplitude
 *   arithmetic and order are unchanged, so results are bit-identical to
 *   QS_FUSE_NONE and to the reference's numpy arithmetic.
 * fuse == QS_FUSE_FACTORED: as EXACT, after a rewrite of every uncontrolled
 *   shared-matrix 1q unitary into k*diag(1,za)*R*diag(1,zb) (R a real
 *   rotation applied as a 4-FMA shear); the diagonals merge across the program
 *   into neighbouring gates and two product diagonals at its ends.  Same
 *   operator, about a quarter of the FP64 work, results within 1e-12 of the
 *   reference (north_star tolerance) but not bit-identical.  States with
 *   fewer than 12 local qubits run EXACT. */
#define QS_FUSE_NONE      0
#define QS_FUSE_EXACT     1
#define QS_FUSE_FACTORED  2
int qs_apply_program(qs_state* st, const qs_gate* gates, int32_t count,
                     const double* mats, uint64_t mats_len,
                     const int32_t* edges, int32_t num_edges, int32_t fuse);
/* init_uniform-style start (statevector.py:137-141) fused with the program:
 * every amplitude of every state is (re, im) before the first gate, whatever
 * the state held.  The result equals qs_init_constant followed by
 * qs_apply_program bit for bit; lean pool passes generate the constant in
 * registers instead of reading it (no fill, no tile loads in the first pass).
 * The Python runtime calls it for a program that starts with H on every qubit
 * of a freshly reset |0..0> (the QAOA pool circuits of optimize.py:172-216):
 * H^(x)n |0..0> is the constant fl(..fl(fl(1*h)*h)..*h), h = fl(1/sqrt 2), in
 * the reference's own arithmetic, so the fold keeps the exact mode bit-identical. */
int qs_apply_program_on_constant(qs_state* st, double re, double im,
                                 const qs_gate* gates, int32_t count,
                                 const double* mats, uint64_t mats_len,
                                 const int32_t* edges, int32_t num_edges, int32_t fuse);
/* Planner only, no device needed: first gate index of every pass the fused
 * program would launch (starts[0..min(cap, *npasses))).  QS_FUSE_FACTORED is
 * planned as QS_FUSE_EXACT here (its rewrite needs the matrices). */
int qs_plan_program(int32_t num_local_qubits, const qs_gate* gates, int32_t count, int32_t fuse,
                    int32_t* starts, int32_t cap, int32_t* npasses);
/* Number of HBM passes the last qs_apply_program launched (planner output). */
int qs_last_program_passes(const qs_state* st, int32_t* passes);
/* The factorisation QS_FUSE_FACTORED applies to one 2x2 unitary u (8 doubles):
 * u = k * diag(1, za) * R * diag(1, zb), R = [[c,-s],[s,c]] = scale *
 * [[1,-t],[t,1]] (scale = c, t = s/c).  out[10] = k.re k.im za.re za.im zb.re
 * zb.im 0 t scale 0.  Returns QS_ERR_VALUE when u is not unitary to 1e-12,
 * exactly diagonal or has c < 1e-9 (those stay unfactored). */
int qs_decompose_2x2(const double* u, double* out);

/* ---- observables: per-state partial sums in the reference's tree order
 *      (statevector.py:29-45, 209-251); out has num_states doubles ------- */
int qs_observable(qs_state* st, int32_t kind, int32_t q, const int32_t* edges,
                  int32_t num_edges, double* out);

/* All per-qubit probabilities P(q=1), q < n, of every state in one pass
 * (cmd_run's report, cli.py:161-172); out has num_states*n doubles, each
 * bit-identical to qs_observable(QS_OBS_PROB, q). */
int qs_marginals(qs_state* st, double* out);

/* ---- host parameter preparation: noise trajectories (noise.py:70-80) ----
 * out[s] = a[s] @ b[s] for `count` complex128 2x2 matrices (row-major,
 * interleaved re/im).  Each entry is the FMA chain
 *   re = fma(-ai1,bi1, fma(ar1,br1, fma(-ai0,bi0, fma(ar0,br0, 0))))
 *   im = fma( ai1,br1, fma(ar1,bi1, fma( ai0,br0, fma(ar0,bi0, 0))))
 * -- the association numpy's `@` (OpenBLAS zgemm) used when the reference's
 * golden noise trajectories were generated -- so noise matrices, and the
 * noisy states built from them, are bit-identical on any host.  Host-only. */
int qs_compose_2x2(const double* a, const double* b, int64_t count, double* out);

/* Philox4x64-10 blocks (Random123; numpy's Philox bit generator, which the
 * reference's RandomStream draws from, pool.py:70): for i < count,
 * out[4i..4i+3] = philox(key = keys[2i..2i+1], counter = (ctr[2i], ctr[2i+1], 0, 0)).
 * Host-only; lets a pool round draw all its noise angles in one call. */
int qs_philox4x64(const uint64_t* keys, const uint64_t* ctr, int64_t count, uint64_t* out);

/* ---- global-qubit path: distribution.py:121-230 ----------------------- */
/* Pairwise exchange gate for a target on a global qubit, computed in one
 * kernel over NVLink peer memory: this rank updates half of the pairs it
 * shares with `peer` (the partner's partition, mapped with
 * qs_peer_open or another handle on the same device) and writes both
 * members.  is_lower: this rank holds the i_q=0 side.  control_local >= 0
 * restricts the update to offsets whose local control bit is 1 (case (c),
 * distribution.py:229-230).  The caller orders the call between two
 * partner barriers (both ranks call it; the pair sets are disjoint). */
int qs_exchange_gate_peer(qs_state* st, void* peer_amps, int32_t is_lower,
                          const double* u, int32_t control_local);
/* The reference's own three-step half-buffer exchange (Fig. 3,
 * distribution.py:121-178) over NCCL send/recv, chunked (chunk amplitudes
 * per message) and double-buffered; requires qs_comm_init. */
int qs_exchange_gate_nccl(qs_state* st, int32_t peer_rank, int32_t is_lower,
                          const double* u, int32_t control_local, uint64_t chunk);
/* Qubit remapping: SWAP the physical position of a global
 * qubit (this rank's bit value rank_bit; the partner is the handle behind
 * peer_amps) with local qubit local_qubit -- half the state crosses NVLink
 * (2^(m-1) amplitudes each way, half of a Fig. 3 exchange) and the gate
 * that needed the global qubit then runs locally (fusable).  qs_swap_qubits_local
 * swaps two local positions (used to restore the canonical layout). */
int qs_swap_qubits_peer(qs_state* st, void* peer_amps, int32_t local_qubit, int32_t rank_bit);
int qs_swap_qubits_local(qs_state* st, int32_t a, int32_t c);
/* CUDA IPC for peer mapping across processes (64-byte handles). */
/* Cross-rank ordering of peer exchange kernels without host stream syncs
 * (distribution._ordered_peer_op): every handle has two interprocess events
 * (0: recorded before its exchange, 1: after).  A rank records its own, the
 * pair meets on the host, and each stream waits on the partner's event, so the
 * exchange queues behind the local passes and the host never blocks.
 * qs_sync_event hands out the event itself (partner in the same process),
 * qs_sync_event_ipc its 64-byte IPC handle, qs_sync_event_open opens a
 * partner's handle (closed with the state).  qs_stream_busy: 1 while the
 * handle's stream still has queued work (cudaStreamQuery). */
int qs_sync_event(qs_state* st, int32_t which, void** ev);
int qs_sync_event_ipc(qs_state* st, int32_t which, unsigned char* handle64);
int qs_sync_event_open(qs_state* st, const unsigned char* handle64, void** ev);
int qs_sync_event_record(qs_state* st, int32_t which);
int qs_stream_wait_event(qs_state* st, void* ev);
int qs_stream_busy(qs_state* st, int32_t* busy);
int qs_state_ipc_handle(const qs_state* st, unsigned char* handle64);
int qs_peer_open(qs_state* st, const unsigned char* handle64, void** peer_amps);
int qs_peer_close(qs_state* st, void* peer_amps);
/* NCCL communicator (libnccl.so.2 is loaded lazily with dlopen). */
int qs_nccl_unique_id(unsigned char* id128);
int qs_comm_init(qs_state* st, const unsigned char* id128, int32_t nranks, int32_t rank);
int qs_comm_destroy(qs_state* st);

/* ---- timing helpers for the benchmark: events on the handle's stream ---- */
int qs_event_record(qs_state* st, int32_t slot);
int qs_event_elapsed_ms(qs_state* st, int32_t slot_a, int32_t slot_b, float* ms);
/* Per-launch log: with enable != 0 every kernel launch is bracketed by CUDA
 * events; qs_launch_log_read returns (and clears) durations in ms and kind
 * codes (1 gate1q, 2 controlled, 3 cut phase, 4 tile pass (k_tile), 5 exchange,
 * 6 reduction, 7 lean factored pass (k_fact*), 8 lean factored pass with a
 * generated constant input -- write-only, qs_apply_program_on_constant,
 * 9 CNOT-only pass of a factored program as one permutation (k_perm)). */
int qs_launch_log(qs_state* st, int32_t enable);
int qs_launch_log_read(qs_state* st, float* ms, int32_t* kinds, int32_t cap, int32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* QSB200_H */
