// Shared declarations of the B200 state-vector core (libqsb200.so).
//
// Arithmetic contract: the reference evaluates
// pair_update (statevector.py:144-150) with numpy complex128 ufuncs, which on
// an FMA host compute x*y as (fma(xr,yr,-(xi*yi)), fma(xr,yi,xi*yr)) with the
// LEFT operand as x, then plain IEEE adds.  Every kernel here spells that out
// with __fma_rn/__dmul_rn/__dadd_rn so no contraction choice of the compiler
// can change a bit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/qsb200.h"

namespace qsb {

// ---- numpy-exact complex arithmetic ----------------------------------------
__device__ __forceinline__ double2 cmul(double2 x, double2 y) {
    return make_double2(__fma_rn(x.x, y.x, -__dmul_rn(x.y, y.y)),
                        __fma_rn(x.x, y.y, __dmul_rn(x.y, y.x)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
// (a, b) <- (u00 a + u01 b, u10 a + u11 b), statevector.py:150
__device__ __forceinline__ void pair_update(double2& a, double2& b, const double2 u[4]) {
    double2 na = cadd(cmul(u[0], a), cmul(u[1], b));
    double2 nb = cadd(cmul(u[2], a), cmul(u[3], b));
    a = na;
    b = nb;
}
// |psi|^2 as the reference evaluates it: a.real*a.real + a.imag*a.imag
// (separate ufuncs, no FMA; statevector.py:212)
__device__ __forceinline__ double abs2(double2 a) {
    return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
}

// insert a zero bit at position b
__host__ __device__ __forceinline__ uint64_t insert0(uint64_t x, int b) {
    uint64_t lowmask = (uint64_t(1) << b) - 1;
    return (x & lowmask) | ((x & ~lowmask) << 1);
}

// cut(i) = sum over edges of bit_u(i) xor bit_v(i) (graphs.py:35-42), grouped by
// vertex distance d = v-u: popc((i ^ (i >> d)) & mask_d).
constexpr int kMaxCutTerms = 64;
struct CutTerms {
    int32_t count;
    int32_t shift[kMaxCutTerms];
    uint64_t mask[kMaxCutTerms];
};
__device__ __forceinline__ int cut_of(uint64_t i, const CutTerms& ct) {
    int c = 0;
    for (int k = 0; k < ct.count; ++k) c += __popcll((i ^ (i >> ct.shift[k])) & ct.mask[k]);
    return c;
}

// Tile pass description for the fused kernel.  Everything the kernel needs
// per pass -- tile layout, register rounds, gate descriptors and shared 2x2
// matrices -- is copied to the device once per pass and staged into shared
// memory by each persistent CTA.
#ifndef QSB_TILE_LOG2
#define QSB_TILE_LOG2 12
#endif
#ifndef QSB_REG_LOG2
#define QSB_REG_LOG2 4
#endif
constexpr int kTileLog2 = QSB_TILE_LOG2;  // 2^12 amplitudes = 64 KiB of shared memory
constexpr int kRegLog2 = QSB_REG_LOG2;    // 16 amplitudes per thread = 4 register qubits
constexpr int kTileThreads = 1 << (kTileLog2 - kRegLog2);
// low qubits every tile keeps (2^kLowBits contiguous amplitudes = 16 << kLowBits
// bytes per HBM row segment)
#ifndef QSB_LOW_BITS
#define QSB_LOW_BITS 3
#endif
constexpr int kLowBits = QSB_LOW_BITS;
constexpr uint64_t kLowMask = (uint64_t(1) << kLowBits) - 1;
constexpr int kLaneLoBits = 4;
constexpr int kLaneHiBits = kTileLog2 - kRegLog2 - kLaneLoBits;
constexpr int kMaxRounds = 24;
constexpr int kMaxPassGates = 64;
constexpr int kMaxPassDiags = 4;

// swizzle of a tile element index into its shared-memory slot; linear over
// GF(2), so swz(a ^ b) == swz(a) ^ swz(b)
__host__ __device__ __forceinline__ int swz(int e) {
    return e ^ (((e >> 3) ^ (e >> 6) ^ (e >> 9) ^ (e >> 12)) & 7);
}

struct alignas(16) TileGate {
    double2 u[4];    // the matrix when stride == 0 (16-byte aligned: LDS.128 broadcasts)
    uint64_t offset; // per-state table (stride != 0) or LUT, in doubles
    uint64_t stride;
    int32_t kind;    // QS_KIND_*
    int32_t variant; // j (target register bit, uncontrolled) or kRegLog2 + kRegLog2*c + j
                     // (controlled by register bit c)
    int32_t ctype;   // 0 none | 1 register bit cval | 2 tile position cval (outside the
                     // round) | 3 local qubit cval outside the tile (tile-uniform)
    int32_t cval;
    int32_t seq;     // > 1 at the first gate of a run of `seq` uncontrolled gates on
                     // register bits 0,1,..,seq-1 in order (compiled fast path)
    int32_t pad[3];
};

struct Round {
    int16_t first_gate, num_gates;
    // tile-element deposits: thread id low/high bits into the positions not
    // held in registers, register index k into the round positions; the s*
    // tables are the same values swizzled
    uint16_t dlo[1 << kLaneLoBits], dhi[1 << kLaneHiBits], dk[1 << kRegLog2];
    uint16_t slo[1 << kLaneLoBits], shi[1 << kLaneHiBits], sk[1 << kRegLog2];
};

struct alignas(16) TilePass {
    int32_t m;                 // local qubits per state
    int32_t num_rounds;
    int32_t low_run;           // tile positions 0..low_run-1 are qubits 0..low_run-1
    int32_t direct_store;      // last round writes registers straight to HBM (coalesced)
    int32_t tile_bits[kTileLog2];  // ascending local qubit of each tile position
    uint64_t tiles_per_state;  // 2^(m - kTileLog2)
    uint64_t num_tiles;        // num_states * tiles_per_state
    uint64_t rank_offset;      // rank_index << m (global index of local offset 0)
    uint64_t zero_off;         // factored programs: a 0.0 in mats (lean-pass t padding)
    uint64_t nbr[64];          // cut-phase graph: neighbour mask of each vertex (qubit)
    Round rounds[kMaxRounds];
    TileGate gates[kMaxPassGates];
    // product diagonals (kKindDiagN, slot in TileGate.pad[0]): the factor of
    // register index k in the gate's round, prod_j z_{qubit of register j}^{k_j}
    double2 diag_r[kMaxPassDiags][1 << kRegLog2];
};

// ---- factored programs (fuse == QS_FUSE_FACTORED, factor.cu) ---------------
// Internal gate kinds the factored rewrite emits; they never appear in a user
// program.  Each 1q unitary U = k * diag(1, za) * R(c, s) * diag(1, zb) with R
// the real rotation [[c,-s],[s,c]] = c*[[1,-t],[t,1]] (t = s/c), so the pair
// update is a 4-FMA shear.  The diagonals commute with every gate not mixing
// their qubit, so they merge into the neighbouring gates' diagonals and, at the
// ends of the program, into one product diagonal over all qubits (D_in before
// everything, D_out with the scalars after everything).
constexpr int kKindShear = 16;  // params [t, 0, has_pre, 0, z.re, z.im, 0, 0]: b *= z (if
                                // has_pre), then (a, b) <- (a - t b, b + t a) on `target`
constexpr int kKindDiag1 = 17;  // params [0, 0, 0, 0, z.re, z.im, 0, 0]: amplitudes with bit
                                // `target` set *= z
constexpr int kKindDiagN = 18;  // psi_i *= prod_c T_c[byte c of i]; `reserved` = table count;
                                // offset -> ntab*256 complex byte tables, then 64 complex z_q
constexpr int kKindScalar = 19; // per-state scalar (stride 8): psi_s *= (params[0], params[1])
// kinds a lean factored pass (k_fact*) can hold; everything else runs on k_tile
inline bool kind_is_lean(int kind) {
    return kind == kKindShear || kind == kKindDiagN || kind == QS_KIND_CUTPHASE;
}
// a CNOT with one matrix for all states (exactly X): k_perm runs passes of these
inline bool gate_is_cnot(const qs_gate& g, const double* mats) {
    if (g.kind != QS_KIND_CTRL || g.stride != 0 || !mats) return false;
    const double* u = mats + g.offset;
    return u[0] == 0 && u[1] == 0 && u[2] == 1 && u[3] == 0 && u[4] == 1 && u[5] == 0 && u[6] == 0 &&
           u[7] == 0;
}
// pass classes of the lean-first schedule: 0 lean (k_fact*), 1 CNOT (k_perm), 2 other (k_tile)
inline int gate_class(const qs_gate& g, const double* mats) {
    return kind_is_lean(g.kind) ? 0 : gate_is_cnot(g, mats) ? 1 : 2;
}
inline bool kind_has_target(int kind) {
    return kind != QS_KIND_CUTPHASE && kind != kKindDiagN && kind != kKindScalar;
}

struct FactoredProgram {
    std::vector<qs_gate> gates;
    std::vector<double> extra;  // parameters/tables, addressed at mats_len + local offset
    int factored = 0;           // 1q gates turned into shears or absorbed as diagonals
    uint64_t zero_off = 0;      // a 0.0 in the extra entries (mats_len + local offset)
};
// Rewrites gates[0..count) (validated, all local) into `out`.  mats_len is the
// size of the caller's table (the extra entries are appended after it).
// batch_flush (large states, with schedule_program's lean_first): the pending
// diagonals of the targets of a run of controlled gates leave as one product
// diagonal before the run instead of one Diag1 per target.
void factor_program(const qs_gate* gates, int count, const double* mats, uint64_t mats_len, int m,
                    int num_states, int num_edges, uint64_t phase_support, FactoredProgram* out,
                    bool batch_flush = false);
// Commutation-aware re-order of a factored program for the pass planner
// (phase_support: the cut-phase graph's vertices).
// lean_first: passes of lean kinds only are kept free of the other kinds (which
// would move the whole pass from k_fact* to k_tile); worth an extra pass on
// large states.
void schedule_program(std::vector<qs_gate>& gates, int m, uint64_t phase_support,
                      const double* mats, int num_states, bool lean_first = false);
// U = k diag(1,za) R diag(1,zb): out = [k, za, zb] (complex), 0, t, scale (= c).
// Returns false when U is not unitary to 1e-12, exactly diagonal or c < 1e-9.
bool decompose_2x2(const double* u, double out[10]);

// ---- launchers (gate_kernels.cu / reduce_kernels.cu / exchange.cu) ---------
void launch_gate1q(double2* psi, int m, int num_states, int q, const double* mats,
                   uint64_t offset, uint64_t stride, cudaStream_t s);
void launch_controlled(double2* psi, int m, int num_states, int c, int t, const double* mats,
                       uint64_t offset, uint64_t stride, bool diag_one, cudaStream_t s);
void launch_cut_phase(double2* psi, int m, int num_states, uint64_t rank_offset,
                      const CutTerms& ct, const double* mats, uint64_t offset, uint64_t stride,
                      cudaStream_t s);
// qs_apply_program_on_constant: the program's input is `v` in every amplitude
// (`total` amplitudes).  The first pass either generates it in registers (lean
// pool passes on the TMA kernel) or is preceded by a fill; whoever does clears `on`.
struct ConstIn {
    bool on;
    double2 v;
    uint64_t total;
};
extern thread_local ConstIn g_const_in;
// A pass of CNOTs right behind a lean pass whose tile holds all its targets:
// the lean pass writes its tile back through shared memory and reads the copy-out
// through the composed permutation (GF(2)-linear smem addressing: no cost per
// amplitude), so the CNOT pass is never launched.  Set by the program loop
// (count > 0), `done` by the lean launcher that took it.
struct AbsorbCnots {
    int count;
    int controls[kMaxPassGates], targets[kMaxPassGates];
    bool done;
};
extern thread_local AbsorbCnots g_absorb;
// the pass can run on the TMA lean kernel with its tile written back through
// shared memory (what folding a CNOT pass into it needs)
bool absorb_tile_feasible(double2* psi, const TilePass& pass);
bool tile_pass_in_params();  // k_tile takes the pass as a kernel parameter
// returns 0: k_tile, 1: the lean factored kernels (k_fact*), 2: a lean pass that
// generated a constant input (g_const_in) instead of loading its tiles
int launch_tile_pass(double2* psi, const TilePass& pass, const TilePass* pass_dev,
                     const double* mats, const CutTerms& ct, cudaStream_t s);
// A pass of CNOTs only (factored programs, one state): one gather per
// 2^13-amplitude box (k_perm).  False when the targets do not fit one box;
// nothing is launched then.
bool launch_perm(double2* psi, int m, const int* controls, const int* targets, int count,
                 cudaStream_t s);
void launch_fill(double2* psi, uint64_t count, double2 value, cudaStream_t s);
void launch_set_basis(double2* psi, uint64_t stride, uint64_t states, uint64_t off, cudaStream_t s);
void launch_gaussian(double2* psi, uint64_t count_per_state, int num_states, uint64_t rank_offset,
                     uint64_t seed, cudaStream_t s);
void launch_scale(double2* psi, uint64_t count, double factor, cudaStream_t s);
void launch_mul_factors(double2* psi, const double2* f, uint64_t count, cudaStream_t s);

// Observables: per-state tree sums.  `scratch` must hold at least
// reduce_scratch_doubles(m, num_states) doubles.
uint64_t reduce_scratch_doubles(int m, int num_states);
void launch_observable(const double2* psi, int m, int num_states, int kind, int q,
                       uint64_t rank_offset, const CutTerms& ct, double* scratch, double* out_dev,
                       cudaStream_t s);

uint64_t marginal_scratch_doubles(int m, int num_states);
// max|a-b|, sum|a-b|^2, sum|b|^2, max|b| into 32 bytes of device scratch
void launch_state_diff(const double2* a, const double2* b, uint64_t count, void* scratch32,
                       cudaStream_t s);
void launch_marginals(const double2* psi, int m, int num_states, double* scratch, double* out_dev,
                      cudaStream_t s);

void launch_exchange_peer(double2* mine, double2* peer, int m, bool is_lower, const double* u_dev,
                          int control_local, cudaStream_t s);
void launch_swap_peer(double2* mine, double2* peer, int m, int l, int rank_bit, cudaStream_t s);
void launch_swap_local(double2* psi, int m, int num_states, int a, int c, cudaStream_t s);
void launch_pair_update_halves(double2* a, double2* b, uint64_t count, uint64_t first_offset,
                               const double* u_dev, int control_local, cudaStream_t s);

}  // namespace qsb
