// Gate kernels of the B200 state-vector core.
//
//  k_gate1q      one 2x2 gate on a local qubit: a streaming pass, 128-bit
//                double2 loads/stores, ILP pairs per thread
//                (reference: apply_local_one_qubit_gate, statevector.py:162-177)
//  k_controlled  control-mask compaction: thread j -> the j-th pair with control
//                bit 1, so only the control=1 half is read and written
//                (reference: apply_local_controlled_gate, statevector.py:180-195)
//  k_cut_phase   psi_i *= lut[cut(i)] (statevector.py:198-206 + graphs.py:35-42)
//  k_tile        fused pass: a 2^12-amplitude tile in shared memory, gates
//                applied in program order in register "rounds" of 4 qubits;
//                one HBM read + write for a whole run of gates.
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace qsb {

namespace {

__device__ __forceinline__ void load_u(double2 u[4], const double* p) {
    const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = __ldg(q + k);
}

constexpr int kThreads = 256;
constexpr int kIlp = 4;

__global__ void __launch_bounds__(kThreads) k_gate1q(double2* __restrict__ psi, int m, int q,
                                                     uint64_t total_pairs,
                                                     const double* __restrict__ mats,
                                                     uint64_t offset, uint64_t stride) {
    const uint64_t first = uint64_t(blockIdx.x) * (kThreads * kIlp) + threadIdx.x;
    const uint64_t qmask = (uint64_t(1) << q) - 1;
    const uint64_t hmask = (uint64_t(1) << (m - 1)) - 1;
    const uint64_t step = uint64_t(1) << q;
    double2 u[4];
    if (stride == 0) load_u(u, mats + offset);
    uint64_t lo[kIlp];
    double2 a[kIlp], b[kIlp];
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t p = first + uint64_t(i) * kThreads;
        if (p < total_pairs) {
            uint64_t s = p >> (m - 1), j = p & hmask;
            lo[i] = (s << m) | ((j & ~qmask) << 1) | (j & qmask);
            a[i] = psi[lo[i]];
            b[i] = psi[lo[i] + step];
        }
    }
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t p = first + uint64_t(i) * kThreads;
        if (p < total_pairs) {
            if (stride != 0) load_u(u, mats + offset + (p >> (m - 1)) * stride);
            pair_update(a[i], b[i], u);
            psi[lo[i]] = a[i];
            psi[lo[i] + step] = b[i];
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_controlled(double2* __restrict__ psi, int m, int c,
                                                         int t, uint64_t total_pairs,
                                                         const double* __restrict__ mats,
                                                         uint64_t offset, uint64_t stride,
                                                         int diag_one) {
    const uint64_t first = uint64_t(blockIdx.x) * (kThreads * kIlp) + threadIdx.x;
    const int lowb = c < t ? c : t, highb = c < t ? t : c;
    const uint64_t qmask = (uint64_t(1) << (m - 2)) - 1;
    const uint64_t cbit = uint64_t(1) << c, tbit = uint64_t(1) << t;
    double2 u[4];
    if (stride == 0) load_u(u, mats + offset);
    uint64_t lo[kIlp];
    double2 a[kIlp], b[kIlp];
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t p = first + uint64_t(i) * kThreads;
        if (p < total_pairs) {
            uint64_t s = p >> (m - 2), j = p & qmask;
            uint64_t x = insert0(insert0(j, lowb), highb) | cbit;
            lo[i] = (s << m) | x;
            a[i] = psi[lo[i]];
            b[i] = psi[lo[i] | tbit];
        }
    }
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t p = first + uint64_t(i) * kThreads;
        if (p < total_pairs) {
            if (stride != 0) load_u(u, mats + offset + (p >> (m - 2)) * stride);
            if (diag_one) {
                // u = diag(1, z): a' equals a except where a signed zero meets
                // the zero terms, so the full update is computed (bit-exact) but
                // a is written back only when its bits changed -- the
                // control=1, target=1 quarter is the only one that moves.
                const double2 a0 = a[i];
                pair_update(a[i], b[i], u);
                if (__double_as_longlong(a[i].x) != __double_as_longlong(a0.x) ||
                    __double_as_longlong(a[i].y) != __double_as_longlong(a0.y))
                    psi[lo[i]] = a[i];
                psi[lo[i] | tbit] = b[i];
            } else {
                pair_update(a[i], b[i], u);
                psi[lo[i]] = a[i];
                psi[lo[i] | tbit] = b[i];
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_cut_phase(double2* __restrict__ psi, int m,
                                                        uint64_t total, uint64_t rank_offset,
                                                        const __grid_constant__ CutTerms ct,
                                                        const double* __restrict__ mats,
                                                        uint64_t offset, uint64_t stride) {
    const uint64_t first = uint64_t(blockIdx.x) * (kThreads * kIlp) + threadIdx.x;
    const uint64_t lmask = (uint64_t(1) << m) - 1;
    double2 v[kIlp];
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t idx = first + uint64_t(i) * kThreads;
        if (idx < total) v[i] = psi[idx];
    }
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        uint64_t idx = first + uint64_t(i) * kThreads;
        if (idx < total) {
            uint64_t s = idx >> m;
            int k = cut_of(rank_offset | (idx & lmask), ct);
            const double2* lut = reinterpret_cast<const double2*>(mats + offset + s * stride);
            // reference: partition.amplitudes *= np.exp(-1j*angles): psi is the left operand
            psi[idx] = cmul(v[i], __ldg(lut + k));
        }
    }
}

// ---- fused tile pass ------------------------------------------------------------

constexpr int kTileAmps = 1 << kTileLog2;
constexpr int kRegAmps = 1 << kRegLog2;
constexpr int kLoadsPerThread = kTileAmps / kTileThreads;

static_assert(kRegLog2 >= 3 && kRegLog2 <= 5, "register paths cover 3..5 register qubits");

__host__ __device__ constexpr int ctz_c(int x) { return (x & 1) ? 0 : 1 + ctz_c(x >> 1); }

// 2x2 update on register bit J of the 16 amplitudes a thread holds.  C < 0:
// uncontrolled; C >= 0: only pairs whose register bit C is 1.  Both are
// compile-time, so the 8 (or 4) pair updates form one basic block the
// scheduler can interleave (the FP64 dependency chains hide each other).
template <int J, int C>
__device__ __forceinline__ void reg_gate(double2 (&a)[kRegAmps], const double2 u[4]) {
#pragma unroll
    for (int k = 0; k < kRegAmps; ++k) {
        if ((k >> J) & 1) continue;
        if (C >= 0 && !((k >> C) & 1)) continue;
        pair_update(a[k], a[k | (1 << J)], u);
    }
}


// TABLES: the pass has per-state matrix tables.  The tile's rows of those
// tables are staged into shared memory with the tile itself (tm: this gate's
// 4 entries there); without tables every matrix is the shared copy in the
// pass descriptor and no table access is compiled in.
template <bool TABLES>
__device__ __forceinline__ void gate_matrix(double2 u[4], const TileGate& G, const double2* tm) {
    if (!TABLES || G.stride == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = G.u[q];  // parameter space (uniform)
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = tm[q];   // staged row (LDS.128 broadcast)
    }
}

// Fast path: n (1..kRegLog2) uncontrolled gates on register bits 0..n-1 in
// program order; later gates are skipped by uniform branches, so one copy of
// the code serves every run length.
template <bool TABLES>
__device__ __forceinline__ void reg_seq(double2 (&a)[kRegAmps], const TileGate* G, int n,
                                        const double2* tm) {
    double2 u[4];
    gate_matrix<TABLES>(u, G[0], tm);
    reg_gate<0, -1>(a, u);
    if (n > 1) {
        gate_matrix<TABLES>(u, G[1], tm + 4);
        reg_gate<1, -1>(a, u);
        if (n > 2) {
            gate_matrix<TABLES>(u, G[2], tm + 8);
            reg_gate<2, -1>(a, u);
            if (kRegLog2 > 3 && n > 3) {
                gate_matrix<TABLES>(u, G[3], tm + 12);
                reg_gate<(kRegLog2 > 3 ? 3 : 0), -1>(a, u);
                if (kRegLog2 > 4 && n > 4) {
                    gate_matrix<TABLES>(u, G[4], tm + 16);
                    reg_gate<(kRegLog2 > 4 ? 4 : 0), -1>(a, u);
                }
            }
        }
    }
}

// The common case, a full run of kRegLog2 gates: straight-line code with no
// branch between gates, so one gate's tail overlaps the next gate's head.
template <bool TABLES>
__device__ __forceinline__ void reg_seq_full(double2 (&a)[kRegAmps], const TileGate* G,
                                             const double2* tm) {
    double2 u[4];
    gate_matrix<TABLES>(u, G[0], tm);
    reg_gate<0, -1>(a, u);
    gate_matrix<TABLES>(u, G[1], tm + 4);
    reg_gate<1, -1>(a, u);
    gate_matrix<TABLES>(u, G[2], tm + 8);
    reg_gate<2, -1>(a, u);
    if (kRegLog2 > 3) {
        gate_matrix<TABLES>(u, G[3], tm + 12);
        reg_gate<(kRegLog2 > 3 ? 3 : 0), -1>(a, u);
    }
    if (kRegLog2 > 4) {
        gate_matrix<TABLES>(u, G[4], tm + 16);
        reg_gate<(kRegLog2 > 4 ? 4 : 0), -1>(a, u);
    }
}

// Generic gate: target register bit j, pairs filtered by a uniform mask over
// the register index of the pair's lower member (controls in registers).
template <int J>
__device__ __forceinline__ void reg_gate_masked(double2 (&a)[kRegAmps], const double2 u[4],
                                                unsigned mask) {
#pragma unroll
    for (int k = 0; k < kRegAmps; ++k) {
        if ((k >> J) & 1) continue;
        if ((mask >> k) & 1) pair_update(a[k], a[k | (1 << J)], u);
    }
}

__device__ __forceinline__ void reg_gate_generic(double2 (&a)[kRegAmps], const double2 u[4], int j,
                                                 unsigned mask) {
    switch (j) {
        case 0: reg_gate_masked<0>(a, u, mask); break;
        case 1: reg_gate_masked<1>(a, u, mask); break;
        case 2: reg_gate_masked<2>(a, u, mask); break;
        case 3: reg_gate_masked<(kRegLog2 > 3 ? 3 : 0)>(a, u, mask); break;
        default: reg_gate_masked<(kRegLog2 > 4 ? 4 : 0)>(a, u, mask); break;
    }
}

// ---- factored gates (QS_FUSE_FACTORED, factor.cu) ---------------------------
// Shear on register bit J: (a, b) <- (a - t b, b + t a), 4 FMAs per pair.
// With a pre-diagonal the b member is first multiplied by z (diag(1, z) on the
// same qubit).  u: the gate's 4 parameter entries [t, 0], [has_pre, 0], z, -
// (from the pass descriptor, or the state's staged table row in pool mode).
template <int J>
__device__ __forceinline__ void reg_shear(double2 (&a)[kRegAmps], const double2 u[4]) {
    const double t = u[0].x;
    if (u[1].x != 0.0) {  // has_pre
        const double2 z = u[2];
#pragma unroll
        for (int k = 0; k < kRegAmps; ++k)
            if ((k >> J) & 1) a[k] = cmul(a[k], z);
    }
#pragma unroll
    for (int k = 0; k < kRegAmps; ++k) {
        if ((k >> J) & 1) continue;
        const double2 x = a[k], y = a[k | (1 << J)];
        a[k] = make_double2(__fma_rn(-t, y.x, x.x), __fma_rn(-t, y.y, x.y));
        a[k | (1 << J)] = make_double2(__fma_rn(t, x.x, y.x), __fma_rn(t, x.y, y.y));
    }
}

template <int J>
__device__ __forceinline__ void reg_diag1(double2 (&a)[kRegAmps], const double2 z) {
#pragma unroll
    for (int k = 0; k < kRegAmps; ++k)
        if ((k >> J) & 1) a[k] = cmul(a[k], z);
}

template <bool TABLES>
__device__ __forceinline__ void reg_fact_generic(double2 (&a)[kRegAmps], const TileGate& G,
                                                 const double2* tm) {
    double2 u[4];
    gate_matrix<TABLES>(u, G, tm);
    if (G.kind == kKindScalar) {
#pragma unroll
        for (int k = 0; k < kRegAmps; ++k) a[k] = cmul(a[k], u[0]);
        return;
    }
    const int j = G.variant % kRegLog2;
    if (G.kind == kKindDiag1) {
        const double2 z = u[2];
        switch (j) {
            case 0: reg_diag1<0>(a, z); break;
            case 1: reg_diag1<1>(a, z); break;
            case 2: reg_diag1<2>(a, z); break;
            case 3: reg_diag1<(kRegLog2 > 3 ? 3 : 0)>(a, z); break;
            default: reg_diag1<(kRegLog2 > 4 ? 4 : 0)>(a, z); break;
        }
        return;
    }
    switch (j) {
        case 0: reg_shear<0>(a, u); break;
        case 1: reg_shear<1>(a, u); break;
        case 2: reg_shear<2>(a, u); break;
        case 3: reg_shear<(kRegLog2 > 3 ? 3 : 0)>(a, u); break;
        default: reg_shear<(kRegLog2 > 4 ? 4 : 0)>(a, u); break;
    }
}

// A full run of kRegLog2 shears on register bits 0..kRegLog2-1 (straight line).
template <bool TABLES>
__device__ __forceinline__ void reg_shear_seq_full(double2 (&a)[kRegAmps], const TileGate* G,
                                                   const double2* tm) {
    double2 u[4];
    gate_matrix<TABLES>(u, G[0], tm);
    reg_shear<0>(a, u);
    gate_matrix<TABLES>(u, G[1], tm + 4);
    reg_shear<1>(a, u);
    gate_matrix<TABLES>(u, G[2], tm + 8);
    reg_shear<2>(a, u);
    if (kRegLog2 > 3) {
        gate_matrix<TABLES>(u, G[3], tm + 12);
        reg_shear<(kRegLog2 > 3 ? 3 : 0)>(a, u);
    }
    if (kRegLog2 > 4) {
        gate_matrix<TABLES>(u, G[4], tm + 16);
        reg_shear<(kRegLog2 > 4 ? 4 : 0)>(a, u);
    }
}

// Product diagonal D(i) = prod_c T_c[byte c of i] (kKindDiagN).  The factor of
// the thread's k = 0 amplitude comes from the byte tables (its register bits
// are 0); register index k adds R[k] = prod_j z_{q_j}^{k_j}, precomputed by the
// host for the round (the same for every thread and tile).  Two complex
// products per amplitude.
// the tile-element part of a product diagonal: one byte-table entry per 8
// non-register qubits (loaded early by the lean kernels: its latency hides
// behind the smem reads / the round's shears)
__device__ __forceinline__ double2 diag_factor(const double2* T, int ntab, uint64_t il) {
    double2 f = __ldg(T + (il & 255));
    for (int c = 1; c < ntab; ++c) f = cmul(f, __ldg(T + (c << 8) + ((il >> (8 * c)) & 255)));
    return f;
}
__device__ __forceinline__ void reg_diag_apply(double2 (&a)[kRegAmps], double2 f, const double2* R) {
    a[0] = cmul(a[0], f);
#pragma unroll
    for (int k = 1; k < kRegAmps; ++k) a[k] = cmul(a[k], cmul(f, R[k]));
}
__device__ __forceinline__ void reg_diag_n(double2 (&a)[kRegAmps], const double2* T, int ntab,
                                           uint64_t il, const double2* R) {
    double2 f = __ldg(T + (il & 255));
    for (int c = 1; c < ntab; ++c) f = cmul(f, __ldg(T + (c << 8) + ((il >> (8 * c)) & 255)));
    a[0] = cmul(a[0], f);
#pragma unroll
    for (int k = 1; k < kRegAmps; ++k) a[k] = cmul(a[k], cmul(f, R[k]));
}

// variant j (uncontrolled, target register bit j) or kRegLog2 + kRegLog2*c + j
// (controlled by register bit c), kRegLog2 == 4
__device__ __forceinline__ void reg_gate_switch(double2 (&a)[kRegAmps], const double2 u[4],
                                                int variant) {
#if QSB_REG_LOG2 == 4
#define QSB_CG(c, j) case 4 + 4 * (c) + (j): reg_gate<j, c>(a, u); break;
    switch (variant) {
        case 0: reg_gate<0, -1>(a, u); break;
        case 1: reg_gate<1, -1>(a, u); break;
        case 2: reg_gate<2, -1>(a, u); break;
        case 3: reg_gate<3, -1>(a, u); break;
        QSB_CG(0, 1) QSB_CG(0, 2) QSB_CG(0, 3)
        QSB_CG(1, 0) QSB_CG(1, 2) QSB_CG(1, 3)
        QSB_CG(2, 0) QSB_CG(2, 1) QSB_CG(2, 3)
        QSB_CG(3, 0) QSB_CG(3, 1) QSB_CG(3, 2)
        default: break;
    }
#undef QSB_CG
#else
    (void)a, (void)u, (void)variant;  // other builds use reg_gate_generic
#endif
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

#ifdef QSB_PROF
__device__ unsigned long long g_prof[8];
#define PROF_T(v) long long v = clock64()
#define PROF_ADD(i, a, b) if ((threadIdx.x & 31) == 0) atomicAdd(&g_prof[i], (unsigned long long)((b) - (a)))
#else
#define PROF_T(v)
#define PROF_ADD(i, a, b)
#endif
// Persistent CTAs, two per SM (QSB_TILE_MINB), each one warp group of 256
// threads owning a 2^12-amplitude tile buffer and walking its own tiles: while
// one CTA runs FP64 sections the other moves data (cp.async tile loads, the
// shared-memory round trips between register rounds, the write-back to HBM),
// interleaved by the warp schedulers.  This measured faster than one CTA of
// two ping-pong groups handing FP64 turns over named barriers (QSB_TILE_GROUPS=2
// QSB_TILE_MINB=1: sweep 38.1 vs 35.1 ms, QAOA step 95 vs 86 ms).
// Barrier ids: 1,2 group-local; 3,4 "turn of group g" (ping-pong builds only).
#ifndef QSB_TILE_GROUPS
#define QSB_TILE_GROUPS 1
#endif
constexpr int kGroups = QSB_TILE_GROUPS;
#ifdef QSB_NO_PINGPONG
constexpr bool kPingPong = false;
#else
constexpr bool kPingPong = kGroups > 1;
#endif
constexpr int kCtaThreads = kGroups * kTileThreads;
constexpr int kDepTables = 4;  // tile index up to 32 bits (m <= 44)

// PHASE: the pass has cut-phase gates; GENERIC: it has gates outside the
// uncontrolled in-order runs (controlled gates, repeated register bits).
#ifndef QSB_TILE_MINB
#define QSB_TILE_MINB 2
#endif
// The pass descriptor is a __grid_constant__ kernel parameter (~12.5 KB of
// the 32 KB parameter space): its fields are uniform constant-bank loads, which
// frees the registers the shared-memory copy needed (spills 136 -> 24 bytes;
// sweep 33.6 -> 29.6 ms).  QSB_PASS_SMEM restores the shared-memory staging.
#ifndef QSB_PASS_SMEM
#define QSB_PASS_PARAM 1
#endif
template <bool PHASE, bool GENERIC, bool TABLES, bool FACT>
__global__ void __launch_bounds__(kCtaThreads, QSB_TILE_MINB)
#ifdef QSB_PASS_PARAM
    k_tile(double2* __restrict__ psi, const __grid_constant__ TilePass pass_param,
           const double* __restrict__ mats, const __grid_constant__ CutTerms ct) {
    // the pass description lives in the kernel's parameter space: every field
    // read is a uniform constant-bank load and needs no shared memory
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* rowoff = reinterpret_cast<uint64_t*>(smem_raw + kGroups * sizeof(double2) * kTileAmps);
    uint64_t* dep = rowoff + (kTileAmps >> kLowBits);
    const TilePass& P = pass_param;
#else
    k_tile(double2* __restrict__ psi, const TilePass* __restrict__ pass_dev,
           const double* __restrict__ mats, const __grid_constant__ CutTerms ct) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* rowoff = reinterpret_cast<uint64_t*>(smem_raw + kGroups * sizeof(double2) * kTileAmps);
    TilePass* pass_s = reinterpret_cast<TilePass*>(smem_raw + kGroups * sizeof(double2) * kTileAmps +
                                                   sizeof(uint64_t) * (kTileAmps >> kLowBits));
    // deposit tables: tile index byte c -> its bits spread over the non-tile qubits
    uint64_t* dep = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(pass_s) +
                                                sizeof(TilePass));
    {
        // the pass description (rounds, gates, shared matrices) is read once per
        // persistent CTA and then served from shared memory (uniform broadcasts)
        const uint4* src = reinterpret_cast<const uint4*>(pass_dev);
        uint4* dst = reinterpret_cast<uint4*>(pass_s);
        for (int i = threadIdx.x; i < int(sizeof(TilePass) / 16); i += kCtaThreads) dst[i] = src[i];
        __syncthreads();
    }
    const TilePass& P = *pass_s;
#endif
    // per-round thread -> tile element deposits (dlo|slo<<16, dhi|shi<<16) in
    // shared memory: indexed by thread id they would be divergent (serialised)
    // constant-bank reads
    uint32_t* rlo = reinterpret_cast<uint32_t*>(dep + 256 * kDepTables);
    uint32_t* rhi = rlo + kMaxRounds * (1 << kLaneLoBits);
    // two buffers of staged per-state matrix rows (tile it uses buffer it & 1)
    double2* tmat = reinterpret_cast<double2*>(rhi + kMaxRounds * (1 << kLaneHiBits));
    for (int i = threadIdx.x; i < P.num_rounds * (1 << kLaneLoBits); i += kCtaThreads) {
        const Round& R = P.rounds[i >> kLaneLoBits];
        const int v = i & ((1 << kLaneLoBits) - 1);
        rlo[i] = uint32_t(R.dlo[v]) | (uint32_t(R.slo[v]) << 16);
    }
    for (int i = threadIdx.x; i < P.num_rounds * (1 << kLaneHiBits); i += kCtaThreads) {
        const Round& R = P.rounds[i >> kLaneHiBits];
        const int v = i & ((1 << kLaneHiBits) - 1);
        rhi[i] = uint32_t(R.dhi[v]) | (uint32_t(R.shi[v]) << 16);
    }
    const int low_run = P.low_run;
    const int nrows = kTileAmps >> low_run;
    const uint64_t lowmask = (uint64_t(1) << low_run) - 1;
    // row offsets: deposit of the row index into the tile bits above the low run
    for (int r = threadIdx.x; r < nrows; r += kCtaThreads) {
        uint64_t off = 0;
        for (int k = 0; k < kTileLog2 - low_run; ++k)
            if ((r >> k) & 1) off |= uint64_t(1) << P.tile_bits[low_run + k];
        rowoff[r] = off;
    }
    {
        // non-tile qubit positions, ascending: tile index bit b lands on nontile[b]
        int nontile[64];
        int cnt = 0;
        for (int b = 0, k = 0; b < P.m; ++b) {
            if (k < kTileLog2 && P.tile_bits[k] == b) {
                ++k;
                continue;
            }
            nontile[cnt++] = b;
        }
        for (int i = threadIdx.x; i < kDepTables * 256; i += kCtaThreads) {
            const int c = i >> 8, v = i & 255;
            uint64_t out = 0;
            for (int b = 0; b < 8; ++b)
                if (((v >> b) & 1) && 8 * c + b < cnt) out |= uint64_t(1) << nontile[8 * c + b];
            dep[i] = out;
        }
    }
    __syncthreads();

    const int group = threadIdx.x / kTileThreads;  // warp-uniform
    const int tid = threadIdx.x % kTileThreads;
    const int gbar = 1 + group;
    const int my_turn = 3 + group, other_turn = 4 - group;
    double2* tile = reinterpret_cast<double2*>(smem_raw) + group * kTileAmps;
    const int m = P.m;
    const int tps_log2 = m - kTileLog2;
    const uint64_t stride_tiles = uint64_t(kGroups) * gridDim.x;
    const uint64_t iters = (P.num_tiles + stride_tiles - 1) / stride_tiles;
    if (kPingPong && group == 1) named_arrive(3, kCtaThreads);  // group 0 computes first

    auto tile_base = [&](uint64_t t) {
        const uint64_t x = t & (P.tiles_per_state - 1);
        uint64_t out = 0;
#pragma unroll
        for (int c = 0; c < kDepTables; ++c) out |= dep[(c << 8) | ((x >> (8 * c)) & 255)];
        return out;
    };
    // Tile element e -> HBM offset is linear over disjoint bit sets (a
    // deposit): off(e | f) = off(e) + off(f), and so is the smem swizzle.  The
    // load/store element e = tid | i*kTileThreads therefore splits into a
    // per-thread part computed once and a uniform part per i.
    auto goff = [&](int e) { return rowoff[e >> low_run] + (uint64_t(e) & lowmask); };
    const uint64_t goff_tid = goff(tid);
    const int swz_tid = swz(tid);
    const int ngates = P.rounds[P.num_rounds - 1].first_gate + P.rounds[P.num_rounds - 1].num_gates;
    auto prefetch = [&](uint64_t t, int buf) {
#if !defined(QSB_NO_GMEM) && !defined(QSB_NO_LOADS)  // diagnostics builds
        if (t < P.num_tiles) {
            const uint64_t st = t >> tps_log2;
            const double2* g = psi + ((st << m) | tile_base(t)) + goff_tid;
#pragma unroll
            for (int i = 0; i < kLoadsPerThread; ++i)
                cp_async16(tile + (swz_tid ^ swz(i * kTileThreads)), g + goff(i * kTileThreads));
            if (TABLES) {
                // this state's row of every per-state matrix table: 4 x 16 B per gate
                double2* tm = tmat + buf * (4 * kMaxPassGates);
                for (int c = tid; c < 4 * ngates; c += kTileThreads) {
                    const TileGate& G = P.gates[c >> 2];
                    if (G.stride != 0 && G.kind != QS_KIND_CUTPHASE)
                        cp_async16(tm + c, mats + G.offset + st * G.stride + 2 * (c & 3));
                }
            }
        }
#endif
        cp_async_commit();
    };
    const bool direct = P.direct_store != 0;
    prefetch(uint64_t(blockIdx.x) * kGroups + group, 0);

    for (uint64_t it = 0; it < iters; ++it) {
        const uint64_t tile_id = it * stride_tiles + uint64_t(blockIdx.x) * kGroups + group;
        const uint64_t next_id = tile_id + stride_tiles;
        const bool valid = tile_id < P.num_tiles;
        const uint64_t s = tile_id >> tps_log2;
        const uint64_t base_local = tile_base(tile_id);
        double2* gbase = psi + ((s << m) | base_local);
        const double2* tm_cur = tmat + int(it & 1) * (4 * kMaxPassGates);
        PROF_T(t0);
        cp_async_wait_all();
        named_sync(gbar, kTileThreads);
        PROF_T(t1);
        PROF_ADD(0, t0, t1);

        for (int r = 0; r < P.num_rounds; ++r) {
            PROF_T(r0);
            const Round& R = P.rounds[r];
            const bool last = r == P.num_rounds - 1;
            const uint32_t lo = rlo[(r << kLaneLoBits) | (tid & ((1 << kLaneLoBits) - 1))];
            const uint32_t hi = rhi[(r << kLaneHiBits) | (tid >> kLaneLoBits)];
            const int eb = int((lo | hi) & 0xffff);
            const int sb = int((lo ^ hi) >> 16);
            // register k sits at tile element eb | dk[k]; dk and its swizzle sk
            // are linear in k's bits, so 4 basis values give all 16 positions
            int skb[kRegLog2];
#pragma unroll
            for (int j = 0; j < kRegLog2; ++j) skb[j] = R.sk[1 << j];
            auto sk_of = [&](int k) {
                int v = 0;
#pragma unroll
                for (int j = 0; j < kRegLog2; ++j)
                    if ((k >> j) & 1) v ^= skb[j];
                return v;
            };
            double2 a[kRegAmps];
#ifdef QSB_NO_SMEM_ROUND
#pragma unroll
            for (int k = 0; k < kRegAmps; ++k) a[k] = make_double2(sb * 1e-3 + k, eb * 1e-3);
#else
#pragma unroll
            for (int k = 0; k < kRegAmps; ++k) a[k] = tile[sb ^ sk_of(k)];
#endif
            if (last && direct) {
                // the tile now lives in registers: the buffer is free for the next tile
                named_sync(gbar, kTileThreads);
                prefetch(next_id, int((it + 1) & 1));
            }

            PROF_T(r1);
            if (kPingPong) named_sync(my_turn, kCtaThreads);
            PROF_T(r2);
            if (valid) {
                const int g_end = R.first_gate + R.num_gates;
                for (int g = R.first_gate; g < g_end; ++g) {
                    const TileGate& G = P.gates[g];
                    if (PHASE && G.kind == QS_KIND_CUTPHASE) {
                        const double2* lut =
                            reinterpret_cast<const double2*>(mats + G.offset + s * G.stride);
                        // cut of the k=0 amplitude in full, then walk the 16 register
                        // indices in Gray-code order: flipping qubit r changes the cut
                        // by deg(r) - 2 * (edges of r currently cut)
                        uint64_t i = P.rank_offset | (base_local + rowoff[eb >> low_run] +
                                                      (uint64_t(eb) & lowmask));
                        const int cut0 = cut_of(i, ct);
                        // register bit j <-> qubit rq[j]: flipping a set F of them
                        // changes the cut by sum_{j in F} d_j plus, per edge inside F,
                        // (4 * cut_e - 2) (both ends flipped: the edge's status stays)
                        int rq[kRegLog2], d[kRegLog2], bq[kRegLog2];
                        uint64_t nbq[kRegLog2];
#pragma unroll
                        for (int j = 0; j < kRegLog2; ++j) {
                            rq[j] = P.tile_bits[__ffs(R.dk[1 << j]) - 1];
                            nbq[j] = P.nbr[rq[j]];
                            bq[j] = int((i >> rq[j]) & 1);
                            d[j] = __popcll(nbq[j]) -
                                   2 * __popcll((i ^ (uint64_t(0) - uint64_t(bq[j]))) & nbq[j]);
                        }
                        int cuts[kRegAmps];
                        cuts[0] = cut0;
#pragma unroll
                        for (int k = 1; k < kRegAmps; ++k) {
                            const int h = 31 - __clz(k);  // highest bit of k (compile time)
                            int c = cuts[k ^ (1 << h)] + d[h];
#pragma unroll
                            for (int j = 0; j < h; ++j)
                                if ((k >> j) & 1)
                                    c += ((nbq[h] >> rq[j]) & 1) ? 4 * (bq[h] ^ bq[j]) - 2 : 0;
                            cuts[k] = c;
                        }
#pragma unroll
                        for (int k = 0; k < kRegAmps; ++k) a[k] = cmul(a[k], __ldg(lut + cuts[k]));
                        continue;
                    }
                    if (FACT && G.kind >= kKindShear) {
                        if (G.kind == kKindDiagN) {
                            const double2* T = reinterpret_cast<const double2*>(mats + G.offset);
                            reg_diag_n(a, T, G.cval,
                                       base_local + rowoff[eb >> low_run] + (uint64_t(eb) & lowmask),
                                       P.diag_r[G.pad[0]]);
                        } else if (G.seq == kRegLog2) {
                            reg_shear_seq_full<TABLES>(a, &G, tm_cur + 4 * g);
                            g += kRegLog2 - 1;
                        } else {
                            reg_fact_generic<TABLES>(a, G, tm_cur + 4 * g);
                        }
                        continue;
                    }
                    if (G.seq == kRegLog2) {
                        reg_seq_full<TABLES>(a, &G, tm_cur + 4 * g);
                        g += kRegLog2 - 1;
                        continue;
                    }
                    if (G.seq > 0) {
                        reg_seq<TABLES>(a, &G, G.seq, tm_cur + 4 * g);
                        g += G.seq - 1;
                        continue;
                    }
                    if (GENERIC) {
                        if (G.ctype == 2 && !((eb >> G.cval) & 1)) continue;
                        if (G.ctype == 3 && !((base_local >> G.cval) & 1)) continue;
                        double2 u[4];
                        gate_matrix<TABLES>(u, G, tm_cur + 4 * g);
                        if (kRegLog2 == 4) {
                            // (control, target) register bits as compile-time cases:
                            // a register-controlled gate runs exactly its 4 pairs
                            reg_gate_switch(a, u, G.variant);
                        } else {
                            // register control c: only pairs whose register index has bit c set
                            unsigned mask = (kRegAmps >= 32) ? 0xffffffffu : ((1u << kRegAmps) - 1);
                            if (G.ctype == 1) {
                                mask = 0;
#pragma unroll
                                for (int k = 0; k < kRegAmps; ++k)
                                    if ((k >> G.cval) & 1) mask |= 1u << k;
                            }
                            reg_gate_generic(a, u, G.variant % kRegLog2, mask);
                        }
                    }
                }
            }
            PROF_T(r3);
            if (kPingPong) named_arrive(other_turn, kCtaThreads);
            if (last && direct) {
                // last round straight from registers to HBM: lanes 0-7 cover tile
                // positions 0,1,2 (128-byte rows), so every warp store is 4 full rows
#if !defined(QSB_NO_GMEM) && !defined(QSB_NO_STORES)
                if (valid) {
                    uint64_t okb[kRegLog2];
#pragma unroll
                    for (int j = 0; j < kRegLog2; ++j) okb[j] = goff(R.dk[1 << j]);
                    double2* gb = gbase + goff(eb);
#pragma unroll
                    for (int k = 0; k < kRegAmps; ++k) {
                        uint64_t o = 0;
#pragma unroll
                        for (int j = 0; j < kRegLog2; ++j)
                            if ((k >> j) & 1) o += okb[j];
                        gb[o] = a[k];
                    }
                }
#endif
                PROF_T(r4);
                PROF_ADD(1, r0, r1);
                PROF_ADD(2, r1, r2);
                PROF_ADD(3, r2, r3);
                PROF_ADD(5, r3, r4);
                break;
            }
#ifdef QSB_NO_SMEM_ROUND
            {
                double2 acc = a[0];
#pragma unroll
                for (int k = 1; k < kRegAmps; ++k) acc = cadd(acc, a[k]);
                if (acc.x == 12345.678) tile[sb] = acc;  // keep the arithmetic alive
            }
#else
            {
                // recompute the 16 positions instead of keeping the load
                // addresses live across the FP64 section (they would spill)
                int sbs = sb;
                asm volatile("" : "+r"(sbs));
#pragma unroll
                for (int k = 0; k < kRegAmps; ++k) tile[sbs ^ sk_of(k)] = a[k];
            }
#endif
            named_sync(gbar, kTileThreads);
            PROF_T(r4);
            PROF_ADD(1, r0, r1);
            PROF_ADD(2, r1, r2);
            PROF_ADD(3, r2, r3);
            PROF_ADD(4, r3, r4);
        }
        if (!direct) {
            PROF_T(s0);
#if !defined(QSB_NO_GMEM) && !defined(QSB_NO_STORES)
            if (valid) {
                double2* gb = gbase + goff_tid;
#pragma unroll
                for (int i = 0; i < kLoadsPerThread; ++i)
                    gb[goff(i * kTileThreads)] = tile[swz_tid ^ swz(i * kTileThreads)];
            }
#endif
            named_sync(gbar, kTileThreads);
            prefetch(next_id, int((it + 1) & 1));
            PROF_T(s1);
            PROF_ADD(5, s0, s1);
        }
    }
    if (kPingPong && group == 0) named_sync(3, kCtaThreads);  // consume group 1's last hand-over
}

// ---- lean fused pass for factored programs -------------------------------------
// A pass whose rounds are runs of shears (QS_FUSE_FACTORED) on register bits
// 0..n-1 in order -- optionally two such runs around one cut phase -- with the
// product diagonals at its ends.  The round's parameters are read at
// compile-time offsets and each round is one straight-line template instance,
// so no per-gate dispatch is left in the loop (k_tile's generic gate loop costs
// more integer work and registers than the 2 FP64 instructions per amplitude a
// shear needs).  TABLES: per-state t (pool mode: the QAOA mixer RX(2 beta_s));
// PHASE: rounds may hold a cut phase (per-state LUT rows, the per-state shear
// scalars folded in by factor.cu).
struct FactRound {
    double t[2][kRegLog2];        // run A / run B; 0 pads bits without a shear (exact identity)
    double2 pre[2][kRegLog2];     // (1, 0) without a pre-diagonal
    uint64_t toff[2][kRegLog2];   // TABLES: t = mats[toff + state * tstride]
    uint32_t tstride[2][kRegLog2];
    int32_t n[2], pre_any, mid;   // mid: a cut phase between run A and run B
    uint64_t lut_off, lut_stride;
};
struct alignas(16) FactPass {
    int32_t m, num_rounds, low_run, direct_store;
    int32_t tile_bits[kTileLog2];
    int32_t ntab, has_din, has_dout;
    int32_t const_in;            // the pass input is the constant `cin` (no tile loads): a
                                 // program that starts from a uniform state (TABLES kernels)
    uint64_t tiles_per_state, num_tiles, rank_offset;
    uint64_t din_off, dout_off;  // DiagN tables in mats (doubles)
    double2 cin;
    double2 din_r[1 << kRegLog2], dout_r[1 << kRegLog2];  // register parts (TilePass::diag_r)
    uint64_t nbr[64];            // cut-phase graph (TilePass::nbr)
    Round rounds[kMaxRounds];
    FactRound fr[kMaxRounds];
};

template <int J, bool PRE, bool TABLES>
__device__ __forceinline__ void fact_shear(double2 (&a)[kRegAmps], const FactRound& F, int grp,
                                           const double* __restrict__ mats, uint64_t st) {
#ifdef QSB_EXP_SHARED_T  // diagnostics build: per-state t replaced by the shared one
    const double t = F.t[grp][J];
#else
    const double t = TABLES ? __ldg(mats + F.toff[grp][J] + st * F.tstride[grp][J]) : F.t[grp][J];
#endif
    if (PRE) {
        // pool passes read the state's pre-diagonal from its row (per-state
        // diagonals of noise trajectories; (1, 0) where there is none)
        const double2 z =
            TABLES ? __ldg(reinterpret_cast<const double2*>(mats + F.toff[grp][J] +
                                                            st * F.tstride[grp][J] + 4))
                   : F.pre[grp][J];
#pragma unroll
        for (int k = 0; k < kRegAmps; ++k)
            if ((k >> J) & 1) a[k] = cmul(a[k], z);
    }
#pragma unroll
    for (int k = 0; k < kRegAmps; ++k) {
        if ((k >> J) & 1) continue;
        const double2 x = a[k], y = a[k | (1 << J)];
        a[k] = make_double2(__fma_rn(-t, y.x, x.x), __fma_rn(-t, y.y, x.y));
        a[k | (1 << J)] = make_double2(__fma_rn(t, x.x, y.x), __fma_rn(t, x.y, y.y));
    }
}

template <bool PRE, bool TABLES>
__device__ __forceinline__ void fact_run(double2 (&a)[kRegAmps], const FactRound& F, int grp,
                                         const double* __restrict__ mats, uint64_t st) {
    fact_shear<0, PRE, TABLES>(a, F, grp, mats, st);
    fact_shear<1, PRE, TABLES>(a, F, grp, mats, st);
    fact_shear<2, PRE, TABLES>(a, F, grp, mats, st);
    if (kRegLog2 > 3) fact_shear<(kRegLog2 > 3 ? 3 : 0), PRE, TABLES>(a, F, grp, mats, st);
    if (kRegLog2 > 4) fact_shear<(kRegLog2 > 4 ? 4 : 0), PRE, TABLES>(a, F, grp, mats, st);
}

// psi_i *= lut[cut(i)] on the 16 register amplitudes: the cut of the k = 0
// amplitude in full, then a Gray walk over the register qubits (flipping
// qubit r changes the cut by deg(r) - 2 * (edges of r currently cut), and an
// edge inside the flipped set keeps its status) -- the same walk as k_tile's.
__device__ __forceinline__ void fact_cut_phase(double2 (&a)[kRegAmps], const FactPass& P,
                                               const Round& R, const CutTerms& ct,
                                               const double2* lut, uint64_t il) {
#ifdef QSB_EXP_NOCUT  // diagnostics build: no cut phase arithmetic
    return;
#endif
    const uint64_t i = P.rank_offset | il;
    const int cut0 = cut_of(i, ct);
    int rq[kRegLog2], d[kRegLog2], bq[kRegLog2];
    uint64_t nbq[kRegLog2];
#pragma unroll
    for (int j = 0; j < kRegLog2; ++j) {
        rq[j] = P.tile_bits[__ffs(R.dk[1 << j]) - 1];
        nbq[j] = P.nbr[rq[j]];
        bq[j] = int((i >> rq[j]) & 1);
        d[j] = __popcll(nbq[j]) - 2 * __popcll((i ^ (uint64_t(0) - uint64_t(bq[j]))) & nbq[j]);
    }
    int cuts[kRegAmps];
    cuts[0] = cut0;
#pragma unroll
    for (int k = 1; k < kRegAmps; ++k) {
        const int h = 31 - __clz(k);
        int c = cuts[k ^ (1 << h)] + d[h];
#pragma unroll
        for (int j = 0; j < h; ++j)
            if ((k >> j) & 1) c += ((nbq[h] >> rq[j]) & 1) ? 4 * (bq[h] ^ bq[j]) - 2 : 0;
        cuts[k] = c;
    }
#pragma unroll
    for (int k = 0; k < kRegAmps; ++k) a[k] = cmul(a[k], __ldg(lut + cuts[k]));
}

// One register round of a lean pass, straight-line for its flags: product
// diagonal before (DIN) / after (DOUT), pre-diagonals (PRE), a cut phase and a
// second shear run (MID), and the store of the 16 amplitudes to HBM (GSTORE)
// or back to the shared tile.  Every run applies kRegLog2 shears (t = 0 is an
// exact identity), so no amplitude register is live across a data-dependent
// branch (each join would cost 64 register moves).
template <bool TABLES, bool DIN, bool PRE, bool DOUT, bool GSTORE, bool MID>
__device__ __forceinline__ void fact_body(double2 (&a)[kRegAmps], const FactPass& P,
                                          const Round& R, const FactRound& F, const CutTerms& ct,
                                          const double* __restrict__ mats, uint64_t st,
                                          uint64_t il, double2* tile, int sb,
                                          const int (&skb)[kRegLog2], double2* gb,
                                          const uint64_t (&okb)[kRegLog2], int acq = 0) {
    if (DIN) reg_diag_apply(a, diag_factor(reinterpret_cast<const double2*>(mats + P.din_off), P.ntab, il),
                            P.din_r);
    fact_run<PRE, TABLES>(a, F, 0, mats, st);
    if (MID) {
        fact_cut_phase(a, P, R, ct,
                       reinterpret_cast<const double2*>(mats + F.lut_off + st * F.lut_stride), il);
        fact_run<PRE, TABLES>(a, F, 1, mats, st);
    }
    // (loading the product-diagonal factors early -- before the tile reads or
    // the shears -- measured slower: pass 1 6.35 -> 6.9 ms)
    if (DOUT)
        reg_diag_apply(a, diag_factor(reinterpret_cast<const double2*>(mats + P.dout_off), P.ntab, il),
                       P.dout_r);
    if (GSTORE) {
#pragma unroll
        for (int k = 0; k < kRegAmps; ++k) {
            uint64_t o = 0;
#pragma unroll
            for (int j = 0; j < kRegLog2; ++j)
                if ((k >> j) & 1) o += okb[j];
#if defined(QSB_NO_GMEM) || defined(QSB_NO_STORES)  // diagnostics: the store goes to the tile
            tile[(uint64_t(sb) + o) & (kTileAmps - 1)] = a[k];
#else
            gb[o] = a[k];
#endif
        }
    } else {
        // k_fact_pair: the two groups share one reslice buffer; take it now
        // (after the round's arithmetic) from the other group
        if (acq) named_sync(acq, 2 * kTileThreads);
        int sbs = sb;
        asm volatile("" : "+r"(sbs));
#pragma unroll
        for (int k = 0; k < kRegAmps; ++k) {
            int v = 0;
#pragma unroll
            for (int j = 0; j < kRegLog2; ++j)
                if ((k >> j) & 1) v ^= skb[j];
            tile[sbs ^ v] = a[k];
        }
    }
}

#define QSB_FB(TB, MI, sel, ...)                                                  \
    switch (sel) {                                                                \
        case 0: fact_body<TB, 0, 0, 0, 0, MI>(__VA_ARGS__); break;                \
        case 1: fact_body<TB, 1, 0, 0, 0, MI>(__VA_ARGS__); break;                \
        case 2: fact_body<TB, 0, 1, 0, 0, MI>(__VA_ARGS__); break;                \
        case 3: fact_body<TB, 1, 1, 0, 0, MI>(__VA_ARGS__); break;                \
        case 4: fact_body<TB, 0, 0, 1, 0, MI>(__VA_ARGS__); break;                \
        case 5: fact_body<TB, 1, 0, 1, 0, MI>(__VA_ARGS__); break;                \
        case 6: fact_body<TB, 0, 1, 1, 0, MI>(__VA_ARGS__); break;                \
        case 7: fact_body<TB, 1, 1, 1, 0, MI>(__VA_ARGS__); break;                \
        case 8: fact_body<TB, 0, 0, 0, 1, MI>(__VA_ARGS__); break;                \
        case 9: fact_body<TB, 1, 0, 0, 1, MI>(__VA_ARGS__); break;                \
        case 10: fact_body<TB, 0, 1, 0, 1, MI>(__VA_ARGS__); break;               \
        case 11: fact_body<TB, 1, 1, 0, 1, MI>(__VA_ARGS__); break;               \
        case 12: fact_body<TB, 0, 0, 1, 1, MI>(__VA_ARGS__); break;               \
        case 13: fact_body<TB, 1, 0, 1, 1, MI>(__VA_ARGS__); break;               \
        case 14: fact_body<TB, 0, 1, 1, 1, MI>(__VA_ARGS__); break;               \
        default: fact_body<TB, 1, 1, 1, 1, MI>(__VA_ARGS__); break;               \
    }

// QSB_FB with the pre-diagonal bodies compiled only when PREOK and the
// product-diagonal bodies only when DIAGOK (passes without them -- every
// config-2 sweep pass has no pre-diagonal, the middle one no product diagonal
// -- get a smaller kernel whose registers are not shared with bodies they
// never run: config-2 pass 1 6.7 -> 6.1 ms without the 20-byte spills)
#define QSB_FBP(TB, MI, PREOK, DIAGOK, sel, ...)                                            \
    switch (sel) {                                                                            \
        case 0: fact_body<TB, 0, 0, 0, 0, MI>(__VA_ARGS__); break;                          \
        case 1: if (DIAGOK) fact_body<TB, DIAGOK, 0, 0, 0, MI>(__VA_ARGS__); break;         \
        case 2: if (PREOK) fact_body<TB, 0, PREOK, 0, 0, MI>(__VA_ARGS__); break;           \
        case 3: if (PREOK && DIAGOK) fact_body<TB, DIAGOK, PREOK, 0, 0, MI>(__VA_ARGS__); break;\
        case 4: if (DIAGOK) fact_body<TB, 0, 0, DIAGOK, 0, MI>(__VA_ARGS__); break;         \
        case 5: if (DIAGOK) fact_body<TB, DIAGOK, 0, DIAGOK, 0, MI>(__VA_ARGS__); break;    \
        case 6: if (PREOK && DIAGOK) fact_body<TB, 0, PREOK, DIAGOK, 0, MI>(__VA_ARGS__); break;\
        case 7: if (PREOK && DIAGOK) fact_body<TB, DIAGOK, PREOK, DIAGOK, 0, MI>(__VA_ARGS__); break;\
        case 8: fact_body<TB, 0, 0, 0, 1, MI>(__VA_ARGS__); break;                          \
        case 9: if (DIAGOK) fact_body<TB, DIAGOK, 0, 0, 1, MI>(__VA_ARGS__); break;         \
        case 10: if (PREOK) fact_body<TB, 0, PREOK, 0, 1, MI>(__VA_ARGS__); break;          \
        case 11: if (PREOK && DIAGOK) fact_body<TB, DIAGOK, PREOK, 0, 1, MI>(__VA_ARGS__); break;\
        case 12: if (DIAGOK) fact_body<TB, 0, 0, DIAGOK, 1, MI>(__VA_ARGS__); break;        \
        case 13: if (DIAGOK) fact_body<TB, DIAGOK, 0, DIAGOK, 1, MI>(__VA_ARGS__); break;   \
        case 14: if (PREOK && DIAGOK) fact_body<TB, 0, PREOK, DIAGOK, 1, MI>(__VA_ARGS__); break;\
        default: if (PREOK && DIAGOK) fact_body<TB, DIAGOK, PREOK, DIAGOK, 1, MI>(__VA_ARGS__); break;\
    }

template <bool TABLES, bool PHASE>
__global__ void __launch_bounds__(kTileThreads, QSB_TILE_MINB)
    k_fact(double2* __restrict__ psi, const __grid_constant__ FactPass P,
           const double* __restrict__ mats, const __grid_constant__ CutTerms ct) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* tile = reinterpret_cast<double2*>(smem_raw);
    uint64_t* rowoff = reinterpret_cast<uint64_t*>(smem_raw + sizeof(double2) * kTileAmps);
    uint64_t* dep = rowoff + (kTileAmps >> kLowBits);
    uint32_t* rlo = reinterpret_cast<uint32_t*>(dep + 256 * kDepTables);
    uint32_t* rhi = rlo + kMaxRounds * (1 << kLaneLoBits);
    const int tid = threadIdx.x;
    for (int i = tid; i < P.num_rounds * (1 << kLaneLoBits); i += kTileThreads) {
        const Round& R = P.rounds[i >> kLaneLoBits];
        const int v = i & ((1 << kLaneLoBits) - 1);
        rlo[i] = uint32_t(R.dlo[v]) | (uint32_t(R.slo[v]) << 16);
    }
    for (int i = tid; i < P.num_rounds * (1 << kLaneHiBits); i += kTileThreads) {
        const Round& R = P.rounds[i >> kLaneHiBits];
        const int v = i & ((1 << kLaneHiBits) - 1);
        rhi[i] = uint32_t(R.dhi[v]) | (uint32_t(R.shi[v]) << 16);
    }
    const int low_run = P.low_run;
    const int nrows = kTileAmps >> low_run;
    const uint64_t lowmask = (uint64_t(1) << low_run) - 1;
    for (int r = tid; r < nrows; r += kTileThreads) {
        uint64_t off = 0;
        for (int k = 0; k < kTileLog2 - low_run; ++k)
            if ((r >> k) & 1) off |= uint64_t(1) << P.tile_bits[low_run + k];
        rowoff[r] = off;
    }
    for (int i = tid; i < kDepTables * 256; i += kTileThreads) {
        // tile index bit b lands on the b-th non-tile qubit (ascending)
        const int c = i >> 8, v = i & 255;
        uint64_t out = 0;
        for (int b = 0; b < 8; ++b) {
            if (!((v >> b) & 1)) continue;
            int want = 8 * c + b, cnt = 0;
            for (int q = 0, k = 0; q < P.m; ++q) {
                if (k < kTileLog2 && P.tile_bits[k] == q) {
                    ++k;
                    continue;
                }
                if (cnt++ == want) {
                    out |= uint64_t(1) << q;
                    break;
                }
            }
        }
        dep[i] = out;
    }
    __syncthreads();

    const int m = P.m;
    const int tps_log2 = m - kTileLog2;
    const uint64_t stride_tiles = gridDim.x;
    auto tile_base = [&](uint64_t t) {
        const uint64_t x = t & (P.tiles_per_state - 1);
        uint64_t out = 0;
#pragma unroll
        for (int c = 0; c < kDepTables; ++c) out |= dep[(c << 8) | ((x >> (8 * c)) & 255)];
        return out;
    };
    auto goff = [&](int e) { return rowoff[e >> low_run] + (uint64_t(e) & lowmask); };
    const uint64_t goff_tid = goff(tid);
    const int swz_tid = swz(tid);
    auto prefetch = [&](uint64_t t) {
#if !defined(QSB_NO_GMEM) && !defined(QSB_NO_LOADS)
        if (t < P.num_tiles) {
#else
        if (false) {
#endif
            const double2* g = psi + (((t >> tps_log2) << m) | tile_base(t)) + goff_tid;
#pragma unroll
            for (int i = 0; i < kLoadsPerThread; ++i)
                cp_async16(tile + (swz_tid ^ swz(i * kTileThreads)), g + goff(i * kTileThreads));
        }
        cp_async_commit();
    };
    const bool direct = P.direct_store != 0;
    prefetch(blockIdx.x);

    for (uint64_t tile_id = blockIdx.x; tile_id < P.num_tiles; tile_id += stride_tiles) {
        const uint64_t st = tile_id >> tps_log2;
        const uint64_t base_local = tile_base(tile_id);
        double2* gbase = psi + ((st << m) | base_local);
        cp_async_wait_all();
        named_sync(1, kTileThreads);
        for (int r = 0; r < P.num_rounds; ++r) {
            const Round& R = P.rounds[r];
            const bool last = r == P.num_rounds - 1;
            const uint32_t lo = rlo[(r << kLaneLoBits) | (tid & ((1 << kLaneLoBits) - 1))];
            const uint32_t hi = rhi[(r << kLaneHiBits) | (tid >> kLaneLoBits)];
            const int eb = int((lo | hi) & 0xffff);
            const int sb = int((lo ^ hi) >> 16);
            int skb[kRegLog2];
#pragma unroll
            for (int j = 0; j < kRegLog2; ++j) skb[j] = R.sk[1 << j];
            auto sk_of = [&](int k) {
                int v = 0;
#pragma unroll
                for (int j = 0; j < kRegLog2; ++j)
                    if ((k >> j) & 1) v ^= skb[j];
                return v;
            };
            double2 a[kRegAmps];
#pragma unroll
            for (int k = 0; k < kRegAmps; ++k) a[k] = tile[sb ^ sk_of(k)];
            if (last && direct) {
                named_sync(1, kTileThreads);
                prefetch(tile_id + stride_tiles);
            }
            const FactRound& F = P.fr[r];
            const bool gstore = last && direct;
            const int sel = int(r == 0 && P.has_din) | (F.pre_any ? 2 : 0) |
                            int(last && P.has_dout) << 2 | int(gstore) << 3;
            const uint64_t il = base_local + rowoff[eb >> low_run] + (uint64_t(eb) & lowmask);
            uint64_t okb[kRegLog2];
#pragma unroll
            for (int j = 0; j < kRegLog2; ++j) okb[j] = gstore ? goff(R.dk[1 << j]) : 0;
            double2* gb = gbase + (gstore ? goff(eb) : 0);
            if (PHASE && F.mid) {
                QSB_FB(TABLES, (PHASE && true), sel, a, P, R, F, ct, mats, st, il, tile, sb, skb, gb, okb)
            } else {
                QSB_FB(TABLES, false, sel, a, P, R, F, ct, mats, st, il, tile, sb, skb, gb, okb)
            }
            if (gstore) break;
            named_sync(1, kTileThreads);
        }
        if (!direct) {
            double2* gb = gbase + goff_tid;
#pragma unroll
            for (int i = 0; i < kLoadsPerThread; ++i)
                gb[goff(i * kTileThreads)] = tile[swz_tid ^ swz(i * kTileThreads)];
            named_sync(1, kTileThreads);
            prefetch(tile_id + stride_tiles);
        }
    }
}

// The lean kernel applies when every round of the pass is a run of shears on
// register bits 0,1,.. in order, or two such runs around one cut phase, with
// product diagonals only first in round 0 / last in the last round.
bool fact_pass_from(const TilePass& T, FactPass* F, bool* tables, bool* phase) {
    memset(F, 0, sizeof(*F));
    *tables = *phase = false;
    F->m = T.m;
    F->num_rounds = T.num_rounds;
    F->low_run = T.low_run;
    F->direct_store = T.direct_store;
    memcpy(F->tile_bits, T.tile_bits, sizeof(F->tile_bits));
    F->tiles_per_state = T.tiles_per_state;
    F->num_tiles = T.num_tiles;
    F->rank_offset = T.rank_offset;
    memcpy(F->nbr, T.nbr, sizeof(F->nbr));
    memcpy(F->rounds, T.rounds, sizeof(Round) * T.num_rounds);
    for (int r = 0; r < T.num_rounds; ++r) {
        const Round& R = T.rounds[r];
        FactRound& FR = F->fr[r];
        for (int h = 0; h < 2; ++h)
            for (int j = 0; j < kRegLog2; ++j) {
                FR.t[h][j] = 0.0;
                FR.pre[h][j] = make_double2(1.0, 0.0);
                FR.toff[h][j] = 0;
                FR.tstride[h][j] = 0;
            }
        int grp = 0;
        for (int g = R.first_gate; g < R.first_gate + R.num_gates; ++g) {
            const TileGate& G = T.gates[g];
            if (G.kind == kKindDiagN) {
                if (r == 0 && g == 0 && !F->has_din) {
                    F->has_din = 1;
                    F->din_off = G.offset;
                    memcpy(F->din_r, T.diag_r[G.pad[0]], sizeof(F->din_r));
                } else if (r == T.num_rounds - 1 && g == R.first_gate + R.num_gates - 1) {
                    F->has_dout = 1;
                    F->dout_off = G.offset;
                    memcpy(F->dout_r, T.diag_r[G.pad[0]], sizeof(F->dout_r));
                } else {
                    return false;
                }
                F->ntab = G.cval;
                continue;
            }
            if (F->has_dout) return false;  // D_out must be the last op
            if (G.kind == QS_KIND_CUTPHASE) {
                if (grp != 0) return false;
                grp = 1;
                FR.mid = 1;
                FR.lut_off = G.offset;
                FR.lut_stride = G.stride;
                *phase = true;
                continue;
            }
            const int n = FR.n[grp];
            if (G.kind != kKindShear || G.variant != n || n >= kRegLog2) return false;
            if (G.u[0].y != 0.0) return false;  // only form A shears exist
            FR.t[grp][n] = G.u[0].x;
            if (G.u[1].x != 0.0) {  // pre-diagonal (shared by construction for per-state t)
                FR.pre_any = 1;
                FR.pre[grp][n] = G.u[2];
            }
            if (G.stride != 0) *tables = true;
            FR.toff[grp][n] = G.offset;
            FR.tstride[grp][n] = uint32_t(G.stride);
            FR.n[grp]++;
            if (G.pad[1] != 0) *tables = true;  // per-state pre-diagonals: read per state
        }
    }
    if (*tables) {
        // per-state runs read every t from mats: shared ones with stride 0, the
        // padding from the zero factor.cu appends to every factored program
        for (int r = 0; r < T.num_rounds; ++r) {
            FactRound& FR = F->fr[r];
            for (int h = 0; h < 2; ++h)
                for (int j = FR.n[h]; j < kRegLog2; ++j) FR.toff[h][j] = T.zero_off;
        }
    }
    return true;
}

size_t fact_smem_bytes() {
    return sizeof(double2) * kTileAmps + sizeof(uint64_t) * (kTileAmps >> kLowBits) +
           sizeof(uint64_t) * 256 * kDepTables +
           sizeof(uint32_t) * kMaxRounds * ((1 << kLaneLoBits) + (1 << kLaneHiBits));
}

template <bool TB, bool PH>
void launch_fact_variant(double2* psi, const FactPass& F, const double* mats, const CutTerms& ct,
                         cudaStream_t s) {
    constexpr int kMaxDevices = 64;
    static std::atomic<int> configured[kMaxDevices];
    static int sms_of[kMaxDevices], per_sm_of[kMaxDevices];
    const size_t smem = fact_smem_bytes();
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    if (configured[dev].load(std::memory_order_acquire) == 0) {
        cudaFuncSetAttribute(k_fact<TB, PH>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        int sms = 148, per_sm = 1;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fact<TB, PH>, kTileThreads, smem);
        sms_of[dev] = sms;
        per_sm_of[dev] = per_sm < 1 ? 1 : per_sm;
        configured[dev].store(1, std::memory_order_release);
    }
    uint64_t grid = uint64_t(sms_of[dev]) * per_sm_of[dev];
    if (grid > F.num_tiles) grid = F.num_tiles;
    k_fact<TB, PH><<<unsigned(grid), kTileThreads, smem, s>>>(psi, F, mats, ct);
}

void launch_fact(double2* psi, const FactPass& F, const double* mats, const CutTerms& ct,
                 bool tables, bool phase, cudaStream_t s) {
    if (tables) {
        if (phase) launch_fact_variant<true, true>(psi, F, mats, ct, s);
        else launch_fact_variant<true, false>(psi, F, mats, ct, s);
    } else {
        if (phase) launch_fact_variant<false, true>(psi, F, mats, ct, s);
        else launch_fact_variant<false, false>(psi, F, mats, ct, s);
    }
}

// ---- lean factored pass with TMA tile movement ----------------------------------
// k_fact_tma: one CTA per SM, two groups of 256 threads.  A tile is fetched by
// ONE tensor-map TMA (cp.async.bulk.tensor, SWIZZLE_128B) into a landing buffer
// L that is separate from the groups' reslice buffers W0/W1 (the round-1
// k_fact landed each tile in its single working buffer, so the next tile could
// only be requested in the last round).  Tiles alternate between the groups;
// group g reads its tile out of L in round 0 (straight into registers) and, as
// soon as the group has read it, one thread requests the next tile -- the other
// group's -- into L, so a load is in flight while both groups compute.  Landing
// is signalled on one mbarrier per group (expect_tx = 64 KiB).  The tile's
// shared-memory layout is the TMA layout: tile position p sits at smem bit
// pi(p) (the tensor map's dim order) and 16-byte chunks are XOR-swizzled with
// smem bits 3..5 (SWIZZLE_128B); the host planner (tma_plan) picks the dim
// order so that every register round's quarter-warp lanes hit 8 distinct bank
// groups, and rewrites the rounds' swizzled deposit tables for that layout,
// so the round bodies are k_fact's.
constexpr int kMaxAbsorbCtl = 16;
struct alignas(64) TmaPass {
    CUtensorMap map;             // 128 bytes, 64-byte aligned
    int32_t rank;                // tensor dims (2..5)
    int32_t ncoord;              // dims whose coordinate comes from the tile index
    int32_t coord_dim[5];
    int32_t coord_shift[5];      // first tile-index bit of the field
    int32_t coord_lsh[5];        // the field sits above the dim's box bits
    int32_t pad_;
    uint64_t coord_mask[5];      // ~0 for the top field
    int32_t sig[kTileLog2];      // smem index of each tile-position basis vector
    int32_t prefetch;            // L2 prefetch distance in tiles of this CTA
    // absorbed CNOTs (AbsorbCnots): `sig` then holds the permuted copy-out
    // columns; controls outside the tile flip these smem bits per tile
    int32_t nctl;
    int32_t ctl_bit[kMaxAbsorbCtl];
    int32_t ctl_sig[kMaxAbsorbCtl];
};
// host only: the tile pieces above qubits 0..2 in the map's dim order (the
// pair plan rebuilds a 13-bit map from them)
struct TmaPieces {
    int32_t npieces, piece_lo[kTileLog2], piece_len[kTileLog2];
};

constexpr int kTmaThreads = 2 * kTileThreads;
constexpr uint32_t kTileBytes = uint32_t(sizeof(double2)) * kTileAmps;

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    unsigned done = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
            "selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}

// thread-uniform: issue the whole tile as one tensor copy, landing on `bar`
__device__ __forceinline__ void tma_load_tile(const TmaPass& T, uint64_t tile, double2* dst,
                                              uint64_t* bar) {
    int c[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 5; ++i)
        if (i < T.ncoord)
            c[T.coord_dim[i]] = int(((tile >> T.coord_shift[i]) & T.coord_mask[i]) << T.coord_lsh[i]);
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kTileBytes)
                 : "memory");
    const void* map = &T.map;
    switch (T.rank) {
        case 2:
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3}], [%4];" ::"r"(d), "l"(map), "r"(c[0]), "r"(c[1]), "r"(b)
                : "memory");
            break;
        case 3:
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(d), "l"(map), "r"(c[0]), "r"(c[1]),
                "r"(c[2]), "r"(b)
                : "memory");
            break;
        case 4:
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(d), "l"(map), "r"(c[0]), "r"(c[1]),
                "r"(c[2]), "r"(c[3]), "r"(b)
                : "memory");
            break;
        default:
            asm volatile(
                "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d), "l"(map), "r"(c[0]),
                "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b)
                : "memory");
            break;
    }
}

// L2 prefetch of a whole tile (one instruction): the DRAM read of tile k+d
// starts while tiles k..k+d-1 are in flight, so the load into L hits L2
__device__ __forceinline__ void tma_prefetch_tile(const TmaPass& T, uint64_t tile) {
    int c[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 5; ++i)
        if (i < T.ncoord)
            c[T.coord_dim[i]] = int(((tile >> T.coord_shift[i]) & T.coord_mask[i]) << T.coord_lsh[i]);
    const void* map = &T.map;
    switch (T.rank) {
        case 2:
            asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map),
                         "r"(c[0]), "r"(c[1])
                         : "memory");
            break;
        case 3:
            asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map),
                         "r"(c[0]), "r"(c[1]), "r"(c[2])
                         : "memory");
            break;
        case 4:
            asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                             map),
                         "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3])
                         : "memory");
            break;
        default:
            asm volatile(
                "cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(map),
                "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
                : "memory");
            break;
    }
}

template <bool TABLES, bool PHASE, bool PREOK, bool DIAGOK>
__global__ void __launch_bounds__(kTmaThreads, 1)
    k_fact_tma(double2* __restrict__ psi, const __grid_constant__ FactPass P,
               const double* __restrict__ mats, const __grid_constant__ CutTerms ct,
               const __grid_constant__ TmaPass T) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double2* Lbuf = reinterpret_cast<double2*>(smem_raw);
    uint64_t* rowoff = reinterpret_cast<uint64_t*>(smem_raw + 3 * kTileBytes);
    uint64_t* dep = rowoff + (kTileAmps >> kLowBits);
    uint32_t* rlo = reinterpret_cast<uint32_t*>(dep + 256 * kDepTables);
    uint32_t* rhi = rlo + kMaxRounds * (1 << kLaneLoBits);
    uint64_t* full = reinterpret_cast<uint64_t*>(rhi + kMaxRounds * (1 << kLaneHiBits));
    for (int i = threadIdx.x; i < P.num_rounds * (1 << kLaneLoBits); i += kTmaThreads) {
        const Round& R = P.rounds[i >> kLaneLoBits];
        const int v = i & ((1 << kLaneLoBits) - 1);
        rlo[i] = uint32_t(R.dlo[v]) | (uint32_t(R.slo[v]) << 16);
    }
    for (int i = threadIdx.x; i < P.num_rounds * (1 << kLaneHiBits); i += kTmaThreads) {
        const Round& R = P.rounds[i >> kLaneHiBits];
        const int v = i & ((1 << kLaneHiBits) - 1);
        rhi[i] = uint32_t(R.dhi[v]) | (uint32_t(R.shi[v]) << 16);
    }
    const int low_run = P.low_run;
    const int nrows = kTileAmps >> low_run;
    const uint64_t lowmask = (uint64_t(1) << low_run) - 1;
    for (int r = threadIdx.x; r < nrows; r += kTmaThreads) {
        uint64_t off = 0;
        for (int k = 0; k < kTileLog2 - low_run; ++k)
            if ((r >> k) & 1) off |= uint64_t(1) << P.tile_bits[low_run + k];
        rowoff[r] = off;
    }
    for (int i = threadIdx.x; i < kDepTables * 256; i += kTmaThreads) {
        const int c = i >> 8, v = i & 255;
        uint64_t out = 0;
        for (int b = 0; b < 8; ++b) {
            if (!((v >> b) & 1)) continue;
            int want = 8 * c + b, cnt = 0;
            for (int q = 0, k = 0; q < P.m; ++q) {
                if (k < kTileLog2 && P.tile_bits[k] == q) {
                    ++k;
                    continue;
                }
                if (cnt++ == want) {
                    out |= uint64_t(1) << q;
                    break;
                }
            }
        }
        dep[i] = out;
    }
    if (threadIdx.x == 0) {
        mbar_init(full + 0, 1);
        mbar_init(full + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // pool programs that start from a uniform state (H on every qubit of |0..0>,
    // folded by the host): the first pass takes its input from P.cin, no loads
    const bool const_in = TABLES && P.const_in != 0;
    if (threadIdx.x == 0 && blockIdx.x < P.num_tiles && !const_in) {
        tma_load_tile(T, blockIdx.x, Lbuf, full);
        for (int d = 1; d <= T.prefetch; ++d) {
            const uint64_t t = blockIdx.x + uint64_t(d) * gridDim.x;
            if (t < P.num_tiles) tma_prefetch_tile(T, t);
        }
    }

    const int group = threadIdx.x / kTileThreads;  // warp-uniform
    const int tid = threadIdx.x % kTileThreads;
    const int gbar = 1 + group;
    double2* W = Lbuf + kTileAmps * (1 + group);
    const int m = P.m;
    const int tps_log2 = m - kTileLog2;
    auto tile_base = [&](uint64_t t) {
        const uint64_t x = t & (P.tiles_per_state - 1);
        uint64_t out = 0;
#pragma unroll
        for (int c = 0; c < kDepTables; ++c) out |= dep[(c << 8) | ((x >> (8 * c)) & 255)];
        return out;
    };
    auto goff = [&](int e) { return rowoff[e >> low_run] + (uint64_t(e) & lowmask); };
    auto sig_of = [&](int e) {
        int v = 0;
#pragma unroll
        for (int b = 0; b < kTileLog2; ++b)
            if ((e >> b) & 1) v ^= T.sig[b];
        return v;
    };
    const bool direct = P.direct_store != 0;
    unsigned parity = 0;
    for (uint64_t k = group;; k += 2, parity ^= 1) {
        const uint64_t tile_id = blockIdx.x + k * gridDim.x;
        if (tile_id >= P.num_tiles) break;
        const uint64_t st = tile_id >> tps_log2;
        const uint64_t base_local = tile_base(tile_id);
        double2* gbase = psi + ((st << m) | base_local);
        if (!const_in) mbar_wait(full + group, parity);
        for (int r = 0; r < P.num_rounds; ++r) {
            const Round& R = P.rounds[r];
            const bool last = r == P.num_rounds - 1;
            const uint32_t lo = rlo[(r << kLaneLoBits) | (tid & ((1 << kLaneLoBits) - 1))];
            const uint32_t hi = rhi[(r << kLaneHiBits) | (tid >> kLaneLoBits)];
            const int eb = int((lo | hi) & 0xffff);
            const int sb = int((lo ^ hi) >> 16);
            int skb[kRegLog2];
#pragma unroll
            for (int j = 0; j < kRegLog2; ++j) skb[j] = R.sk[1 << j];
            auto sk_of = [&](int kk) {
                int v = 0;
#pragma unroll
                for (int j = 0; j < kRegLog2; ++j)
                    if ((kk >> j) & 1) v ^= skb[j];
                return v;
            };
            const double2* src = r == 0 ? Lbuf : W;
            double2 a[kRegAmps];
            if (r == 0 && const_in) {
                const double2 c = P.cin;
#pragma unroll
                for (int kk = 0; kk < kRegAmps; ++kk) a[kk] = c;
            } else {
#pragma unroll
                for (int kk = 0; kk < kRegAmps; ++kk) a[kk] = src[sb ^ sk_of(kk)];
            }
            if (r == 0 && !const_in) {
                // the group has read L: request the next tile (the other group's)
                named_sync(gbar, kTileThreads);
                if (tid == 0) {
                    const uint64_t next = blockIdx.x + (k + 1) * gridDim.x;
                    if (next < P.num_tiles) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        tma_load_tile(T, next, Lbuf, full + ((k + 1) & 1));
                    }
                    const uint64_t ahead = next + uint64_t(T.prefetch) * gridDim.x;
                    if (T.prefetch > 0 && ahead < P.num_tiles) tma_prefetch_tile(T, ahead);
                }
            }
            const FactRound& F = P.fr[r];
            const bool gstore = last && direct;
            const int sel = int(r == 0 && P.has_din) | (F.pre_any ? 2 : 0) |
                            int(last && P.has_dout) << 2 | int(gstore) << 3;
            const uint64_t il = base_local + rowoff[eb >> low_run] + (uint64_t(eb) & lowmask);
            uint64_t okb[kRegLog2];
#pragma unroll
            for (int j = 0; j < kRegLog2; ++j) okb[j] = gstore ? goff(R.dk[1 << j]) : 0;
            double2* gb = gbase + (gstore ? goff(eb) : 0);
            if (PHASE && F.mid) {
                QSB_FBP(TABLES, (PHASE && true), PREOK, DIAGOK, sel, a, P, R, F, ct, mats, st, il, W, sb, skb, gb, okb)
            } else {
                QSB_FBP(TABLES, false, PREOK, DIAGOK, sel, a, P, R, F, ct, mats, st, il, W, sb, skb, gb, okb)
            }
            if (gstore) break;
            named_sync(gbar, kTileThreads);
        }
        if (!direct) {
            double2* gb = gbase + goff(tid);
            int s_tid = sig_of(tid);
            for (int j = 0; j < T.nctl; ++j)  // absorbed CNOTs controlled from outside the tile
                if ((base_local >> T.ctl_bit[j]) & 1) s_tid ^= T.ctl_sig[j];
#pragma unroll
            for (int i = 0; i < kLoadsPerThread; ++i)
                gb[goff(i * kTileThreads)] = W[s_tid ^ sig_of(i * kTileThreads)];
        }
    }
}

size_t fact_tma_smem_bytes() {
    return 3 * size_t(kTileBytes) + sizeof(uint64_t) * (kTileAmps >> kLowBits) +
           sizeof(uint64_t) * 256 * kDepTables +
           sizeof(uint32_t) * kMaxRounds * ((1 << kLaneLoBits) + (1 << kLaneHiBits)) +
           2 * sizeof(uint64_t);
}

// ---- host: the TMA plan of a lean pass ------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = []() -> EncodeTiledFn {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// One dimension of the tensor map: `len` consecutive local qubits from `lo`
// (tile: box covers them; non-tile: box 1, coordinate = tile-index field),
// or the pool's state index on top.
struct TmaDim {
    int lo, len;
    bool tile;
    bool states;        // the top non-tile run merged with the state index
    int field_shift;    // non-tile: first tile-index bit of this run
};

// Rewrite the rounds' lane orders and swizzled deposits for smem index
// sigma(e) = pi(e) ^ ((pi(e) >> 3) & 7), where pi sends tile position p to
// smem bit pos_bit[p]; lanes 0..2 (a quarter warp) take one position of each
// bank class, preferring tile positions 0,1,2 (128-byte rows for direct stores).
bool retarget_rounds(FactPass& F, const int pos_bit[kTileLog2], int sig[kTileLog2]) {
    auto pi = [&](int e) {
        int v = 0;
        for (int p = 0; p < kTileLog2; ++p)
            if ((e >> p) & 1) v |= 1 << pos_bit[p];
        return v;
    };
    auto sigma = [&](int e) {
        const int v = pi(e);
        return v ^ ((v >> 3) & 7);
    };
    int cls[kTileLog2];
    for (int p = 0; p < kTileLog2; ++p) {
        const int b = pos_bit[p];
        cls[p] = b < 3 ? b : (b < 6 ? b - 3 : -1);
        sig[p] = sigma(1 << p);
    }
    for (int r = 0; r < F.num_rounds; ++r) {
        Round& R = F.rounds[r];
        unsigned regs = 0;
        for (int j = 0; j < kRegLog2; ++j) regs |= R.dk[1 << j];
        int lanes[kTileLog2 - kRegLog2], nl = 0;
        for (int p = 0; p < kTileLog2; ++p)
            if (!((regs >> p) & 1)) lanes[nl++] = p;
        if (nl != kTileLog2 - kRegLog2) return false;
        int order[kTileLog2 - kRegLog2], no = 0;
        unsigned used = 0;
        if (!((regs >> 0) & 1) && !((regs >> 1) & 1) && !((regs >> 2) & 1)) {
            for (int p = 0; p < 3; ++p) order[no++] = p, used |= 1u << p;
        } else {
            for (int c = 0; c < 3; ++c) {
                int pick = -1;
                for (int i = 0; i < nl && pick < 0; ++i)
                    if (cls[lanes[i]] == c && !((used >> lanes[i]) & 1)) pick = lanes[i];
                if (pick < 0) return false;  // a class with no lane: conflicts
                order[no++] = pick;
                used |= 1u << pick;
            }
        }
        for (int i = 0; i < nl; ++i)
            if (!((used >> lanes[i]) & 1)) order[no++] = lanes[i];
        auto deposit = [](int v, const int* pos, int nbits) {
            int out = 0;
            for (int b = 0; b < nbits; ++b)
                if ((v >> b) & 1) out |= 1 << pos[b];
            return out;
        };
        for (int v = 0; v < (1 << kLaneLoBits); ++v) {
            R.dlo[v] = uint16_t(deposit(v, order, kLaneLoBits));
            R.slo[v] = uint16_t(sigma(R.dlo[v]));
        }
        for (int v = 0; v < (1 << kLaneHiBits); ++v) {
            R.dhi[v] = uint16_t(deposit(v, order + kLaneLoBits, kLaneHiBits));
            R.shi[v] = uint16_t(sigma(R.dhi[v]));
        }
        for (int v = 0; v < (1 << kRegLog2); ++v) R.sk[v] = uint16_t(sigma(R.dk[v]));
    }
    if (F.direct_store) {
        // the last round must still put tile positions 0,1,2 on lanes 0..2
        const Round& R = F.rounds[F.num_rounds - 1];
        for (int p = 0; p < 3; ++p)
            if (R.dlo[1 << p] != (1 << p)) return false;
    }
    return true;
}

CUtensorMapL2promotion l2_promotion() {
    static const int v = getenv("QSB_TMA_PROMO") ? atoi(getenv("QSB_TMA_PROMO")) : 128;
    return v >= 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                    : v >= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
}

bool tma_plan(FactPass& F, double2* psi, TmaPass* T, TmaPieces* pieces = nullptr) {
    static const bool off = getenv("QSB_NO_TMA") != nullptr;
    static const bool dbg = getenv("QSB_DEBUG_TMA") != nullptr;
    if (dbg) {
        fprintf(stderr, "tma_plan: m=%d low_run=%d rounds=%d tile_bits=", F.m, F.low_run, F.num_rounds);
        for (int p = 0; p < kTileLog2; ++p) fprintf(stderr, "%d%s", F.tile_bits[p], p + 1 < kTileLog2 ? "," : "\n");
    }
    if (off || F.low_run < 3 || !encode_fn()) return false;
    const int m = F.m;
    const uint64_t num_states = F.num_tiles / F.tiles_per_state;
    uint64_t is_tile = 0;  // over local qubits
    for (int p = 0; p < kTileLog2; ++p) is_tile |= uint64_t(1) << F.tile_bits[p];
    if (m > 62) return false;
    // position of each qubit among the tile positions (or -1)
    auto pos_of = [&](int q) {
        for (int p = 0; p < kTileLog2; ++p)
            if (F.tile_bits[p] == q) return p;
        return -1;
    };
    // maximal runs above qubit 2
    std::vector<TmaDim> tile_runs, nontile;
    int below = 0;
    for (int q = 3; q < m;) {
        const bool t = ((is_tile >> q) & 1) != 0;
        int e = q;
        while (e + 1 < m && (((is_tile >> (e + 1)) & 1) != 0) == t) ++e;
        TmaDim d{q, e - q + 1, t, false, 0};
        if (t) {
            tile_runs.push_back(d);
        } else {
            d.field_shift = below;
            below += d.len;
            nontile.push_back(d);
        }
        q = e + 1;
    }
    if (num_states > 1) {
        if (!nontile.empty() && nontile.back().lo + nontile.back().len == m)
            nontile.back().states = true;
        else
            nontile.push_back(TmaDim{m, 0, false, true, below});
    }
    // candidate XOR sources: 3 consecutive positions of one tile run, that
    // piece first in dim order; the monotone order is tried first
    struct Cand { int run, start; };
    std::vector<Cand> cands;
    for (int i = 0; i < (int)tile_runs.size(); ++i)
        if (tile_runs[i].len >= 3) cands.push_back({i, tile_runs[i].lo});
    for (int i = 0; i < (int)tile_runs.size(); ++i)
        for (int s = tile_runs[i].lo + 1; s + 2 < tile_runs[i].lo + tile_runs[i].len; ++s)
            cands.push_back({i, s});
    for (const Cand& c : cands) {
        // tile pieces: [start, start+len') first (<= 8 qubits), then the rest
        std::vector<TmaDim> dims;
        auto push_tile = [&](int lo, int len) {
            while (len > 0) {
                const int l = std::min(len, 8);
                dims.push_back(TmaDim{lo, l, true, false, 0});
                lo += l;
                len -= l;
            }
        };
        const TmaDim& R0 = tile_runs[c.run];
        push_tile(c.start, R0.lo + R0.len - c.start);
        push_tile(R0.lo, c.start - R0.lo);
        for (int i = 0; i < (int)tile_runs.size(); ++i)
            if (i != c.run) push_tile(tile_runs[i].lo, tile_runs[i].len);
        // every non-tile run rides on the dim just below it in qubit order
        // (box = that dim's tile bits, the run's field is the coordinate above
        // them), so the map has one dim per tile piece: dim0 (qubits 0..2) and
        // the pieces above
        // (measured slower than separate box-1 dims -- config-2 pass 2 6.6 ->
        // 7.4 ms -- so only when the separate dims would exceed rank 5)
        std::vector<int> absorbed(dims.size() + 1, -1);  // index into nontile, per dim (0 = dim0)
        bool merged_all = true;
        const bool merge = 1 + dims.size() + nontile.size() > 5;
        for (int j = 0; merge && j < (int)nontile.size(); ++j) {
            const TmaDim& N = nontile[j];
            int host = -1;
            const int below_q = N.len == 0 ? m : N.lo;  // the state index alone sits above m-1
            if (below_q == 3) host = 0;
            for (int i = 0; i < (int)dims.size() && host < 0; ++i)
                if (dims[i].lo + dims[i].len == below_q) host = i + 1;
            if (host < 0 || absorbed[host] >= 0) {
                merged_all = false;
                break;
            }
            absorbed[host] = j;
        }
        if (!merged_all || 1 + dims.size() > 5) continue;
        std::vector<int> own_dim(nontile.size(), -1);  // unmerged: the run's own dim after the pieces
        if (!merge)
            for (int j = 0; j < (int)nontile.size(); ++j) own_dim[j] = int(dims.size()) + 1 + j;
        // smem bit of each tile position: dim0 = qubits 0..2, then dim order
        int pos_bit[kTileLog2], bit = 3;
        for (int p = 0; p < 3; ++p) pos_bit[p] = p;
        for (const TmaDim& d : dims)
            if (d.tile)
                for (int q = d.lo; q < d.lo + d.len; ++q) pos_bit[pos_of(q)] = bit++;
        if (bit != kTileLog2) continue;
        FactPass G = F;
        int sig[kTileLog2];
        if (!retarget_rounds(G, pos_bit, sig)) continue;
        // the tensor map
        cuuint64_t gdim[5], gstride[4];
        cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
        T->ncoord = 0;
        auto field = [&](int di, int box_lsh, uint64_t* extent) {
            const int j = absorbed[di];
            if (j < 0) return;
            const TmaDim& N = nontile[j];
            *extent *= (uint64_t(1) << N.len) * (N.states ? num_states : 1);
            const int k = T->ncoord++;
            T->coord_dim[k] = di;
            T->coord_shift[k] = N.field_shift;
            T->coord_lsh[k] = box_lsh;
            T->coord_mask[k] = N.states ? ~uint64_t(0) : (uint64_t(1) << N.len) - 1;
        };
        uint64_t ext0 = 16;  // re/im doubles of qubits 0..2
        field(0, 4, &ext0);
        gdim[0] = ext0;
        box[0] = 16;
        bool fits = ext0 <= (uint64_t(1) << 31);
        for (size_t i = 0; i < dims.size(); ++i) {
            const TmaDim& d = dims[i];
            uint64_t extent = uint64_t(1) << d.len;
            field(int(i + 1), d.len, &extent);
            gdim[i + 1] = extent;
            gstride[i] = uint64_t(sizeof(double2)) << d.lo;
            box[i + 1] = 1u << d.len;
            fits &= extent <= (uint64_t(1) << 31);
        }
        for (int j = 0; j < (int)nontile.size(); ++j) {
            if (own_dim[j] < 0) continue;
            const TmaDim& N = nontile[j];
            const int di = own_dim[j];
            const uint64_t extent = (uint64_t(1) << N.len) * (N.states ? num_states : 1);
            gdim[di] = extent;
            gstride[di - 1] = uint64_t(sizeof(double2)) << (N.len == 0 ? m : N.lo);
            box[di] = 1;
            fits &= extent <= (uint64_t(1) << 31);
            const int k = T->ncoord++;
            T->coord_dim[k] = di;
            T->coord_shift[k] = N.field_shift;
            T->coord_lsh[k] = 0;
            T->coord_mask[k] = N.states ? ~uint64_t(0) : (uint64_t(1) << N.len) - 1;
        }
        if (!fits) continue;
        const int rank = int(dims.size()) + 1 + (merge ? 0 : int(nontile.size()));
        if (rank < 2) continue;
        const CUresult rc = encode_fn()(&T->map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, cuuint32_t(rank),
                                        psi, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (rc != CUDA_SUCCESS) continue;
        T->rank = rank;
        for (int p = 0; p < kTileLog2; ++p) T->sig[p] = sig[p];
        if (pieces) {
            pieces->npieces = int(dims.size());
            for (size_t i = 0; i < dims.size(); ++i)
                pieces->piece_lo[i] = dims[i].lo, pieces->piece_len[i] = dims[i].len;
        }
        // L2 prefetch of this CTA's tile after next (QSB_TMA_PF=d: d tiles
        // ahead): measured with the round-1 kernel to help tiles of 128-byte
        // rows over a few 2 MiB pages (config-2 pass 2: 7.2 -> 6.6 ms) and to
        // hurt contiguous tiles and tiles over hundreds of pages (pass 3: 8.1
        // -> 11.2 ms); with the spill-free lean kernels it hurts pass 2 too
        // (6.5 -> 7.5 ms), so it is off by default
        static const int pf_env = getenv("QSB_TMA_PF") ? atoi(getenv("QSB_TMA_PF")) : 0;
        T->prefetch = pf_env;
        F = G;
        if (dbg) fprintf(stderr, "tma_plan: rank %d, prefetch %d\n", rank, T->prefetch);
        return true;
    }
    if (dbg) fprintf(stderr, "tma_plan: no candidate (%zu tried)\n", cands.size());
    return false;
}

template <bool TB, bool PH, bool PO, bool DG>
void launch_fact_tma_variant(double2* psi, const FactPass& F, const double* mats,
                             const CutTerms& ct, const TmaPass& T, cudaStream_t s) {
    constexpr int kMaxDevices = 64;
    static std::atomic<int> configured[kMaxDevices];
    static int sms_of[kMaxDevices];
    const size_t smem = fact_tma_smem_bytes();
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    if (configured[dev].load(std::memory_order_acquire) == 0) {
        cudaFuncSetAttribute(k_fact_tma<TB, PH, PO, DG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem));
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        sms_of[dev] = sms;
        configured[dev].store(1, std::memory_order_release);
    }
    uint64_t grid = uint64_t(sms_of[dev]);
    const uint64_t need = (F.num_tiles + 1) / 2;
    if (grid > need) grid = need;
    k_fact_tma<TB, PH, PO, DG><<<unsigned(grid), kTmaThreads, smem, s>>>(psi, F, mats, ct, T);
}

// ---- lean factored pass over tile PAIRS (256-byte rows) ---------------------------
// k_fact_pair: a 2^12 tile with 128-byte rows (qubits 0..2 + 9 targets, the
// middle and last passes of the config-2 sweep) moves at the copy speed of
// 128-byte rows at large strides (profiles/r02_notes.md: 6.9-8.2 ms per pass
// with no arithmetic); rows of 256 bytes copy in 5.8-6.0 ms.  Here one CTA
// processes the two tiles that differ in the lowest non-tile qubit p (p = 3:
// the rows become 256 bytes) as ONE 128 KiB TMA box: group g (256 threads)
// owns the tile with qubit p = g and runs k_fact's rounds on it.  Shared memory
// holds the 128 KiB landing buffer L and ONE 64 KiB reslice buffer W, which
// the groups take in turns: a group's data lives in registers between rounds
// and occupies W only from the write at the end of a round to the read at the
// start of the next (named-barrier hand-over, turn barriers 3/4).  L is
// re-filled as soon as both groups have read the pair out of it in round 0,
// so 128 KiB per SM are in flight during the whole pair.
struct alignas(64) PairPass {
    CUtensorMap map;             // the 13-bit box
    int32_t ncoord;
    int32_t coord_dim[5], coord_shift[5], coord_lsh[5];
    uint64_t coord_mask[5];
    int32_t gx;                  // smem index of the pair bit (group 1's XOR offset in L)
    uint16_t slo0[1 << kLaneLoBits], shi0[1 << kLaneHiBits], sk0[1 << kRegLog2];  // round 0 in L
};

__device__ __forceinline__ void tma_load_pair(const PairPass& X, uint64_t pair, double2* dst,
                                              uint64_t* bar) {
    int c[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 5; ++i)
        if (i < X.ncoord)
            c[X.coord_dim[i]] = int(((pair >> X.coord_shift[i]) & X.coord_mask[i]) << X.coord_lsh[i]);
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2 * kTileBytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d), "l"(&X.map), "r"(c[0]), "r"(c[1]),
        "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b)
        : "memory");
}

template <bool PREOK, bool DIAGOK>
__global__ void __launch_bounds__(kTmaThreads, 1)
    k_fact_pair(double2* __restrict__ psi, const __grid_constant__ FactPass P,
                const double* __restrict__ mats, const __grid_constant__ CutTerms ct,
                const __grid_constant__ TmaPass T, const __grid_constant__ PairPass X) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double2* Lbuf = reinterpret_cast<double2*>(smem_raw);
    double2* W = Lbuf + 2 * kTileAmps;
    uint64_t* rowoff = reinterpret_cast<uint64_t*>(smem_raw + 3 * kTileBytes);
    uint64_t* dep = rowoff + (kTileAmps >> kLowBits);
    uint32_t* rlo = reinterpret_cast<uint32_t*>(dep + 256 * kDepTables);
    uint32_t* rhi = rlo + kMaxRounds * (1 << kLaneLoBits);
    uint32_t* rlo0 = rhi + kMaxRounds * (1 << kLaneHiBits);
    uint32_t* rhi0 = rlo0 + (1 << kLaneLoBits);
    uint64_t* full = reinterpret_cast<uint64_t*>(rhi0 + (1 << kLaneHiBits));
    unsigned* consumed = reinterpret_cast<unsigned*>(full + 1);
    for (int i = threadIdx.x; i < P.num_rounds * (1 << kLaneLoBits); i += kTmaThreads) {
        const Round& R = P.rounds[i >> kLaneLoBits];
        const int v = i & ((1 << kLaneLoBits) - 1);
        rlo[i] = uint32_t(R.dlo[v]) | (uint32_t(R.slo[v]) << 16);
    }
    for (int i = threadIdx.x; i < P.num_rounds * (1 << kLaneHiBits); i += kTmaThreads) {
        const Round& R = P.rounds[i >> kLaneHiBits];
        const int v = i & ((1 << kLaneHiBits) - 1);
        rhi[i] = uint32_t(R.dhi[v]) | (uint32_t(R.shi[v]) << 16);
    }
    if (threadIdx.x < (1 << kLaneLoBits)) rlo0[threadIdx.x] = X.slo0[threadIdx.x];
    if (threadIdx.x < (1 << kLaneHiBits)) rhi0[threadIdx.x] = X.shi0[threadIdx.x];
    const int low_run = P.low_run;
    const int nrows = kTileAmps >> low_run;
    const uint64_t lowmask = (uint64_t(1) << low_run) - 1;
    for (int r = threadIdx.x; r < nrows; r += kTmaThreads) {
        uint64_t off = 0;
        for (int k = 0; k < kTileLog2 - low_run; ++k)
            if ((r >> k) & 1) off |= uint64_t(1) << P.tile_bits[low_run + k];
        rowoff[r] = off;
    }
    for (int i = threadIdx.x; i < kDepTables * 256; i += kTmaThreads) {
        const int c = i >> 8, v = i & 255;
        uint64_t out = 0;
        for (int b = 0; b < 8; ++b) {
            if (!((v >> b) & 1)) continue;
            int want = 8 * c + b, cnt = 0;
            for (int q = 0, k = 0; q < P.m; ++q) {
                if (k < kTileLog2 && P.tile_bits[k] == q) {
                    ++k;
                    continue;
                }
                if (cnt++ == want) {
                    out |= uint64_t(1) << q;
                    break;
                }
            }
        }
        dep[i] = out;
    }
    const uint64_t num_pairs = P.num_tiles >> 1;
    if (threadIdx.x == 0) {
        mbar_init(full, 1);
        *consumed = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < num_pairs) tma_load_pair(X, blockIdx.x, Lbuf, full);

    const int group = threadIdx.x / kTileThreads;  // warp-uniform: the pair bit of its tile
    const int tid = threadIdx.x % kTileThreads;
    const int gbar = 1 + group;
    const int turn_me = 3 + group, turn_other = 4 - group;
    const int m = P.m;
    const int tps_log2 = m - kTileLog2;
    auto tile_base = [&](uint64_t t) {
        const uint64_t x = t & (P.tiles_per_state - 1);
        uint64_t out = 0;
#pragma unroll
        for (int c = 0; c < kDepTables; ++c) out |= dep[(c << 8) | ((x >> (8 * c)) & 255)];
        return out;
    };
    auto goff = [&](int e) { return rowoff[e >> low_run] + (uint64_t(e) & lowmask); };
    auto sig_of = [&](int e) {
        int v = 0;
#pragma unroll
        for (int b = 0; b < kTileLog2; ++b)
            if ((e >> b) & 1) v ^= T.sig[b];
        return v;
    };
    const bool direct = P.direct_store != 0;
    const int gxg = group ? X.gx : 0;
    bool skip_acq = group == 0;  // group 0 takes W first, without a hand-over
    bool used_w = false;
    unsigned parity = 0;
    for (uint64_t k = 0;; ++k, parity ^= 1) {
        const uint64_t pair = blockIdx.x + k * gridDim.x;
        if (pair >= num_pairs) break;
        const uint64_t tile_id = (pair << 1) | uint64_t(group);
        const uint64_t st = tile_id >> tps_log2;
        const uint64_t base_local = tile_base(tile_id);
        double2* gbase = psi + ((st << m) | base_local);
        mbar_wait(full, parity);
        for (int r = 0; r < P.num_rounds; ++r) {
            const Round& R = P.rounds[r];
            const bool last = r == P.num_rounds - 1;
            const uint32_t lo = rlo[(r << kLaneLoBits) | (tid & ((1 << kLaneLoBits) - 1))];
            const uint32_t hi = rhi[(r << kLaneHiBits) | (tid >> kLaneLoBits)];
            const int eb = int((lo | hi) & 0xffff);
            const int sb = int((lo ^ hi) >> 16);
            int skb[kRegLog2];
#pragma unroll
            for (int j = 0; j < kRegLog2; ++j) skb[j] = R.sk[1 << j];
            double2 a[kRegAmps];
            if (r == 0) {
                // the pair's half of this group, in the 13-bit layout of L
                const int sb0 = int(rlo0[tid & ((1 << kLaneLoBits) - 1)] ^ rhi0[tid >> kLaneLoBits]) ^ gxg;
                int sk0[kRegLog2];
#pragma unroll
                for (int j = 0; j < kRegLog2; ++j) sk0[j] = X.sk0[1 << j];
#pragma unroll
                for (int kk = 0; kk < kRegAmps; ++kk) {
                    int v = 0;
#pragma unroll
                    for (int j = 0; j < kRegLog2; ++j)
                        if ((kk >> j) & 1) v ^= sk0[j];
                    a[kk] = Lbuf[sb0 ^ v];
                }
                named_sync(gbar, kTileThreads);
                if (tid == 0) {
                    // the second group to finish reading requests the next pair
                    __threadfence_block();
                    if (atomicAdd(consumed, 1u) & 1u) {
                        const uint64_t next = pair + gridDim.x;
                        if (next < num_pairs) {
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            tma_load_pair(X, next, Lbuf, full);
                        }
                    }
                }
            } else {
#pragma unroll
                for (int kk = 0; kk < kRegAmps; ++kk) {
                    int v = 0;
#pragma unroll
                    for (int j = 0; j < kRegLog2; ++j)
                        if ((kk >> j) & 1) v ^= skb[j];
                    a[kk] = W[sb ^ v];
                }
                // every thread of the group has its data: W goes to the other group
                named_sync(gbar, kTileThreads);
                named_arrive(turn_other, 2 * kTileThreads);
            }
            const FactRound& F = P.fr[r];
            const bool gstore = last && direct;
            const int sel = int(r == 0 && P.has_din) | (F.pre_any ? 2 : 0) |
                            int(last && P.has_dout) << 2 | int(gstore) << 3;
            const uint64_t il = base_local + rowoff[eb >> low_run] + (uint64_t(eb) & lowmask);
            uint64_t okb[kRegLog2];
#pragma unroll
            for (int j = 0; j < kRegLog2; ++j) okb[j] = gstore ? goff(R.dk[1 << j]) : 0;
            double2* gb = gbase + (gstore ? goff(eb) : 0);
            const int acq = gstore || skip_acq ? 0 : turn_me;
            if (!gstore) skip_acq = false, used_w = true;
            QSB_FBP(false, false, PREOK, DIAGOK, sel, a, P, R, F, ct, mats, st, il, W, sb, skb, gb, okb, acq)
            if (gstore) break;
            named_sync(gbar, kTileThreads);
        }
        if (!direct) {
            double2* gb = gbase + goff(tid);
            int s_tid = sig_of(tid);
            for (int j = 0; j < T.nctl; ++j)  // absorbed CNOTs controlled from outside the tile
                if ((base_local >> T.ctl_bit[j]) & 1) s_tid ^= T.ctl_sig[j];
#pragma unroll
            for (int i = 0; i < kLoadsPerThread; ++i)
                gb[goff(i * kTileThreads)] = W[s_tid ^ sig_of(i * kTileThreads)];
            named_sync(gbar, kTileThreads);
            named_arrive(turn_other, 2 * kTileThreads);
        }
    }
    // group 1's last hand-over has no taker: consume it
    if (group == 0 && used_w) named_sync(turn_me, 2 * kTileThreads);
}

size_t fact_pair_smem_bytes() {
    return 3 * size_t(kTileBytes) + sizeof(uint64_t) * (kTileAmps >> kLowBits) +
           sizeof(uint64_t) * 256 * kDepTables +
           sizeof(uint32_t) * (kMaxRounds + 1) * ((1 << kLaneLoBits) + (1 << kLaneHiBits)) +
           sizeof(uint64_t) + sizeof(unsigned) + 8;
}

// The 13-bit map of a pair: the 12-bit plan's tile pieces in its order, the
// pair bit p as its own dim -- dim 1 when p = 3 (256-byte rows), the last dim
// when p is above every tile qubit -- and every non-tile run riding on the dim
// just below it in qubit order.  Round 0's deposits re-swizzled for L.
bool pair_plan(const FactPass& F, const TmaPieces& T, double2* psi, PairPass* X) {
    static const bool off = getenv("QSB_NO_PAIR") != nullptr;
    if (off || F.low_run < 3 || (F.num_tiles & 1)) return false;
    const int m = F.m;
    uint64_t is_tile = 0;
    for (int q = 0; q < kTileLog2; ++q) is_tile |= uint64_t(1) << F.tile_bits[q];
    int p = 0;
    while (p < m && ((is_tile >> p) & 1)) ++p;
    if (p >= m || p >= 31) return false;
    // only where the pair doubles 128-byte rows: contiguous tiles (pass 1 of the
    // sweep) measured slower paired (6.2 -> 6.8 ms)
    const bool pair_row = p == 3;
    static const bool any_pair = getenv("QSB_PAIR_ALL") != nullptr;
    if (!pair_row && (!any_pair || p < F.tile_bits[kTileLog2 - 1])) return false;
    if (uint64_t(1) << (m - kTileLog2) < 2) return false;
    const uint64_t num_states = F.num_tiles / F.tiles_per_state;
    // dims: (lo, len, box bits); the pair dim first or last among the pieces
    struct D { int lo, len; };
    std::vector<D> dims;  // tile dims after dim0, in smem order
    if (pair_row) dims.push_back({3, 1});
    for (int i = 0; i < T.npieces; ++i) dims.push_back({T.piece_lo[i], T.piece_len[i]});
    if (!pair_row) dims.push_back({p, 1});
    if (1 + dims.size() > 5) return false;
    // non-tile runs of the 13-bit set, each on the dim below it
    const uint64_t set13 = is_tile | (uint64_t(1) << p);
    struct N { int lo, len, field_shift; bool states; };
    std::vector<N> nontile;
    int below = 0;
    for (int q = 0; q < m;) {
        if ((set13 >> q) & 1) { ++q; continue; }
        int e = q;
        while (e + 1 < m && !((set13 >> (e + 1)) & 1)) ++e;
        nontile.push_back({q, e - q + 1, below, false});
        below += e - q + 1;
        q = e + 1;
    }
    if (num_states > 1) {
        if (!nontile.empty() && nontile.back().lo + nontile.back().len == m) nontile.back().states = true;
        else nontile.push_back({m, 0, below, true});
    }
    cuuint64_t gdim[5], gstride[4];
    cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
    uint64_t ext[5];
    ext[0] = 16;
    box[0] = 16;
    for (size_t i = 0; i < dims.size(); ++i) {
        ext[i + 1] = uint64_t(1) << dims[i].len;
        gstride[i] = uint64_t(sizeof(double2)) << dims[i].lo;
        box[i + 1] = 1u << dims[i].len;
    }
    X->ncoord = 0;
    for (const N& n : nontile) {
        int host = -1;
        for (size_t i = 0; i < dims.size() && host < 0; ++i)
            if (dims[i].lo + dims[i].len == n.lo) host = int(i) + 1;
        if (host < 0 && n.lo == 3) host = 0;
        if (host < 0 || X->ncoord >= 5) return false;
        const int lsh = host == 0 ? 4 : dims[host - 1].len;
        ext[host] *= (uint64_t(1) << n.len) * (n.states ? num_states : 1);
        const int k = X->ncoord++;
        X->coord_dim[k] = host;
        X->coord_shift[k] = n.field_shift;
        X->coord_lsh[k] = lsh;
        X->coord_mask[k] = n.states ? ~uint64_t(0) : (uint64_t(1) << n.len) - 1;
    }
    const int rank = int(dims.size()) + 1;
    for (int i = 0; i < rank; ++i) {
        if (ext[i] > (uint64_t(1) << 31)) return false;
        gdim[i] = ext[i];
    }
    for (int i = rank; i < 5; ++i) {  // 5-d map: unit dims on top
        gdim[i] = 1;
        gstride[i - 1] = gstride[i - 2] * 2;
        box[i] = 1;
    }
    if (encode_fn()(&X->map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, psi, gdim, gstride, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    // smem bit of each tile position in L: 0..2 for qubits 0..2, then the dims in order
    auto pos_of = [&](int q) {
        for (int i = 0; i < kTileLog2; ++i)
            if (F.tile_bits[i] == q) return i;
        return -1;
    };
    int pos_bit[kTileLog2], bit = 3, pbit = -1;
    for (int i = 0; i < 3; ++i) pos_bit[i] = i;
    for (const D& d : dims)
        for (int q = d.lo; q < d.lo + d.len; ++q) {
            if (q == p) pbit = bit++;
            else pos_bit[pos_of(q)] = bit++;
        }
    if (bit != kTileLog2 + 1 || pbit < 0) return false;
    auto sigma = [&](int e) {
        int v = 0;
        for (int i = 0; i < kTileLog2; ++i)
            if ((e >> i) & 1) v |= 1 << pos_bit[i];
        return v ^ ((v >> 3) & 7);
    };
    X->gx = (1 << pbit) ^ (((1 << pbit) >> 3) & 7);
    const Round& R0 = F.rounds[0];
    for (int v = 0; v < (1 << kLaneLoBits); ++v) X->slo0[v] = uint16_t(sigma(R0.dlo[v]));
    for (int v = 0; v < (1 << kLaneHiBits); ++v) X->shi0[v] = uint16_t(sigma(R0.dhi[v]));
    for (int v = 0; v < (1 << kRegLog2); ++v) X->sk0[v] = uint16_t(sigma(R0.dk[v]));
    return true;
}

// ---- permutation pass: CNOT-only passes of a factored program ---------------------
// A run of CNOTs is a GF(2)-linear permutation of the index bits (bit t ^= bit
// c per gate); when every target lies in one 2^13-amplitude box (qubits 0..3 =
// 256-byte rows + 9 more bits) the whole run is ONE gather inside the box,
// whatever the number of gates: out[i] = in[A i + B x] (i: box element, x: the
// qubits outside the box, constant per box).  One CTA of 512 threads per SM:
// TMA load of the 128 KiB box (SWIZZLE_128B), every thread reads its 16 source
// elements into registers, the next box is requested, then the registers are
// stored in 256-byte rows (the copy ceiling of these tiles, profiles/
// r02_bigtile_copy.txt).  Factored programs only: the exact mode keeps numpy's
// 0 * a + 1 * b (signed zeros).
constexpr int kPermLog2 = 13;
constexpr int kPermThreads = 512;
constexpr int kPermMaxOut = 32;
struct alignas(64) PermPass {
    CUtensorMap map;
    int32_t ncoord;
    int32_t coord_dim[5], coord_shift[5], coord_lsh[5];
    uint64_t coord_mask[5];
    int32_t m, nout;
    int32_t box_bits[kPermLog2];   // local qubit of each box position (0..3 = qubits 0..3)
    uint64_t num_boxes;
    uint16_t col_sig[kPermLog2];   // swizzled smem index of the SOURCE element of output bit p
    int32_t out_bit[kPermMaxOut];  // qubits outside the box that control a target
    uint16_t out_sig[kPermMaxOut];
};

__global__ void __launch_bounds__(kPermThreads, 1)
    k_perm(double2* __restrict__ psi, const __grid_constant__ PermPass X) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const double2* L = reinterpret_cast<const double2*>(smem_raw);
    uint64_t* dep = reinterpret_cast<uint64_t*>(smem_raw + (sizeof(double2) << kPermLog2));
    uint64_t* full = dep + 256 * kDepTables;
    const int tid = threadIdx.x;
    // box index -> local offset of the box (its bits deposited into the qubits
    // outside the box), one byte of the index per table
    for (int i = tid; i < kDepTables * 256; i += kPermThreads) {
        const int c = i >> 8, v = i & 255;
        uint64_t out = 0;
        for (int b = 0; b < 8; ++b) {
            if (!((v >> b) & 1)) continue;
            int want = 8 * c + b, cnt = 0;
            for (int q = 0, k = 0; q < X.m; ++q) {
                if (k < kPermLog2 && X.box_bits[k] == q) {
                    ++k;
                    continue;
                }
                if (cnt++ == want) {
                    out |= uint64_t(1) << q;
                    break;
                }
            }
        }
        dep[i] = out;
    }
    if (tid == 0) {
        mbar_init(full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto load = [&](uint64_t box) {
        int c[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < 5; ++i)
            if (i < X.ncoord)
                c[X.coord_dim[i]] += int(((box >> X.coord_shift[i]) & X.coord_mask[i]) << X.coord_lsh[i]);
        const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(full));
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_raw));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                     "r"(unsigned(sizeof(double2)) << kPermLog2)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d), "l"(&X.map), "r"(c[0]), "r"(c[1]),
            "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b)
            : "memory");
    };
    if (tid == 0 && blockIdx.x < X.num_boxes) load(blockIdx.x);
    // element e = tid + 512 k: positions 0..8 from the thread, 9..12 from k
    int thr_sig = 0;
    uint64_t thr_off = 0;
#pragma unroll
    for (int p = 0; p < 9; ++p)
        if ((tid >> p) & 1) {
            thr_sig ^= X.col_sig[p];
            thr_off |= uint64_t(1) << X.box_bits[p];
        }
    int ksig[4];
    uint64_t koff[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        ksig[j] = X.col_sig[9 + j];
        koff[j] = uint64_t(1) << X.box_bits[9 + j];
    }
    unsigned parity = 0;
    for (uint64_t box = blockIdx.x; box < X.num_boxes; box += gridDim.x, parity ^= 1) {
        uint64_t base = 0;
#pragma unroll
        for (int c = 0; c < kDepTables; ++c) base |= dep[(c << 8) | ((box >> (8 * c)) & 255)];
        int sig = thr_sig;
        for (int j = 0; j < X.nout; ++j)
            if ((base >> X.out_bit[j]) & 1) sig ^= X.out_sig[j];
        mbar_wait(full, parity);
        double2 a[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            int v = sig;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if ((k >> j) & 1) v ^= ksig[j];
            a[k] = L[v];
        }
        __syncthreads();  // every thread holds its elements: the box buffer is free
        const uint64_t next = box + gridDim.x;
        if (tid == 0 && next < X.num_boxes) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            load(next);
        }
        double2* gb = psi + (base | thr_off);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            uint64_t o = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if ((k >> j) & 1) o |= koff[j];
            gb[o] = a[k];
        }
    }
}

// Host plan of a permutation pass: gates = (control, target) pairs in program
// order, all local, single state.  False when the targets do not fit one box
// or the tensor map cannot be built (the caller falls back to k_tile).
bool launch_perm_pass(double2* psi, int m, const int* controls, const int* targets, int count,
                      cudaStream_t s) {
    static const bool off = getenv("QSB_NO_PERM") != nullptr;
    if (off || m < kPermLog2 + 1 || count < 1 || !encode_fn()) return false;
    uint64_t boxset = 0xF;  // qubits 0..3: 256-byte rows
    for (int i = 0; i < count; ++i) {
        if (targets[i] < 0 || targets[i] >= m || controls[i] < 0 || controls[i] >= m) return false;
        boxset |= uint64_t(1) << targets[i];
    }
    if (__builtin_popcountll(boxset) > kPermLog2) return false;
    for (int q = 4; q < m && __builtin_popcountll(boxset) < kPermLog2; ++q) boxset |= uint64_t(1) << q;
    if (__builtin_popcountll(boxset) != kPermLog2) return false;
    static thread_local PermPass X;
    memset(&X, 0, sizeof(X));
    X.m = m;
    X.num_boxes = uint64_t(1) << (m - kPermLog2);
    // dims: d0 = qubits 0..2 (16 doubles), then the runs of box bits from qubit 3
    // up, each at most 8 bits (box dims are limited to 256 elements)
    struct D { int lo, len; };
    std::vector<D> dims;
    for (int q = 3; q < m;) {
        if (!((boxset >> q) & 1)) { ++q; continue; }
        int e = q;
        while (e + 1 < m && ((boxset >> (e + 1)) & 1) && e + 1 - q < 8) ++e;
        dims.push_back({q, e - q + 1});
        q = e + 1;
    }
    if (1 + dims.size() > 5) return false;
    cuuint64_t gdim[5], gstride[4];
    cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
    uint64_t ext[5];
    ext[0] = 16;
    box[0] = 16;
    for (size_t i = 0; i < dims.size(); ++i) {
        ext[i + 1] = uint64_t(1) << dims[i].len;
        gstride[i] = uint64_t(sizeof(double2)) << dims[i].lo;
        box[i + 1] = 1u << dims[i].len;
    }
    // runs of qubits outside the box ride on the dim just below them; their
    // field of the box index is the coordinate
    int below = 0;
    for (int q = 4; q < m;) {
        if ((boxset >> q) & 1) { ++q; continue; }
        int e = q;
        while (e + 1 < m && !((boxset >> (e + 1)) & 1)) ++e;
        const int len = e - q + 1;
        int host = -1;
        for (size_t i = 0; i < dims.size(); ++i)
            if (dims[i].lo + dims[i].len == q) host = int(i) + 1;
        if (host < 0 || X.ncoord >= 5) return false;
        ext[host] <<= len;
        const int k = X.ncoord++;
        X.coord_dim[k] = host;
        X.coord_shift[k] = below;
        X.coord_lsh[k] = dims[host - 1].len;
        X.coord_mask[k] = (uint64_t(1) << len) - 1;
        below += len;
        q = e + 1;
    }
    const int rank = int(dims.size()) + 1;
    for (int i = 0; i < rank; ++i) {
        if (ext[i] > (uint64_t(1) << 31)) return false;
        gdim[i] = ext[i];
    }
    for (int i = rank; i < 5; ++i) {  // 5-d map: unit dims on top
        gdim[i] = 1;
        gstride[i - 1] = gstride[i - 2] * 2;
        box[i] = 1;
    }
    if (encode_fn()(&X.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, psi, gdim, gstride, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    // box positions in memory order: qubits 0..2, then the dims
    int pos_of_qubit[64];
    for (int q = 0; q < 64; ++q) pos_of_qubit[q] = -1;
    int np = 0;
    for (int q = 0; q < 3; ++q) X.box_bits[np] = q, pos_of_qubit[q] = np++;
    for (const D& d : dims)
        for (int q = d.lo; q < d.lo + d.len; ++q) X.box_bits[np] = q, pos_of_qubit[q] = np++;
    if (np != kPermLog2) return false;
    // the kernel deposits positions in qubit order (box_bits ascending): the dims
    // are in ascending qubit order, so positions and qubits agree
    // source index bits: out[i] = in[f_1(f_2(..f_k(i)))], f_j: bit t_j ^= bit c_j
    uint64_t row[64];
    for (int q = 0; q < m; ++q) row[q] = uint64_t(1) << q;
    for (int j = count - 1; j >= 0; --j) row[targets[j]] ^= row[controls[j]];
    auto sigma = [](int v) { return v ^ ((v >> 3) & 7); };
    auto column = [&](int q) {  // source box positions whose bit depends on output qubit q
        int v = 0;
        for (int b = 0; b < m; ++b)
            if ((row[b] >> q) & 1) {
                if (pos_of_qubit[b] < 0) return -1;  // cannot happen: only targets change
                v |= 1 << pos_of_qubit[b];
            }
        return v;
    };
    for (int p = 0; p < kPermLog2; ++p) {
        const int v = column(X.box_bits[p]);
        if (v < 0) return false;
        X.col_sig[p] = uint16_t(sigma(v));
    }
    for (int q = 0; q < m; ++q) {
        if (pos_of_qubit[q] >= 0) continue;
        int v = 0;
        for (int b = 0; b < m; ++b)
            if (b != q && ((row[b] >> q) & 1)) {
                if (pos_of_qubit[b] < 0) return false;
                v |= 1 << pos_of_qubit[b];
            }
        if (!v) continue;
        if (X.nout >= kPermMaxOut) return false;
        X.out_bit[X.nout] = q;
        X.out_sig[X.nout++] = uint16_t(sigma(v));
    }
    constexpr int kMaxDevices = 64;
    static std::atomic<int> configured[kMaxDevices];
    static int sms_of[kMaxDevices];
    const size_t smem = (sizeof(double2) << kPermLog2) + sizeof(uint64_t) * (256 * kDepTables + 1);
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    if (configured[dev].load(std::memory_order_acquire) == 0) {
        cudaFuncSetAttribute(k_perm, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        sms_of[dev] = sms;
        configured[dev].store(1, std::memory_order_release);
    }
    uint64_t grid = uint64_t(sms_of[dev]);
    if (grid > X.num_boxes) grid = X.num_boxes;
    k_perm<<<unsigned(grid), kPermThreads, smem, s>>>(psi, X);
    return true;
}

template <bool PO, bool DG>
void launch_fact_pair_variant(double2* psi, const FactPass& F, const double* mats,
                              const CutTerms& ct, const TmaPass& T, const PairPass& X,
                              cudaStream_t s) {
    constexpr int kMaxDevices = 64;
    static std::atomic<int> configured[kMaxDevices];
    static int sms_of[kMaxDevices];
    const size_t smem = fact_pair_smem_bytes();
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    if (configured[dev].load(std::memory_order_acquire) == 0) {
        cudaFuncSetAttribute(k_fact_pair<PO, DG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem));
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        sms_of[dev] = sms;
        configured[dev].store(1, std::memory_order_release);
    }
    uint64_t grid = uint64_t(sms_of[dev]);
    const uint64_t need = F.num_tiles / 2;
    if (grid > need) grid = need;
    k_fact_pair<PO, DG><<<unsigned(grid), kTmaThreads, smem, s>>>(psi, F, mats, ct, T, X);
}

bool launch_fact_tma(double2* psi, FactPass& F, const double* mats, const CutTerms& ct,
                     bool tables, bool phase, cudaStream_t s) {
    static thread_local TmaPass T;
    static thread_local TmaPieces pieces;
    // a CNOT pass behind this one (g_absorb): composed into the copy-out when all
    // its targets are tile qubits (out[i] = in[f_1(..f_k(i))], f_j: bit t_j ^= bit c_j)
    AbsorbCnots& ab = g_absorb;
    static const bool absorb_ok = getenv("QSB_NO_ABSORB") == nullptr;
    bool absorb = absorb_ok && ab.count > 0 && !ab.done && F.num_tiles == F.tiles_per_state;
    uint64_t row[64];
    int pos_of_qubit[64];
    if (absorb) {
        for (int q = 0; q < 64; ++q) row[q] = uint64_t(1) << q, pos_of_qubit[q] = -1;
        for (int p = 0; p < kTileLog2; ++p) pos_of_qubit[F.tile_bits[p]] = p;
        for (int j = ab.count - 1; j >= 0 && absorb; --j) {
            const int t = ab.targets[j], c = ab.controls[j];
            if (t < 0 || t >= F.m || c < 0 || c >= F.m || pos_of_qubit[t] < 0) absorb = false;
            else row[t] ^= row[c];
        }
        int outside = 0;
        for (int q = 0; q < F.m && absorb; ++q) {
            if (pos_of_qubit[q] >= 0) continue;
            bool used = false;
            for (int p = 0; p < kTileLog2; ++p) used |= ((row[F.tile_bits[p]] >> q) & 1) != 0;
            outside += used;
        }
        if (outside > kMaxAbsorbCtl) absorb = false;
    }
    const int saved_direct = F.direct_store;
    if (absorb) F.direct_store = 0;  // the tile goes back through shared memory
    if (!tma_plan(F, psi, &T, &pieces)) {
        F.direct_store = saved_direct;
        if (!absorb) return false;
        absorb = false;  // no conflict-free lane order without the direct store: plain pass
        if (!tma_plan(F, psi, &T, &pieces)) return false;
    }
    T.nctl = 0;
    if (absorb) {
        int sig2[kTileLog2];
        auto column = [&](int q) {
            int v = 0;
            for (int p = 0; p < kTileLog2; ++p)
                if ((row[F.tile_bits[p]] >> q) & 1) v ^= T.sig[p];
            return v;
        };
        for (int b = 0; b < kTileLog2; ++b) sig2[b] = column(F.tile_bits[b]);
        for (int q = 0; q < F.m; ++q) {
            if (pos_of_qubit[q] >= 0) continue;
            const int v = column(q);
            if (!v) continue;
            T.ctl_bit[T.nctl] = q;
            T.ctl_sig[T.nctl++] = v;
        }
        for (int b = 0; b < kTileLog2; ++b) T.sig[b] = sig2[b];
        ab.done = true;
    }
    bool pre = false;
    for (int r = 0; r < F.num_rounds; ++r) pre |= F.fr[r].pre_any != 0;
    const bool diag = F.has_din || F.has_dout;
    if (!tables && !phase) {
        static thread_local PairPass X;
        if (pair_plan(F, pieces, psi, &X)) {
            if (pre) {
                if (diag) launch_fact_pair_variant<true, true>(psi, F, mats, ct, T, X, s);
                else launch_fact_pair_variant<true, false>(psi, F, mats, ct, T, X, s);
            } else {
                if (diag) launch_fact_pair_variant<false, true>(psi, F, mats, ct, T, X, s);
                else launch_fact_pair_variant<false, false>(psi, F, mats, ct, T, X, s);
            }
            return true;
        }
    }
    const int v = int(tables) | int(phase) << 1 | int(pre) << 2 | int(diag) << 3;
    switch (v) {
#define QSB_TMA_CASE(V) \
    case V: launch_fact_tma_variant<(V & 1) != 0, (V & 2) != 0, (V & 4) != 0, (V & 8) != 0>(psi, F, mats, ct, T, s); break;
        QSB_TMA_CASE(0) QSB_TMA_CASE(1) QSB_TMA_CASE(2) QSB_TMA_CASE(3)
        QSB_TMA_CASE(4) QSB_TMA_CASE(5) QSB_TMA_CASE(6) QSB_TMA_CASE(7)
        QSB_TMA_CASE(8) QSB_TMA_CASE(9) QSB_TMA_CASE(10) QSB_TMA_CASE(11)
        QSB_TMA_CASE(12) QSB_TMA_CASE(13) QSB_TMA_CASE(14) QSB_TMA_CASE(15)
#undef QSB_TMA_CASE
    }
    return true;
}

// |index> in every state of a pool after a zero fill: one amplitude per state
__global__ void k_set_basis(double2* __restrict__ psi, uint64_t stride, uint64_t states,
                            uint64_t off) {
    for (uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < states;
         s += uint64_t(gridDim.x) * blockDim.x)
        psi[s * stride + off] = make_double2(1.0, 0.0);
}

__global__ void k_fill(double2* __restrict__ psi, uint64_t count, double2 value) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x)
        psi[i] = value;
}

__global__ void k_scale(double2* __restrict__ psi, uint64_t count, double f) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        double2 v = psi[i];
        psi[i] = make_double2(__dmul_rn(v.x, f), __dmul_rn(v.y, f));
    }
}

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Box-Muller on two 53-bit uniforms derived from (seed, state, global index):
// the same amplitude gets the same value for any rank split.
__global__ void k_gaussian(double2* __restrict__ psi, uint64_t per_state, int m, uint64_t total,
                           uint64_t rank_offset, uint64_t seed) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t s = i >> m, g = rank_offset | (i & (per_state - 1));
        uint64_t h = splitmix(seed ^ splitmix(s * 0x632BE59BD9B4E019ull ^ splitmix(g)));
        uint64_t h2 = splitmix(h);
        double u1 = (double((h >> 11) + 1)) * 0x1.0p-53;  // (0, 1]
        double u2 = double(h2 >> 11) * 0x1.0p-53;         // [0, 1)
        double r = sqrt(-2.0 * log(u1));
        double sn, cs;
        sincospi(2.0 * u2, &sn, &cs);
        psi[i] = make_double2(r * cs, r * sn);
    }
}

inline unsigned grid_for(uint64_t work, uint64_t per_block) {
    uint64_t g = (work + per_block - 1) / per_block;
    return unsigned(g == 0 ? 1 : g);
}

inline unsigned stream_grid(uint64_t count) {
    // grid-stride loops: a few waves over the 148 SMs
    uint64_t g = (count + 255) / 256;
    uint64_t cap = 148ull * 16;
    return unsigned(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

void launch_gate1q(double2* psi, int m, int num_states, int q, const double* mats, uint64_t offset,
                   uint64_t stride, cudaStream_t s) {
    uint64_t total = uint64_t(num_states) << (m - 1);
    k_gate1q<<<grid_for(total, kThreads * kIlp), kThreads, 0, s>>>(psi, m, q, total, mats, offset,
                                                                    stride);
}

void launch_controlled(double2* psi, int m, int num_states, int c, int t, const double* mats,
                       uint64_t offset, uint64_t stride, bool diag_one, cudaStream_t s) {
    uint64_t total = uint64_t(num_states) << (m - 2);
    k_controlled<<<grid_for(total, kThreads * kIlp), kThreads, 0, s>>>(
        psi, m, c, t, total, mats, offset, stride, diag_one ? 1 : 0);
}

void launch_cut_phase(double2* psi, int m, int num_states, uint64_t rank_offset, const CutTerms& ct,
                      const double* mats, uint64_t offset, uint64_t stride, cudaStream_t s) {
    uint64_t total = uint64_t(num_states) << m;
    k_cut_phase<<<grid_for(total, kThreads * kIlp), kThreads, 0, s>>>(psi, m, total, rank_offset,
                                                                       ct, mats, offset, stride);
}

bool tile_pass_in_params() {
#ifdef QSB_PASS_PARAM
    return true;
#else
    return false;
#endif
}

size_t tile_smem_bytes() {
#ifdef QSB_PASS_PARAM
    const size_t pass_bytes = 0;
#else
    const size_t pass_bytes = sizeof(TilePass);
#endif
    return kGroups * sizeof(double2) * kTileAmps + sizeof(uint64_t) * (kTileAmps >> kLowBits) +
           pass_bytes + sizeof(uint64_t) * 256 * kDepTables +
           sizeof(uint32_t) * kMaxRounds * ((1 << kLaneLoBits) + (1 << kLaneHiBits)) +
           2 * sizeof(double2) * 4 * kMaxPassGates;
}

template <bool PH, bool GE, bool TB, bool FA>
void launch_tile_variant(double2* psi, const TilePass& pass, const TilePass* pass_dev,
                         const double* mats,
                         const CutTerms& ct, uint64_t num_tiles, cudaStream_t s) {
    // per device: the shared-memory opt-in is a per-device function attribute
    constexpr int kMaxDevices = 64;
    static std::atomic<int> configured[kMaxDevices];
    static int sms_of[kMaxDevices], per_sm_of[kMaxDevices];
    const size_t smem = tile_smem_bytes();
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    if (configured[dev].load(std::memory_order_acquire) == 0) {
        cudaFuncSetAttribute(k_tile<PH, GE, TB, FA>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        int sms = 148, per_sm = 1;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tile<PH, GE, TB, FA>, kCtaThreads, smem);
        sms_of[dev] = sms;
        per_sm_of[dev] = per_sm < 1 ? 1 : per_sm;
        configured[dev].store(1, std::memory_order_release);
    }
    uint64_t grid = uint64_t(sms_of[dev]) * per_sm_of[dev];
    const uint64_t need = (num_tiles + kGroups - 1) / kGroups;
    if (grid > need) grid = need;
#ifdef QSB_PASS_PARAM
    (void)pass_dev;
    k_tile<PH, GE, TB, FA><<<unsigned(grid), kCtaThreads, smem, s>>>(psi, pass, mats, ct);
#else
    (void)pass;
    k_tile<PH, GE, TB, FA><<<unsigned(grid), kCtaThreads, smem, s>>>(psi, pass_dev, mats, ct);
#endif
}

int launch_tile_pass(double2* psi, const TilePass& pass, const TilePass* pass_dev,
                     const double* mats, const CutTerms& ct, cudaStream_t s) {
    bool phase = false, generic = false, tables = false, fact = false;
    for (int r = 0; r < pass.num_rounds; ++r) {
        const Round& R = pass.rounds[r];
        for (int g = R.first_gate; g < R.first_gate + R.num_gates; ++g) {
            const TileGate& G = pass.gates[g];
            if (G.kind == QS_KIND_CUTPHASE) {
                phase = true;
            } else if (G.kind >= kKindShear) {
                fact = true;
                const int run = G.seq > 0 ? G.seq : 1;
                for (int j = 0; j < run; ++j) tables |= pass.gates[g + j].stride != 0;
                g += run - 1;
            } else {
                // a sequence run covers G.seq gates; any of them may use a table
                const int run = G.seq > 0 ? G.seq : 1;
                for (int j = 0; j < run; ++j) tables |= pass.gates[g + j].stride != 0;
                if (G.seq > 0) g += G.seq - 1;
                else generic = true;
            }
        }
    }
    const uint64_t nt = pass.num_tiles;
    static const bool lean_ok = getenv("QSB_NO_LEAN") == nullptr;
    ConstIn& cin = g_const_in;
    auto fill_now = [&] {  // the constant input written out (no kernel takes it virtually)
        if (cin.on) launch_fill(psi, cin.total, cin.v, s);
        cin.on = false;
    };
    if (fact && !generic && kGroups == 1 && lean_ok) {
        static thread_local FactPass F;
        bool tb = false, ph = false;
        if (fact_pass_from(pass, &F, &tb, &ph)) {
            // a pool pass on the TMA kernel generates a constant input in
            // registers (no fill, no tile loads); everything else fills first
            const bool virt = cin.on && tb;
            if (!virt) fill_now();
            if (virt) F.const_in = 1, F.cin = cin.v;
            if (launch_fact_tma(psi, F, mats, ct, tb, ph, s)) {
                cin.on = false;
                return virt ? 2 : 1;
            }
            F.const_in = 0;
            fill_now();
            launch_fact(psi, F, mats, ct, tb, ph, s);
            return 1;
        }
    }
    fill_now();
#define QSB_TILE_CASE(PH, GE, TB, FA) \
    if (phase == PH && generic == GE && tables == TB && fact == FA) {       \
        launch_tile_variant<PH, GE, TB, FA>(psi, pass, pass_dev, mats, ct, nt, s); \
        return 0;                                                            \
    }
#define QSB_TILE_CASES(FA)               \
    QSB_TILE_CASE(false, false, false, FA) \
    QSB_TILE_CASE(false, false, true, FA)  \
    QSB_TILE_CASE(false, true, false, FA)  \
    QSB_TILE_CASE(false, true, true, FA)   \
    QSB_TILE_CASE(true, false, false, FA)  \
    QSB_TILE_CASE(true, false, true, FA)   \
    QSB_TILE_CASE(true, true, false, FA)   \
    QSB_TILE_CASE(true, true, true, FA)
    QSB_TILE_CASES(false)
    QSB_TILE_CASES(true)
#undef QSB_TILE_CASES
#undef QSB_TILE_CASE
    return 0;
}

thread_local ConstIn g_const_in = {false, {0.0, 0.0}, 0};
thread_local AbsorbCnots g_absorb = {};

bool absorb_tile_feasible(double2* psi, const TilePass& pass) {
    static thread_local FactPass F;
    static thread_local TmaPass T;
    static thread_local TmaPieces pieces;
    bool tb = false, ph = false;
    if (kGroups != 1 || !fact_pass_from(pass, &F, &tb, &ph)) return false;
    F.direct_store = 0;
    return tma_plan(F, psi, &T, &pieces);
}

bool launch_perm(double2* psi, int m, const int* controls, const int* targets, int count,
                 cudaStream_t s) {
    return launch_perm_pass(psi, m, controls, targets, count, s);
}

int prof_read(unsigned long long* out) {
#ifdef QSB_PROF
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_prof, sizeof(g_prof));
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_prof, z, sizeof(z));
    return 1;
#else
    (void)out;
    return 0;
#endif
}

void launch_set_basis(double2* psi, uint64_t stride, uint64_t states, uint64_t off,
                      cudaStream_t s) {
    const unsigned grid = unsigned(std::min<uint64_t>((states + 255) / 256, 1024));
    k_set_basis<<<grid, 256, 0, s>>>(psi, stride, states, off);
}

void launch_fill(double2* psi, uint64_t count, double2 value, cudaStream_t s) {
    k_fill<<<stream_grid(count), 256, 0, s>>>(psi, count, value);
}

void launch_scale(double2* psi, uint64_t count, double factor, cudaStream_t s) {
    k_scale<<<stream_grid(count), 256, 0, s>>>(psi, count, factor);
}

// psi_i *= f_i with numpy's complex product (psi the left operand), the
// reference's `partition.amplitudes *= np.exp(-1j * angles)`
// (statevector.py:198-206) for a host-evaluated phase function.
__global__ void k_mul_factors(double2* __restrict__ psi, const double2* __restrict__ f,
                              uint64_t count) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x)
        psi[i] = cmul(psi[i], f[i]);
}

void launch_mul_factors(double2* psi, const double2* f, uint64_t count, cudaStream_t s) {
    k_mul_factors<<<stream_grid(count), 256, 0, s>>>(psi, f, count);
}

void launch_gaussian(double2* psi, uint64_t per_state, int num_states, uint64_t rank_offset,
                     uint64_t seed, cudaStream_t s) {
    int m = 0;
    while ((uint64_t(1) << m) < per_state) ++m;
    uint64_t total = per_state * uint64_t(num_states);
    k_gaussian<<<stream_grid(total), 256, 0, s>>>(psi, per_state, m, total, rank_offset, seed);
}

}  // namespace qsb
