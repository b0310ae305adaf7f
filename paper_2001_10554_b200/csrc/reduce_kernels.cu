// Observable reductions in the reference's exact association.
//
// The reference sums every observable with tree_sum (statevector.py:29-45): a
// perfect binary tree over element order (x.reshape(-1,2).sum(axis=1) until one
// value).  Here each block reduces an aligned 2^L-element chunk with the same
// pairing (a pairwise tree in shared memory), writes one partial, and the
// partials are reduced again with the same kernel until one value per state
// remains -- exactly the reference's tree, level by level, so the result is
// bit-identical for any chunking.
#include <algorithm>

#include "common.cuh"

namespace qsb {
namespace {

constexpr int kChunkLog2 = 10;
constexpr int kChunk = 1 << kChunkLog2;
constexpr int kThreads = 256;

// element value of one observable (statevector.py:209-251)
__device__ __forceinline__ double obs_value(const double2* __restrict__ psi, int m, int kind,
                                            int q, uint64_t rank_offset, const CutTerms& ct,
                                            uint64_t s, uint64_t j) {
    const uint64_t base = s << m;
    switch (kind) {
        case QS_OBS_PROB: {
            // elements of psi[(idx >> q) & 1 == 1] in ascending order
            uint64_t off = insert0(j, q) | (uint64_t(1) << q);
            return abs2(psi[base | off]);
        }
        case QS_OBS_Z: {
            double w = ((rank_offset | j) >> q) & 1 ? -1.0 : 1.0;
            return __dmul_rn(w, abs2(psi[base | j]));
        }
        case QS_OBS_MAXCUT: {
            double c = double(cut_of(rank_offset | j, ct));
            return __dmul_rn(c, abs2(psi[base | j]));
        }
        default:
            return abs2(psi[base | j]);
    }
}

// Tree over aligned chunks of `chunk` (power of two, <= kChunk) elements.
// Level 0 reads the state; later levels read `src` partials.
__global__ void __launch_bounds__(kThreads)
    k_tree(const double2* __restrict__ psi, const double* __restrict__ src, double* __restrict__ dst,
           int m, int kind, int q, uint64_t rank_offset, const __grid_constant__ CutTerms ct,
           uint64_t elems_per_state, int chunk_log2, uint64_t total_chunks) {
    __shared__ double buf[kChunk];
    const int chunk = 1 << chunk_log2;
    const uint64_t chunks_per_state = elems_per_state >> chunk_log2;
    for (uint64_t c = blockIdx.x; c < total_chunks; c += gridDim.x) {
        const uint64_t s = c / chunks_per_state;
        const uint64_t first = (c - s * chunks_per_state) << chunk_log2;
        for (int i = threadIdx.x; i < chunk; i += kThreads) {
            double v;
            if (psi)
                v = obs_value(psi, m, kind, q, rank_offset, ct, s, first + i);
            else
                v = src[s * elems_per_state + first + i];
            buf[i] = v;
        }
        __syncthreads();
        for (int w = 1; w < chunk; w <<= 1) {
            for (int i = threadIdx.x; i * 2 * w < chunk; i += kThreads)
                buf[i * 2 * w] = __dadd_rn(buf[i * 2 * w], buf[i * 2 * w + w]);
            __syncthreads();
        }
        if (threadIdx.x == 0) dst[c] = buf[0];
        __syncthreads();
    }
}

// Fast path for chunks of exactly 2048 elements: warp w of the block covers
// elements [256w, 256w+256) as 8 coalesced groups of 32; each group is reduced
// by a shuffle butterfly (xor 1,2,4,8,16 pairs adjacent elements first, and
// IEEE addition is commutative, so every lane ends with the tree sum of the
// group), the 8 group sums are combined as a tree in registers, and the 8
// warp sums as a tree in shared memory -- the same association as tree_sum.
constexpr int kWideLog2 = 11;
__device__ __forceinline__ double warp_tree(double v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__global__ void __launch_bounds__(kThreads)
    k_tree_wide(const double2* __restrict__ psi, const double* __restrict__ src,
                double* __restrict__ dst, int m, int kind, int q, uint64_t rank_offset,
                const __grid_constant__ CutTerms ct, uint64_t elems_per_state,
                uint64_t total_chunks) {
    __shared__ double wsum[kThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t chunks_per_state = elems_per_state >> kWideLog2;
    // MAXCUT: a thread's 8 elements differ in qubits 5,6,7 only, so after one
    // full cut_of the other 7 cuts follow by a Gray-code walk (flipping qubit
    // r changes the cut by deg(r) - 2 * (edges of r currently cut))
    const bool walk = psi != nullptr && kind == QS_OBS_MAXCUT;
    uint64_t nbq[3] = {0, 0, 0};
    int degq[3] = {0, 0, 0};
    if (walk) {
        for (int b = 0; b < 3; ++b) {
            const int r = 5 + b;
            for (int k = 0; k < ct.count; ++k) {
                const int sh = ct.shift[k];
                if ((ct.mask[k] >> r) & 1) nbq[b] |= uint64_t(1) << (r + sh);
                if (r >= sh && ((ct.mask[k] >> (r - sh)) & 1)) nbq[b] |= uint64_t(1) << (r - sh);
            }
            degq[b] = __popcll(nbq[b]);
        }
    }
    for (uint64_t c = blockIdx.x; c < total_chunks; c += gridDim.x) {
        const uint64_t s = c / chunks_per_state;
        const uint64_t first = ((c - s * chunks_per_state) << kWideLog2) + warp * 256 + lane;
        double v[8];
        if (walk) {
            const double2* p = psi + (s << m) + first;
            uint64_t i = rank_offset | first;
            int cut = cut_of(i, ct);
            v[0] = __dmul_rn(double(cut), abs2(p[0]));
#pragma unroll
            for (int step = 1; step < 8; ++step) {
                const int b = step & 1 ? 0 : (step & 2 ? 1 : 2);  // bit flipped
                const int gray = step ^ (step >> 1);               // element reached
                const uint64_t bit = (i >> (5 + b)) & 1;
                cut += degq[b] - 2 * __popcll((i ^ (uint64_t(0) - bit)) & nbq[b]);
                i ^= uint64_t(1) << (5 + b);
                v[gray] = __dmul_rn(double(cut), abs2(p[gray * 32]));
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint64_t j = first + i * 32;
                v[i] = psi ? obs_value(psi, m, kind, q, rank_offset, ct, s, j)
                           : src[s * elems_per_state + j];
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = warp_tree(v[i]);
        double t = __dadd_rn(__dadd_rn(__dadd_rn(v[0], v[1]), __dadd_rn(v[2], v[3])),
                             __dadd_rn(__dadd_rn(v[4], v[5]), __dadd_rn(v[6], v[7])));
        if (lane == 0) wsum[warp] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            double b = __dadd_rn(__dadd_rn(__dadd_rn(wsum[0], wsum[1]), __dadd_rn(wsum[2], wsum[3])),
                                 __dadd_rn(__dadd_rn(wsum[4], wsum[5]), __dadd_rn(wsum[6], wsum[7])));
            dst[c] = b;
        }
        __syncthreads();
    }
}

// All marginals P(q=1), q < m, in one pass (states with m >= 11).  A block
// builds the full tree of one aligned 2048-amplitude chunk in shared memory
// (levels 0..11).  For q < 11 the amplitudes with bit q set form the odd nodes
// of level q, so their tree inside the chunk is a tree over those nodes; for
// q >= 11 the chunk is either wholly selected (its root) or not at all.  The
// per-chunk partials are aligned subtrees of each q's selected list, so the
// second level (k_tree over partials) reproduces get_probability's tree_sum.
constexpr int kMargChunkLog2 = 11;
// A block reduces one aligned 2048-amplitude chunk; thread t holds amplitudes
// 8t..8t+7.  With every |psi|^2 >= 0, zeroing the amplitudes whose bit q is 0
// and summing the whole chunk in tree order gives exactly get_probability's
// tree over the selected ones (0 + x == x), so each q is one masked tree:
//  * q < 3: the masking happens inside the thread's 8 values (levels 0..3);
//  * 3 <= q < 11: the thread's level-3 node is kept or zeroed by a thread-id bit;
//  * the chunk total (q >= 11 and the norm) is the unmasked tree.
// The 12 per-thread values go through a transpose-reduce butterfly (each
// step halves the values a lane keeps: 8+4+2+1+1 shuffles instead of 12x5),
// whose pairings are the tree's, then a tree over the 8 warps.
__global__ void __launch_bounds__(kThreads)
    k_marginals(const double2* __restrict__ psi, int m, uint64_t total_chunks,
                double* __restrict__ low_out, double* __restrict__ high_out) {
    __shared__ double wsum[16][kThreads / 32];
    // |psi|^2 of the chunk, loaded coalesced, one pad double per 8 so that
    // thread t's 8 consecutive values read without bank conflicts
    __shared__ double sq[(1 << kMargChunkLog2) + (1 << kMargChunkLog2) / 8];
    const uint64_t cps = uint64_t(1) << (m - kMargChunkLog2);  // chunks per state
    const int nlow = kMargChunkLog2;                           // q < 11
    const int nhigh = m - kMargChunkLog2;                      // 11 <= q < m
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint64_t c = blockIdx.x; c < total_chunks; c += gridDim.x) {
        const uint64_t st = c / cps, cl = c - st * cps;
        const double2* src = psi + (st << m) + (cl << kMargChunkLog2);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int e = tid + j * kThreads;
            sq[e + (e >> 3)] = abs2(src[e]);
        }
        __syncthreads();
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = sq[9 * tid + j];
        const double l1[4] = {__dadd_rn(v[0], v[1]), __dadd_rn(v[2], v[3]),
                              __dadd_rn(v[4], v[5]), __dadd_rn(v[6], v[7])};
        const double l2[2] = {__dadd_rn(l1[0], l1[1]), __dadd_rn(l1[2], l1[3])};
        const double l3 = __dadd_rn(l2[0], l2[1]);
        double x[16];
        x[0] = __dadd_rn(__dadd_rn(v[1], v[3]), __dadd_rn(v[5], v[7]));  // q = 0
        x[1] = __dadd_rn(l1[1], l1[3]);                                   // q = 1
        x[2] = l2[1];                                                     // q = 2
#pragma unroll
        for (int q = 3; q < 11; ++q) x[q] = ((tid >> (q - 3)) & 1) ? l3 : 0.0;
        x[11] = l3;                                                       // total
#pragma unroll
        for (int q = 12; q < 16; ++q) x[q] = 0.0;
        // transpose-reduce: after step s a lane keeps 8 >> s values
#pragma unroll
        for (int s = 0, n = 16; s < 4; ++s, n >>= 1) {
            const bool up = (lane >> s) & 1;
#pragma unroll
            for (int i = 0; i < n / 2; ++i) {
                const double keep = up ? x[i + n / 2] : x[i];
                const double give = up ? x[i] : x[i + n / 2];
                x[i] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, give, 1 << s));
            }
        }
        x[0] = __dadd_rn(x[0], __shfl_xor_sync(0xffffffffu, x[0], 16));
        // lane l (< 16) now holds the warp sum of slot bitrev4(l)
        if (lane < 16) {
            const int slot = ((lane & 1) << 3) | ((lane & 2) << 1) | ((lane & 4) >> 1) |
                             ((lane & 8) >> 3);
            wsum[slot][warp] = x[0];
        }
        __syncthreads();
        if (tid < 12) {
            const double* w = wsum[tid];
            const double b = __dadd_rn(__dadd_rn(__dadd_rn(w[0], w[1]), __dadd_rn(w[2], w[3])),
                                       __dadd_rn(__dadd_rn(w[4], w[5]), __dadd_rn(w[6], w[7])));
            if (tid < nlow) {
                low_out[(st * nlow + tid) * cps + cl] = b;
            } else {
                for (int h = 0; h < nhigh; ++h)  // q = 11 + h: the chunk if its bit h is set
                    if ((cl >> h) & 1) {
                        const uint64_t idx =
                            ((cl >> (h + 1)) << h) | (cl & ((uint64_t(1) << h) - 1));
                        high_out[(st * nhigh + h) * (cps >> 1) + idx] = b;
                    }
            }
        }
        __syncthreads();
    }
}

inline unsigned grid_cap(uint64_t n) {
    uint64_t cap = 148ull * 16;
    return unsigned(n < cap ? (n ? n : 1) : cap);
}

}  // namespace

uint64_t reduce_scratch_doubles(int m, int num_states) {
    uint64_t per_state = uint64_t(1) << m;
    uint64_t first = (per_state + kChunk - 1) / kChunk;
    return 2 * (first * uint64_t(num_states) + 1);
}

// Reduce `lists` lists of `len` partials (power of two, contiguous) to one value
// each, with the same tree: level after level of k_tree over partials.
void tree_lists(const double* src, double* scratch_a, double* scratch_b, uint64_t len,
                uint64_t lists, double* out, cudaStream_t s) {
    CutTerms ct;
    ct.count = 0;
    const double* cur = src;
    int level = 0;
    while (true) {
        int lg = 0;
        while ((uint64_t(1) << lg) < len) ++lg;
        const bool wide = lg >= kWideLog2;
        const int chunk_log2 = wide ? kWideLog2 : lg;
        const uint64_t per = len >> chunk_log2;
        const uint64_t total = per * lists;
        double* dst = per == 1 ? out : (level & 1 ? scratch_b : scratch_a);
        if (wide)
            k_tree_wide<<<grid_cap(total), kThreads, 0, s>>>(nullptr, cur, dst, 0, 0, 0, 0, ct, len,
                                                             total);
        else
            k_tree<<<grid_cap(total), kThreads, 0, s>>>(nullptr, cur, dst, 0, 0, 0, 0, ct, len,
                                                        chunk_log2, total);
        if (per == 1) break;
        cur = dst;
        len = per;
        ++level;
    }
}

uint64_t marginal_scratch_doubles(int m, int num_states) {
    const uint64_t cps = uint64_t(1) << (m - kMargChunkLog2);
    const uint64_t partials = uint64_t(num_states) * uint64_t(m) * cps;
    return 3 * partials + 2 * uint64_t(num_states) * m + 16;
}

// out_dev: [num_states][m] marginals of the local qubits (m >= 12)
void launch_marginals(const double2* psi, int m, int num_states, double* scratch, double* out_dev,
                      cudaStream_t s) {
    const uint64_t cps = uint64_t(1) << (m - kMargChunkLog2);
    const int nlow = kMargChunkLog2, nhigh = m - kMargChunkLog2;
    const uint64_t S = uint64_t(num_states);
    double* low = scratch;                                     // [S][11][cps]
    double* high = low + S * nlow * cps;                       // [S][nhigh][cps/2]
    double* sa = high + S * nhigh * (cps >> 1) + 8;
    double* sb = sa + S * uint64_t(m) * cps;
    double* low_res = out_dev;                                 // [S][11] then [S][nhigh]
    double* high_res = out_dev + S * nlow;
    const uint64_t total = S * cps;
    k_marginals<<<grid_cap(total), kThreads, 0, s>>>(psi, m, total, low, high);
    tree_lists(low, sa, sb, cps, S * nlow, low_res, s);
    if (nhigh > 0) tree_lists(high, sa, sb, cps >> 1, S * nhigh, high_res, s);
}

void launch_observable(const double2* psi, int m, int num_states, int kind, int q,
                       uint64_t rank_offset, const CutTerms& ct, double* scratch, double* out_dev,
                       cudaStream_t s) {
    uint64_t elems = uint64_t(1) << m;
    if (kind == QS_OBS_PROB) elems >>= 1;
    const uint64_t half_scratch = reduce_scratch_doubles(m, num_states) / 2;
    double* bufs[2] = {scratch, scratch + half_scratch};
    int level = 0;
    const double* src = nullptr;
    const double2* state = psi;
    while (true) {
        int lg = 0;
        while ((uint64_t(1) << lg) < elems) ++lg;
        const bool wide = lg >= kWideLog2;
        int chunk_log2 = wide ? kWideLog2 : lg;
        uint64_t chunks_per_state = elems >> chunk_log2;
        uint64_t total = chunks_per_state * uint64_t(num_states);
        double* dst = chunks_per_state == 1 ? out_dev : bufs[level & 1];
        if (wide)
            k_tree_wide<<<grid_cap(total), kThreads, 0, s>>>(state, src, dst, m, kind, q,
                                                             rank_offset, ct, elems, total);
        else
            k_tree<<<grid_cap(total), kThreads, 0, s>>>(state, src, dst, m, kind, q, rank_offset,
                                                        ct, elems, chunk_log2, total);
        if (chunks_per_state == 1) break;
        src = dst;
        state = nullptr;
        elems = chunks_per_state;
        ++level;
    }
}

// ---- numerics diagnostics: distance between two states ----------------------
// out[0] = max_i |a_i - b_i|, out[1] = sum |a_i - b_i|^2, out[2] = sum |b_i|^2,
// out[3] = max_i |b_i| (diagnostic association: atomics, not the tree order).
__global__ void __launch_bounds__(256)
    k_state_diff(const double2* __restrict__ a, const double2* __restrict__ b, uint64_t count,
                 unsigned long long* __restrict__ maxbits, double* __restrict__ sums) {
    double mx = 0.0, mb = 0.0, sd = 0.0, sb = 0.0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double2 x = a[i], y = b[i];
        const double dr = x.x - y.x, di = x.y - y.y;
        const double d2 = dr * dr + di * di, b2 = y.x * y.x + y.y * y.y;
        mx = fmax(mx, d2);
        mb = fmax(mb, b2);
        sd += d2;
        sb += b2;
    }
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mb = fmax(mb, __shfl_xor_sync(0xffffffffu, mb, o));
        sd += __shfl_xor_sync(0xffffffffu, sd, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if ((threadIdx.x & 31) == 0) {
        // non-negative doubles order like their bit patterns
        atomicMax(maxbits + 0, __double_as_longlong(sqrt(mx)));
        atomicMax(maxbits + 1, __double_as_longlong(sqrt(mb)));
        atomicAdd(sums + 0, sd);
        atomicAdd(sums + 1, sb);
    }
}

void launch_state_diff(const double2* a, const double2* b, uint64_t count, void* scratch32,
                       cudaStream_t s) {
    cudaMemsetAsync(scratch32, 0, 32, s);
    unsigned long long* mb = reinterpret_cast<unsigned long long*>(scratch32);
    double* sums = reinterpret_cast<double*>(mb + 2);
    const unsigned grid = unsigned(std::min<uint64_t>((count + 255) / 256, 148 * 8));
    k_state_diff<<<grid, 256, 0, s>>>(a, b, count, mb, sums);
}

}  // namespace qsb
