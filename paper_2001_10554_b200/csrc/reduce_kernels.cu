// Observable reductions in the reference's exact association.
//
// The reference sums every observable with tree_sum (statevector.py:29-45): a
// perfect binary tree over element order (x.reshape(-1,2).sum(axis=1) until one
// value).  Here each block reduces an aligned 2^L-element chunk with the same
// pairing (a pairwise tree in shared memory), writes one partial, and the
// partials are reduced again with the same kernel until one value per state
// remains -- exactly the reference's tree, level by level, so the result is
// bit-identical for any chunking.
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
    for (uint64_t c = blockIdx.x; c < total_chunks; c += gridDim.x) {
        const uint64_t s = c / chunks_per_state;
        const uint64_t first = ((c - s * chunks_per_state) << kWideLog2) + warp * 256 + lane;
        double v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint64_t j = first + i * 32;
            v[i] = psi ? obs_value(psi, m, kind, q, rank_offset, ct, s, j)
                       : src[s * elems_per_state + j];
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

}  // namespace qsb
