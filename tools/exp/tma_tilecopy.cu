// Ceiling of tile-shaped data movement: every 2^12-amplitude tile of a
// 2^30-amplitude complex128 state, tile = qubits {0,1,2} + [lo, lo+8], is
// loaded by TMA into one of S shared-memory slots per CTA and stored back by
// TMA (in place), S tiles in flight per SM; one thread drives the pipeline.
// Prints GB/s (read + write, 32 B per amplitude) per (lo, S).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
struct alignas(64) Map { CUtensorMap m; int rank; int nc; int cd[4]; int cs[4]; unsigned long long cm[4]; };

__device__ __forceinline__ void coords(const Map& M, unsigned long long t, int* c) {
    for (int i = 0; i < 5; ++i) c[i] = 0;
    for (int i = 0; i < M.nc; ++i) c[M.cd[i]] = int((t >> M.cs[i]) & M.cm[i]);
}

__global__ void __launch_bounds__(32, 1) k_copy(const __grid_constant__ Map M, const __grid_constant__ Map MS, unsigned long long ntiles, int S) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[8];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < S; ++s) {
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    auto load = [&](unsigned long long t, int s) {
        int c[5];
        coords(M, t, c);
        unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
        unsigned d = (unsigned)__cvta_generic_to_shared(smem + (size_t)s * 65536);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(65536));
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d), "l"(&M.m), "r"(c[0]), "r"(c[1]),
                     "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b) : "memory");
    };
    auto store = [&](unsigned long long t, int s) {
        int c[5];
        coords(MS, t, c);
        unsigned d = (unsigned)__cvta_generic_to_shared(smem + (size_t)s * 65536);
        asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                     ::"l"(&MS.m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(d) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
    };
    const unsigned long long first = blockIdx.x, step = gridDim.x;
    int k = 0;
    for (int s = 0; s < S; ++s)
        if (first + s * step < ntiles) load(first + s * step, s);
    for (unsigned long long t = first; t < ntiles; t += step, ++k) {
        const int s = k % S;
        const unsigned par = (k / S) & 1;
        unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(b), "r"(par));
        store(t, s);
        const unsigned long long nt = t + (unsigned long long)S * step;
        if (nt < ntiles) {
            // the slot is reusable once the store has read it
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            load(nt, s);
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static EncodeFn enc = nullptr;
static double2* dbuf = nullptr;
static const int m = 30;

// tile = qubits {0..low-1} + [lo, lo + 12 - low), rows of 2^low amplitudes
static bool make_map(Map& M, int lo, int low) {
    cuuint64_t dim[5], str[4];
    cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
    int r = 0;
    const int k = 12 - low;  // target bits
    dim[r] = 2u << 3, box[r] = 16, ++r;                              // q0..2
    if (low > 3) dim[r] = 1u << (low - 3), str[r - 1] = 16ull << 3, box[r] = 1u << (low - 3), ++r;
    int a = k > 8 ? 8 : k;
    dim[r] = 1ull << a, str[r - 1] = 16ull << lo, box[r] = 1u << a, ++r;
    if (k > 8) dim[r] = 1ull << (k - 8), str[r - 1] = 16ull << (lo + 8), box[r] = 1u << (k - 8), ++r;
    M.nc = 0;
    int below = lo - low;
    if (below > 0) {
        dim[r] = 1ull << below, str[r - 1] = 16ull << low, box[r] = 1;
        M.cd[M.nc] = r, M.cs[M.nc] = 0, M.cm[M.nc] = (1ull << below) - 1, ++M.nc, ++r;
    }
    int above = m - (lo + k);
    if (above > 0) {
        dim[r] = 1ull << above, str[r - 1] = 16ull << (lo + k), box[r] = 1;
        M.cd[M.nc] = r, M.cs[M.nc] = below, M.cm[M.nc] = ~0ull, ++M.nc, ++r;
    }
    if (r > 5) return false;
    while (r < 5) dim[r] = 1, str[r - 1] = str[r - 2] * 2, box[r] = 1, ++r;
    M.rank = 5;
    return enc(&M.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, dbuf, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int main(int argc, char** argv) {
    const size_t N = size_t(1) << m;
    if (cudaMalloc(&dbuf, N * 16) != cudaSuccess) return 1;
    cudaMemset(dbuf, 0, N * 16);
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // (load lo, load low, store lo, store low)
    const int cases[][4] = {{3, 3, 3, 3}, {21, 3, 21, 3}, {3, 3, 21, 3}, {21, 3, 3, 3}, {12, 3, 12, 3},
                            {3, 3, 12, 3}, {12, 3, 3, 3}, {22, 4, 22, 4}, {23, 5, 23, 5}, {13, 4, 13, 4},
                            {9, 3, 9, 3}, {6, 3, 6, 3}};
    for (auto& c : cases) {
        Map ML, MS;
        if (!make_map(ML, c[0], c[1]) || !make_map(MS, c[2], c[3])) { printf("map failed\n"); continue; }
        const int S = 2;
        const unsigned long long nt = N >> 12;
        k_copy<<<sms, 32, S * 65536>>>(ML, MS, nt, S);
        cudaEventRecord(e0);
        for (int it = 0; it < 3; ++it) k_copy<<<sms, 32, S * 65536>>>(ML, MS, nt, S);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 3;
        printf("load lo=%2d low=%d  store lo=%2d low=%d  %.3f ms  %.0f GB/s  %s\n", c[0], c[1], c[2], c[3], ms,
               32.0 * N / (ms * 1e6), cudaGetErrorString(e));
    }
    return 0;
}
