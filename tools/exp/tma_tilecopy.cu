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

__global__ void __launch_bounds__(32, 1) k_copy(const __grid_constant__ Map M, const __grid_constant__ Map MS, const __grid_constant__ Map MP, unsigned long long ntiles, int S, int mode, unsigned slot) {
    // mode 3: pairs + an L2 prefetch of the PAIR box (MP: both tiles, 2x wider rows)
    // mode 0: CTA b takes tiles b, b+grid, ...; mode 1: CTA b takes tile pairs
    // (2p, 2p+1), p = b, b+grid, ... (the pair differs in the lowest non-tile
    // qubit: adjacent rows); mode 2: pairs + an L2 prefetch of the odd tile
    // issued with the even tile's load
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
        unsigned d = (unsigned)__cvta_generic_to_shared(smem + (size_t)s * slot);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(slot));
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d), "l"(&M.m), "r"(c[0]), "r"(c[1]),
                     "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b) : "memory");
    };
    auto store = [&](unsigned long long t, int s) {
        int c[5];
        coords(MS, t, c);
        unsigned d = (unsigned)__cvta_generic_to_shared(smem + (size_t)s * slot);
        asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                     ::"l"(&MS.m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(d) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
    };
    auto prefetch_map = [&](const Map& PM, unsigned long long t) {
        int c[5];
        coords(PM, t, c);
        asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];"
                     ::"l"(&PM.m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
    };
    auto prefetch = [&](unsigned long long t) { prefetch_map(M, t); };
    const unsigned long long first = blockIdx.x, step = gridDim.x;
    auto tile_of = [&](unsigned long long k) {
        return mode == 0 ? first + k * step : 2 * (first + (k >> 1) * step) + (k & 1);
    };
    auto load_k = [&](unsigned long long k, int s) {
        const unsigned long long t = tile_of(k);
        load(t, s);
        if (mode == 2 && !(k & 1) && t + 1 < ntiles) prefetch(t + 1);
        if (mode == 3 && !(k & 1)) prefetch_map(MP, t >> 1);
    };
    int k = 0;
    for (int s = 0; s < S; ++s)
        if (tile_of(s) < ntiles) load_k(s, s);
    for (unsigned long long t = tile_of(0); t < ntiles; ++k, t = tile_of(k)) {
        const int s = k % S;
        const unsigned par = (k / S) & 1;
        unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(b), "r"(par));
        store(t, s);
        const unsigned long long nt = tile_of(k + S);
        if (nt < ntiles) {
            // the slot is reusable once the store has read it
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            load_k(k + S, s);
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static EncodeFn enc = nullptr;
static double2* dbuf = nullptr;
static const int m = 30;

// tile = qubits {0..low-1} + [lo, lo + T - low), rows of 2^low amplitudes
static int T = 12;
static bool make_map(Map& M, int lo, int low) {
    cuuint64_t dim[8], str[8];
    cuuint32_t box[8], es[5] = {1, 1, 1, 1, 1};
    int r = 0;
    const int k = T - low;  // target bits
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
    if (argc > 1) {
        // big tiles: T=13 (128 KiB boxes, one slot), rows of 2^low amplitudes
        T = 13;
        const int big[][2] = {{3, 3}, {4, 4}, {12, 3}, {21, 4}, {21, 3}};
        for (int mode = 0; mode < 3; mode += 2)
            for (auto& c : big) {
                Map ML, MS;
                if (!make_map(ML, c[0], c[1]) || !make_map(MS, c[0], c[1])) { printf("map failed\n"); continue; }
                const unsigned long long nt = N >> T;
                k_copy<<<sms, 32, 131072>>>(ML, MS, ML, nt, 1, mode, 131072);
                cudaEventRecord(e0);
                for (int it = 0; it < 3; ++it) k_copy<<<sms, 32, 131072>>>(ML, MS, ML, nt, 1, mode, 131072);
                cudaEventRecord(e1);
                cudaError_t e = cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                ms /= 3;
                printf("T=13 mode=%d S=1 lo=%2d low=%d  %.3f ms  %.0f GB/s  %s\n", mode, c[0], c[1], ms,
                       32.0 * N / (ms * 1e6), cudaGetErrorString(e));
            }
        return 0;
    }
    // (load lo, load low, store lo, store low)
    const int cases[][4] = {{3, 3, 3, 3}, {21, 3, 21, 3}, {3, 3, 21, 3}, {21, 3, 3, 3}, {12, 3, 12, 3},
                            {3, 3, 12, 3}, {12, 3, 3, 3}, {22, 4, 22, 4}, {23, 5, 23, 5}, {13, 4, 13, 4},
                            {9, 3, 9, 3}, {6, 3, 6, 3}};
    for (int mode = 0; mode < 4; ++mode)
    for (int S = 1; S <= 3; ++S)
    for (auto& c : cases) {
        if ((S != 2 || mode) && c[0] != c[2]) continue;
        if (mode && c[1] != 3) continue;
        Map ML, MS, MP;
        if (mode == 3) {
            if (c[0] != 21 || S == 1) continue;
            T = 13;
            bool ok = make_map(MP, c[0], 4);
            T = 12;
            if (!ok) { printf("pair map failed\n"); continue; }
        }
        if (!make_map(ML, c[0], c[1]) || !make_map(MS, c[2], c[3])) { printf("map failed\n"); continue; }
        const unsigned long long nt = N >> 12;
        k_copy<<<sms, 32, S * 65536>>>(ML, MS, MP, nt, S, mode, 65536);
        cudaEventRecord(e0);
        for (int it = 0; it < 3; ++it) k_copy<<<sms, 32, S * 65536>>>(ML, MS, MP, nt, S, mode, 65536);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 3;
        printf("mode=%d S=%d load lo=%2d low=%d  store lo=%2d low=%d  %.3f ms  %.0f GB/s  %s\n", mode, S, c[0], c[1], c[2], c[3], ms,
               32.0 * N / (ms * 1e6), cudaGetErrorString(e));
    }
    return 0;
}
