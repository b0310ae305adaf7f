// 2^13-amplitude tiles (rows of 256 B = qubits 0..3, plus 9 targets at
// [lo, lo+9)) moved by one CTA of 512 threads per SM: TMA load of the 128 KiB
// box into shared memory, every thread reads 16 amplitudes into registers,
// the next tile is requested, then the registers are stored with STG.
// mapping 0 ("rows"): lanes 0..7 cover qubits 0..2 (128-B rows per quarter
// warp, 256 B per half warp) -- the coalesced store; mapping 1 ("warp
// chunks"): warp w = qubits 0..3, lanes and registers = the 9 targets (what a
// register-resident tile with warp-local reslices would store: 16 B of each of
// 32 rows per instruction).  Prints ms and GB/s (32 B per amplitude).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
struct alignas(64) Map { CUtensorMap m; int nc; int cd[4]; int cs[4]; int lsh[4]; unsigned long long cm[4]; int lo; };
static const int m = 30;

template <int MAP>
__global__ void __launch_bounds__(512, 1) k_copy(const __grid_constant__ Map M, double2* psi,
                                                 unsigned long long ntiles) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto load = [&](unsigned long long t) {
        int c[5] = {0, 0, 0, 0, 0};
        for (int i = 0; i < M.nc; ++i) c[M.cd[i]] = int(((t >> M.cs[i]) & M.cm[i]) << M.lsh[i]);
        unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
        unsigned d = (unsigned)__cvta_generic_to_shared(smem);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(131072));
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d), "l"(&M.m), "r"(c[0]), "r"(c[1]),
                     "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b) : "memory");
    };
    unsigned long long t = blockIdx.x;
    if (tid == 0 && t < ntiles) load(t);
    const double2* L = reinterpret_cast<const double2*>(smem);
    unsigned par = 0;
    for (; t < ntiles; t += gridDim.x, par ^= 1) {
        {
            unsigned b = (unsigned)__cvta_generic_to_shared(&bar), done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(b), "r"(par) : "memory");
        }
        double2 a[16];
        int e[16];  // tile element: bits 0..3 = qubits 0..3, bits 4..12 = targets
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            e[k] = MAP == 0 ? tid + 512 * k : (w | (lane << 4) | (k << 9));
            a[k] = L[e[k] ^ ((e[k] >> 3) & 7)];
        }
        __syncthreads();
        const unsigned long long nt = t + gridDim.x;
        if (tid == 0 && nt < ntiles) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            load(nt);
        }
        const unsigned long long below = t & ((1ull << (M.lo - 4)) - 1), above = t >> (M.lo - 4);
        const unsigned long long base = (below << 4) | (above << (M.lo + 9));
#pragma unroll
        for (int k = 0; k < 16; ++k)
            psi[base | (e[k] & 15) | ((unsigned long long)(e[k] >> 4) << M.lo)] = a[k];
    }
}

int main() {
    const size_t N = size_t(1) << m;
    double2* dbuf;
    if (cudaMalloc(&dbuf, N * 16) != cudaSuccess) return 1;
    cudaMemset(dbuf, 0, N * 16);
    EncodeFn enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_copy<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    cudaFuncSetAttribute(k_copy<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int lo : {12, 21}) {
        Map M;
        cuuint64_t dim[5], str[4];
        cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
        int r = 0;
        dim[r] = 16, box[r] = 16, ++r;                                   // q0..2
        dim[r] = 2, str[r - 1] = 128, box[r] = 2, ++r;                   // q3
        dim[r] = 256, str[r - 1] = 16ull << lo, box[r] = 256, ++r;       // t0..7
        const int above = m - lo - 9, below = lo - 4;
        // t8 rides with the qubits above it (extent 2 * 2^above, box 2)
        dim[r] = 2ull << above, str[r - 1] = 16ull << (lo + 8), box[r] = 2, ++r;
        M.nc = 0;
        M.lo = lo;
        M.cd[M.nc] = r - 1, M.cs[M.nc] = below, M.lsh[M.nc] = 1, M.cm[M.nc] = ~0ull, ++M.nc;
        dim[r] = 1ull << below, str[r - 1] = 16ull << 4, box[r] = 1;    // qubits 4..lo-1
        M.cd[M.nc] = r, M.cs[M.nc] = 0, M.lsh[M.nc] = 0, M.cm[M.nc] = (1ull << below) - 1, ++M.nc, ++r;
        CUresult rc = enc(&M.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, dbuf, dim, str, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (rc != CUDA_SUCCESS) { printf("encode failed lo=%d rc=%d\n", lo, (int)rc); continue; }
        // the t8/above dim's coordinate: 2 * (above bits of the tile index)
        // handled below by a second field (shift below, value << 1)
        for (int map = 0; map < 2; ++map) {
            const unsigned long long nt = N >> 13;
            auto run = [&]() {
                if (map == 0) k_copy<0><<<sms, 512, 131072>>>(M, dbuf, nt);
                else k_copy<1><<<sms, 512, 131072>>>(M, dbuf, nt);
            };
            run();
            cudaEventRecord(e0);
            for (int it = 0; it < 3; ++it) run();
            cudaEventRecord(e1);
            cudaError_t e = cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            ms /= 3;
            printf("lo=%2d %s  %.3f ms  %.0f GB/s  %s\n", lo, map ? "warp-chunk stores" : "row stores       ",
                   ms, 32.0 * N / (ms * 1e6), cudaGetErrorString(e));
        }
    }
    return 0;
}
