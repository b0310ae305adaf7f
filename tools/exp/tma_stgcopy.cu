// Ceiling of the k_fact_tma data movement with G groups per CTA, one 2^12
// tile slot per group (the in-place design): a group waits for its TMA tile,
// reads it from shared memory into registers (16 amplitudes per thread),
// then requests its next tile into the same slot and stores the registers to
// HBM with STG in 128-byte rows (a quarter warp per row).  No arithmetic.
// Prints ms and GB/s (32 B per amplitude) per (tile shape, G, threads/group).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
struct alignas(64) Map { CUtensorMap m; int nc; int cd[4]; int cs[4]; unsigned long long cm[4]; int lo; };

static const int m = 30;

__device__ __forceinline__ void wait_bar(uint64_t* bar, unsigned par) {
    unsigned b = (unsigned)__cvta_generic_to_shared(bar), done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(b), "r"(par) : "memory");
}

// tile = qubits 0..2 + [lo, lo+9); amplitude e of the tile (e = q0..2 | t << 3)
// sits at smem double2 index sw(e) = e ^ ((e >> 3) & 7) (SWIZZLE_128B, 128-B rows)
template <int AMPS>
__global__ void __launch_bounds__(512, 1) k_copy(const __grid_constant__ Map M, double2* psi,
                                                 unsigned long long ntiles, int G, int TPG) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[4];
    const int g = threadIdx.x / TPG, tid = threadIdx.x % TPG;
    if (threadIdx.x < G) {
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar[threadIdx.x]);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncthreads();
    auto load = [&](unsigned long long t, int s) {
        int c[5] = {0, 0, 0, 0, 0};
        for (int i = 0; i < M.nc; ++i) c[M.cd[i]] = int((t >> M.cs[i]) & M.cm[i]);
        unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
        unsigned d = (unsigned)__cvta_generic_to_shared(smem + (size_t)s * 65536);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(65536));
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d), "l"(&M.m), "r"(c[0]), "r"(c[1]),
                     "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b) : "memory");
    };
    if (g >= G) return;
    const unsigned long long step = (unsigned long long)gridDim.x * G;
    unsigned long long t = (unsigned long long)blockIdx.x * G + g;
    if (tid == 0 && t < ntiles) load(t, g);
    const double2* L = reinterpret_cast<const double2*>(smem + (size_t)g * 65536);
    unsigned par = 0;
    for (; t < ntiles; t += step, par ^= 1) {
        wait_bar(&bar[g], par);
        double2 a[AMPS];
        // thread owns tile rows tid, tid + TPG, ...: lanes 0..7 of a quarter
        // warp take the 8 chunks of one 128-B row
#pragma unroll
        for (int k = 0; k < AMPS; ++k) {
            const int e = (tid + k * TPG);
            a[k] = L[e ^ ((e >> 3) & 7)];
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(TPG) : "memory");
        const unsigned long long nt = t + step;
        if (tid == 0 && nt < ntiles) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            load(nt, g);
        }
        // HBM offset of tile t: non-tile bits are qubits 3..lo-1 and lo+9..m-1
        const unsigned long long below = t & ((1ull << (M.lo - 3)) - 1), above = t >> (M.lo - 3);
        const unsigned long long base = (below << 3) | (above << (M.lo + 9));
#pragma unroll
        for (int k = 0; k < AMPS; ++k) {
            const int e = tid + k * TPG;
            psi[base | (e & 7) | ((unsigned long long)(e >> 3) << M.lo)] = a[k];
        }
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
    cudaFuncSetAttribute(k_copy<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536);
    cudaFuncSetAttribute(k_copy<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int lo : {3, 12, 21}) {
        Map M;
        cuuint64_t dim[5], str[4];
        cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
        int r = 0;
        dim[r] = 16, box[r] = 16, ++r;
        if (lo == 3) {
            dim[r] = 512, str[r - 1] = 128, box[r] = 256, ++r;  // q3..q10 (8) + q11 as 2 dims
            dim[r - 1] = 256, box[r - 1] = 256;
            dim[r] = 2, str[r - 1] = 128ull << 8, box[r] = 2, ++r;
        } else {
            dim[r] = 256, str[r - 1] = 16ull << lo, box[r] = 256, ++r;
            dim[r] = 2, str[r - 1] = 16ull << (lo + 8), box[r] = 2, ++r;
        }
        M.nc = 0;
        M.lo = lo;
        const int below = lo - 3, above = m - lo - 9;
        if (below > 0) {
            dim[r] = 1ull << below, str[r - 1] = 128, box[r] = 1;
            M.cd[M.nc] = r, M.cs[M.nc] = 0, M.cm[M.nc] = (1ull << below) - 1, ++M.nc, ++r;
        }
        if (above > 0) {
            dim[r] = 1ull << above, str[r - 1] = 16ull << (lo + 9), box[r] = 1;
            M.cd[M.nc] = r, M.cs[M.nc] = below, M.cm[M.nc] = ~0ull, ++M.nc, ++r;
        }
        while (r < 5) dim[r] = 1, str[r - 1] = str[r - 2] * 2, box[r] = 1, ++r;
        CUresult rc = enc(&M.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, dbuf, dim, str, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (rc != CUDA_SUCCESS) { printf("encode failed lo=%d\n", lo); continue; }
        const int cfg[][2] = {{1, 256}, {2, 256}, {1, 128}, {2, 128}, {3, 128}};
        for (auto& c : cfg) {
            const int G = c[0], TPG = c[1];
            const unsigned long long nt = N >> 12;
            auto run = [&]() {
                if (TPG == 256) k_copy<16><<<sms, G * TPG, G * 65536>>>(M, dbuf, nt, G, TPG);
                else k_copy<32><<<sms, G * TPG, G * 65536>>>(M, dbuf, nt, G, TPG);
            };
            run();
            cudaEventRecord(e0);
            for (int it = 0; it < 3; ++it) run();
            cudaEventRecord(e1);
            cudaError_t e = cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            ms /= 3;
            printf("lo=%2d G=%d threads/group=%d  %.3f ms  %.0f GB/s  %s\n", lo, G, TPG, ms,
                   32.0 * N / (ms * 1e6), cudaGetErrorString(e));
        }
    }
    return 0;
}
