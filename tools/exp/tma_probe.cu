// Probe: does cuTensorMapEncodeTiled accept non-monotone dim strides, and is
// the SWIZZLE_128B smem layout what the planner predicts?  A 2^16-amplitude
// complex128 array (value = index) is loaded as one 12-position tile:
// dim0 = re/im x qubits 0..2 (128 B rows), dim1 = qubits 6..8, dim2 = qubits
// 3..5, dim3 = qubits 9..11, dim4 = qubits 12..15 (box 1, coordinate 5).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap map, double2* out, int c4) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
    const unsigned sd = (unsigned)__cvta_generic_to_shared(smem);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(65536));
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sd),
            "l"(&map), "r"(0), "r"(0), "r"(0), "r"(0), "r"(c4), "r"(sb)
            : "memory");
    }
    unsigned done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(sb), "r"(0));
    const double2* t = reinterpret_cast<const double2*>(smem);
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = t[i];
}

int main() {
    const int n = 16;
    const size_t N = size_t(1) << n;
    std::vector<double2> h(N);
    for (size_t i = 0; i < N; ++i) h[i] = make_double2(double(i), -double(i));
    double2 *d, *o;
    cudaMalloc(&d, N * 16);
    cudaMalloc(&o, 4096 * 16);
    cudaMemcpy(d, h.data(), N * 16, cudaMemcpyHostToDevice);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no entry point\n"); return 1; }
    // dims: (elements) 16 doubles | q6..8 | q3..5 | q9..11 | q12..15
    cuuint64_t dim[5] = {16, 8, 8, 8, 16};
    cuuint64_t stride[4] = {uint64_t(16) << 6, uint64_t(16) << 3, uint64_t(16) << 9, uint64_t(16) << 12};
    cuuint32_t box[5] = {16, 8, 8, 8, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUtensorMap map;
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, d, dim, stride, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode (non-monotone strides): %d\n", int(r));
    if (r != CUDA_SUCCESS) return 2;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    k<<<1, 256, 65536 + 1024>>>(map, o, 5);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<double2> got(4096);
    cudaMemcpy(got.data(), o, 4096 * 16, cudaMemcpyDeviceToHost);
    // predicted: smem index s (16-B units) = sigma(tile element); tile element
    // bits: pos0..2 = q0..2, smem bits 3..5 = q6..8, 6..8 = q3..5, 9..11 = q9..11;
    // swizzle: s ^= (s >> 3) & 7
    int bad = 0;
    for (int s = 0; s < 4096; ++s) {
        const int lin = s ^ ((s >> 3) & 7);  // un-swizzle
        const int q02 = lin & 7, q68 = (lin >> 3) & 7, q35 = (lin >> 6) & 7, q911 = (lin >> 9) & 7;
        const size_t idx = size_t(q02) | (size_t(q35) << 3) | (size_t(q68) << 6) | (size_t(q911) << 9) |
                           (size_t(5) << 12);
        if (got[s].x != double(idx) || got[s].y != -double(idx)) {
            if (bad < 5) printf("s=%d got %g expected %zu\n", s, got[s].x, idx);
            ++bad;
        }
    }
    printf("layout mismatches: %d of 4096\n", bad);
    return bad ? 3 : 0;
}
