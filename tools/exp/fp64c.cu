// Compute-section probe: the tile kernel's register rounds without memory traffic.
#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ double2 cmul(double2 x, double2 y) {
    return make_double2(__fma_rn(x.x, y.x, -__dmul_rn(x.y, y.y)), __fma_rn(x.x, y.y, __dmul_rn(x.y, y.x)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ void pair_update(double2& a, double2& b, const double2 u[4]) {
    double2 na = cadd(cmul(u[0], a), cmul(u[1], b));
    double2 nb = cadd(cmul(u[2], a), cmul(u[3], b));
    a = na; b = nb;
}
template <int J>
__device__ __forceinline__ void reg_gate(double2 (&a)[16], const double2 u[4]) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if ((k >> J) & 1) continue;
        pair_update(a[k], a[k | (1 << J)], u);
    }
}
template <int MODE>
__global__ void __launch_bounds__(256) kround(double2* out, const double2* um, int iters) {
    __shared__ double2 us[16];
    if (threadIdx.x < 16) us[threadIdx.x] = um[threadIdx.x];
    __syncthreads();
    double2 a[16];
    for (int i = 0; i < 16; ++i) a[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
    double2 ureg[4];
    for (int q = 0; q < 4; ++q) ureg[q] = us[q];
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {  // u from shared memory per gate
            double2 u[4];
            for (int q = 0; q < 4; ++q) u[q] = us[q];
            reg_gate<0>(a, u);
            for (int q = 0; q < 4; ++q) u[q] = us[4 + q];
            reg_gate<1>(a, u);
            for (int q = 0; q < 4; ++q) u[q] = us[8 + q];
            reg_gate<2>(a, u);
            for (int q = 0; q < 4; ++q) u[q] = us[12 + q];
            reg_gate<3>(a, u);
        } else if (MODE == 2) {  // u per gate from smem at a thread-dependent (but equal) address
            double2 u[4];
            const int z = (threadIdx.x >> 10);  // 0 for all threads, unknown to the compiler
            for (int q = 0; q < 4; ++q) u[q] = us[(q + it) % 4 + z];
            reg_gate<0>(a, u);
            for (int q = 0; q < 4; ++q) u[q] = us[(4 + q + it) % 16 + z];
            reg_gate<1>(a, u);
            for (int q = 0; q < 4; ++q) u[q] = us[(8 + q + it) % 16 + z];
            reg_gate<2>(a, u);
            for (int q = 0; q < 4; ++q) u[q] = us[(12 + q + it) % 16 + z];
            reg_gate<3>(a, u);
        } else if (MODE == 3) {  // u per gate from smem, uniform address, varying per iteration
            double2 u[4];
            for (int q = 0; q < 4; ++q) u[q] = us[(q + it) % 16];
            reg_gate<0>(a, u);
            for (int q = 0; q < 4; ++q) u[q] = us[(4 + q + it) % 16];
            reg_gate<1>(a, u);
            for (int q = 0; q < 4; ++q) u[q] = us[(8 + q + it) % 16];
            reg_gate<2>(a, u);
            for (int q = 0; q < 4; ++q) u[q] = us[(12 + q + it) % 16];
            reg_gate<3>(a, u);
        } else {  // u in registers
            reg_gate<0>(a, ureg);
            reg_gate<1>(a, ureg);
            reg_gate<2>(a, ureg);
            reg_gate<3>(a, ureg);
        }
    }
    double2 s = make_double2(0, 0);
    for (int i = 0; i < 16; ++i) s = cadd(s, a[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double2* d; double2* um;
    int blocks = atoi(getenv("BLOCKS") ? getenv("BLOCKS") : "296"), threads = 256, iters = 256;
    cudaMalloc(&d, sizeof(double2) * blocks * threads);
    cudaMalloc(&um, 16 * sizeof(double2));
    double2 hu[16]; for (int i = 0; i < 16; ++i) hu[i] = make_double2(0.3 + 0.01 * i, 0.1 - 0.02 * i);
    cudaMemcpy(um, hu, sizeof(hu), cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float ms;
    double ops = double(blocks) * threads * iters * 4 * 8 * 20;
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(a); kround<0><<<blocks, threads>>>(d, um, iters); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b);
    printf("blocks %d: u from smem: %.3f ms %.2f fp64 thread-ops/clk/SM\n", blocks, ms, ops / (ms * 1e-3) / 148 / (clk * 1e3));
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(a); kround<1><<<blocks, threads>>>(d, um, iters); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b);
    printf("blocks %d: u in regs:  %.3f ms %.2f fp64 thread-ops/clk/SM\n", blocks, ms, ops / (ms * 1e-3) / 148 / (clk * 1e3));
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(a); kround<2><<<blocks, threads>>>(d, um, iters); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b);
    printf("blocks %d: u varying non-uniform regs:  %.3f ms %.2f fp64 thread-ops/clk/SM\n", blocks, ms, ops / (ms * 1e-3) / 148 / (clk * 1e3));
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(a); kround<3><<<blocks, threads>>>(d, um, iters); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b);
    printf("blocks %d: u varying uniform:  %.3f ms %.2f fp64 thread-ops/clk/SM\n", blocks, ms, ops / (ms * 1e-3) / 148 / (clk * 1e3));
    return 0;
}
