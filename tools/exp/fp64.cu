// FP64 pipe throughput probe: independent DFMA / DMUL / DADD chains.
#include <cstdio>
template <int OP>
__global__ void k(double* out, int iters, double x) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = x + threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) a[i] = __fma_rn(a[i], 0.999999, 1e-9);
            if (OP == 1) a[i] = __dmul_rn(a[i], 0.999999);
            if (OP == 2) a[i] = __dadd_rn(a[i], 1e-9);
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double* d;
    int blocks = 148 * 8, threads = 256, iters = 4096;
    cudaMalloc(&d, sizeof(double) * blocks * threads);
    const char* names[] = {"DFMA", "DMUL", "DADD"};
    for (int op = 0; op < 3; ++op) {
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (op == 0) k<0><<<blocks, threads>>>(d, iters, 1.0);
            if (op == 1) k<1><<<blocks, threads>>>(d, iters, 1.0);
            if (op == 2) k<2><<<blocks, threads>>>(d, iters, 1.0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = double(blocks) * threads * iters * 8;
        int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("%s: %.3f ms, %.2f Tops/s, %.2f thread-ops/clk/SM at %d MHz\n", names[op], ms,
               ops / ms / 1e9, ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
    }
    return 0;
}
