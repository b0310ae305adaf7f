// FP64 throughput with register operands: the pair_update pattern.
#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ double2 cmul(double2 x, double2 y) {
    return make_double2(__fma_rn(x.x, y.x, -__dmul_rn(x.y, y.y)), __fma_rn(x.x, y.y, __dmul_rn(x.y, y.x)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
template <int NP>
__global__ void kpair(double2* out, const double2* um, int iters) {
    double2 u[4];
    for (int i = 0; i < 4; ++i) u[i] = um[i];
    double2 a[2 * NP];
    for (int i = 0; i < 2 * NP; ++i) a[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            double2 x = a[2 * p], y = a[2 * p + 1];
            a[2 * p] = cadd(cmul(u[0], x), cmul(u[1], y));
            a[2 * p + 1] = cadd(cmul(u[2], x), cmul(u[3], y));
        }
    }
    double2 s = make_double2(0, 0);
    for (int i = 0; i < 2 * NP; ++i) s = cadd(s, a[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void kfma_reg(double* out, const double* c, int iters) {
    double b = c[0], d = c[1];
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    double e[8];
    for (int i = 0; i < 8; ++i) e[i] = c[2 + i];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __fma_rn(a[i], b, e[i]);
    }
    double s = d;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double2* d; double2* um; double* c;
    int blocks = 148 * 4, threads = 256, iters = 2048;
    if (getenv("BLOCKS")) blocks = atoi(getenv("BLOCKS"));
    if (getenv("THREADS")) threads = atoi(getenv("THREADS"));
    cudaMalloc(&d, sizeof(double2) * blocks * threads);
    cudaMalloc(&um, 4 * sizeof(double2));
    cudaMalloc(&c, 16 * sizeof(double));
    double2 hu[4] = {{0.6, 0.1}, {0.2, -0.3}, {-0.1, 0.4}, {0.5, 0.2}};
    cudaMemcpy(um, hu, sizeof(hu), cudaMemcpyHostToDevice);
    double hc[16]; for (int i = 0; i < 16; ++i) hc[i] = 0.999 + i * 1e-6;
    cudaMemcpy(c, hc, sizeof(hc), cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float ms;
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(a); kpair<4><<<blocks, threads>>>(d, um, iters); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b);
    double ops = double(blocks) * threads * iters * 4 * 20;
    printf("pair_update x4: %.3f ms  %.2f fp64 thread-ops/clk/SM\n", ms, ops / (ms * 1e-3) / 148 / (clk * 1e3));
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(a); kpair<8><<<blocks, threads>>>(d, um, iters); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b);
    ops = double(blocks) * threads * iters * 8 * 20;
    printf("pair_update x8: %.3f ms  %.2f fp64 thread-ops/clk/SM\n", ms, ops / (ms * 1e-3) / 148 / (clk * 1e3));
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(a); kfma_reg<<<blocks, threads>>>((double*)d, c, iters * 4); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b);
    ops = double(blocks) * threads * iters * 4 * 8;
    printf("DFMA 3-reg: %.3f ms  %.2f fp64 thread-ops/clk/SM\n", ms, ops / (ms * 1e-3) / 148 / (clk * 1e3));
    return 0;
}
