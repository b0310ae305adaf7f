#include <cstdio>
#include <cstdint>
struct Big { int32_t a[3000]; };
__global__ void k(const __grid_constant__ Big b, int* out) {
    out[threadIdx.x] = b.a[threadIdx.x * 11 % 3000] + b.a[2999];
}
int main() {
    static Big b; for (int i = 0; i < 3000; ++i) b.a[i] = i;
    int* d; cudaMalloc(&d, 256 * 4);
    k<<<1, 256>>>(b, d);
    cudaError_t e = cudaDeviceSynchronize();
    int h[256]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("err=%s h[1]=%d (expect %d) h[255]=%d (expect %d)\n", cudaGetErrorString(e), h[1], 11 + 2999, h[255], 255*11%3000 + 2999);
    return 0;
}
