// Host<->device copy variants for the e2e path (pinned memory).
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const int rows = 4 * 8 * 375, W = 1242, P = 1248;
    size_t dense = size_t(rows) * W;
    unsigned char *h, *d; float ms;
    cudaMallocHost(&h, dense); cudaMalloc(&d, size_t(rows) * P);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        cudaMemcpy2DAsync(d, P, h, W, W, rows, cudaMemcpyHostToDevice, 0);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("memcpy2D H2D %d rows x %d B: %.3f ms (%.1f GB/s)\n", rows, W, ms, dense / ms / 1e6);
        cudaEventRecord(a);
        cudaMemcpyAsync(d, h, dense, cudaMemcpyHostToDevice, 0);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("memcpy 1D H2D %zu B: %.3f ms (%.1f GB/s)\n", dense, ms, dense / ms / 1e6);
    }
    return 0;
}
