// Which register counts allow a 544-thread CTA on sm_100a? (cudaOccupancy query)
#include <cstdio>
#include <cuda_runtime.h>
template <int N> __global__ void __maxnreg__(N) k(float *o) {
    float a[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) a[i] = o[threadIdx.x * 64 + i];
    float s = 0;
#pragma unroll
    for (int r = 0; r < 50; ++r)
#pragma unroll
        for (int i = 0; i < 64; ++i) { a[i] = a[i] * a[(i + 7) & 63] + s; s += a[i]; }
    o[threadIdx.x] = s;
}
template <int N> void q() {
    cudaFuncAttributes at; cudaFuncGetAttributes(&at, k<N>);
    int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k<N>, 544, 0);
    printf("maxnreg %d: numRegs %d maxThreads %d, blocks of 544 per SM: %d\n", N, at.numRegs, at.maxThreadsPerBlock, nb);
}
int main() { q<96>(); q<104>(); q<112>(); q<120>(); return 0; }
