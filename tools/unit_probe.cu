// Throughput of warp-collective / uniform units on sm_100a: CREDUX, SHFL, POPC, LDS,
// mbarrier arrive.  32 warps per block, 4 independent chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
#define ITER 1024
template <int OP>
__global__ void k(unsigned *out, long long *cyc, unsigned s) {
    __shared__ unsigned sm[4096];
    __shared__ __align__(8) unsigned long long bar[32];
    if (threadIdx.x < 32) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[threadIdx.x])));
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 7;
    __syncthreads();
    unsigned v0 = threadIdx.x + s, v1 = v0 * 3, v2 = v0 * 5, v3 = v0 * 7;
    long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < ITER; ++i) {
        if (OP == 0) {
            v0 = __reduce_min_sync(~0u, v0) ^ threadIdx.x; v1 = __reduce_min_sync(~0u, v1) ^ threadIdx.x;
            v2 = __reduce_min_sync(~0u, v2) ^ threadIdx.x; v3 = __reduce_min_sync(~0u, v3) ^ threadIdx.x;
        } else if (OP == 1) {
            v0 = __shfl_up_sync(~0u, v0, 1) + 1; v1 = __shfl_up_sync(~0u, v1, 1) + 1;
            v2 = __shfl_up_sync(~0u, v2, 1) + 1; v3 = __shfl_up_sync(~0u, v3, 1) + 1;
        } else if (OP == 2) {
            v0 = __popc(v0) + v1; v1 = __popc(v1) + v2; v2 = __popc(v2) + v3; v3 = __popc(v3) + v0;
        } else if (OP == 3) {
            v0 = sm[(v0 + threadIdx.x) & 4095]; v1 = sm[(v1 + threadIdx.x) & 4095];
            v2 = sm[(v2 + threadIdx.x) & 4095]; v3 = sm[(v3 + threadIdx.x) & 4095];
        } else if (OP == 4) {
            unsigned a = (unsigned)__cvta_generic_to_shared(&bar[(threadIdx.x >> 5)]);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
        } else if (OP == 5) {   // single-lane arrive after syncwarp
            unsigned a = (unsigned)__cvta_generic_to_shared(&bar[(threadIdx.x >> 5)]);
            for (int q = 0; q < 4; ++q) { __syncwarp(); if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory"); }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    out[threadIdx.x] = v0 ^ v1 ^ v2 ^ v3;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    unsigned *o; long long *c, h;
    cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 64);
    const char *n[] = {"CREDUX.MIN", "SHFL.UP", "POPC", "LDS (random)", "mbarrier.arrive x32 lanes", "syncwarp+lane0 arrive"};
    auto run = [&](int which, auto kern) {
        kern<<<1, 1024>>>(o, c, 3); cudaDeviceSynchronize();
        kern<<<1, 1024>>>(o, c, 3); cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        double ops = 32.0 * 4 * ITER;   // warp-ops per SM
        printf("%-28s %.3f warp-ops/cycle/SM  (%s)\n", n[which], ops / h, cudaGetErrorString(e));
    };
    run(0, k<0>); run(1, k<1>); run(2, k<2>); run(3, k<3>); run(4, k<4>); run(5, k<5>);
}
