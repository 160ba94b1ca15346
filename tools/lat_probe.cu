// Latency microbenchmarks (dependent chains timed with clock64) for the sweep's building
// blocks on sm_100a: CREDUX (__reduce_min_sync), SHFL, VIMNMX.U16x2, VIADDMNMX, LDS,
// POPC and an mbarrier arrive->try_wait round trip between two warps.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N 1024
__global__ void k_credux(unsigned *out, long long *cyc, unsigned seed) {
    unsigned v = threadIdx.x ^ seed;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) v = __reduce_min_sync(0xffffffffu, v) + threadIdx.x;
    long long t1 = clock64();
    out[threadIdx.x] = v; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl(unsigned *out, long long *cyc, unsigned seed) {
    unsigned v = threadIdx.x ^ seed;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) v = __shfl_up_sync(0xffffffffu, v, 1) + 1u;
    long long t1 = clock64();
    out[threadIdx.x] = v; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_vmin(unsigned *out, long long *cyc, unsigned seed) {
    unsigned v = threadIdx.x ^ seed, w = seed * 3u;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) v = __vminu2(v, w) ^ 0x10001u;
    long long t1 = clock64();
    out[threadIdx.x] = v; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_vaddmin(unsigned *out, long long *cyc, unsigned seed) {
    unsigned v = threadIdx.x ^ seed, w = seed * 3u;
#pragma unroll 1
    for (int i = 0; i < 4; ++i) w += i;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) v = __viaddmin_u16x2(v, 0x10001u, w);
    long long t1 = clock64();
    out[threadIdx.x] = v; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_popc(unsigned *out, long long *cyc, unsigned seed) {
    unsigned v = threadIdx.x ^ seed;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) v = __popc(v) + seed;
    long long t1 = clock64();
    out[threadIdx.x] = v; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(unsigned *out, long long *cyc, unsigned seed) {
    __shared__ unsigned s[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) s[i] = (i + 1) & 1023;
    __syncwarp();
    unsigned v = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) v = s[v];
    long long t1 = clock64();
    out[threadIdx.x] = v; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
// ping-pong between warp 0 and warp 1 through two mbarriers: round trip = 2 handoffs
__global__ void k_mbar(unsigned *out, long long *cyc, unsigned hint) {
    __shared__ __align__(8) unsigned long long b[2];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&b[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&b[1])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) {
        if (w == 0) {
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&b[0])) : "memory");
            asm volatile("{\n .reg .pred P;\nW1: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n @!P bra W1;\n}" ::"r"(sa(&b[1])), "r"(i & 1), "r"(hint) : "memory");
        } else {
            asm volatile("{\n .reg .pred P;\nW2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n @!P bra W2;\n}" ::"r"(sa(&b[0])), "r"(i & 1), "r"(hint) : "memory");
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&b[1])) : "memory");
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = 0;
}

// gpu-scope fence latency right after a global store (the band producer's publish)
__global__ void k_fence(unsigned *out, long long *cyc, unsigned mode) {
    long long t0 = clock64();
    for (int i = 0; i < 64; ++i) {
        out[threadIdx.x + 32 * (i & 7)] = i;
        if (mode == 0) __threadfence();
        else asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    unsigned *o; long long *c, h;
    cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
    auto run = [&](const char *name, void (*k)(unsigned *, long long *, unsigned), int threads, int iters, unsigned arg) {
        k<<<1, threads>>>(o, c, arg); cudaDeviceSynchronize();
        k<<<1, threads>>>(o, c, arg); cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %7.1f cycles/op  (%s)\n", name, double(h) / iters, cudaGetErrorString(e));
    };
    run("CREDUX.MIN + IADD", k_credux, 32, N, 7);
    run("SHFL.UP + IADD", k_shfl, 32, N, 7);
    run("VIMNMX.U16x2 + LOP3", k_vmin, 32, N, 7);
    run("VIADDMNMX.U16x2", k_vaddmin, 32, N, 7);
    run("POPC + IADD", k_popc, 32, N, 7);
    run("LDS (dependent)", k_lds, 32, N, 7);
    run("st + __threadfence (sc.gpu)", k_fence, 32, 64, 0);
    run("st + fence.acq_rel.gpu", k_fence, 32, 64, 1);
    run("mbarrier ping-pong (hint 0)", k_mbar, 64, 512, 0);
    run("mbarrier ping-pong (hint 20us)", k_mbar, 64, 512, 20000);
    return 0;
}
