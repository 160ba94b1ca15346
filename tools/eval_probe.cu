// eval_probe.cu -- read-bandwidth variants for the evaluation reduction (34 B/px over
// 7 arrays).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/eval_probe tools/eval_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

template <int HINT> __device__ __forceinline__ float4 ld4(const float4 *p) {
    float4 v;
    if (HINT == 1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    else
        v = __ldcs(p);
    return v;
}
template <int HINT> __device__ __forceinline__ float2 ld2(const float2 *p) {
    float2 v;
    if (HINT == 1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f32 {%0,%1}, [%2];"
                     : "=f"(v.x), "=f"(v.y) : "l"(p));
    else
        v = __ldcs(p);
    return v;
}
template <int HINT> __device__ __forceinline__ float ld1(const float *p) {
    float v;
    if (HINT == 1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.f32 %0, [%1];" : "=f"(v) : "l"(p));
    else
        v = __ldcs(p);
    return v;
}
template <int HINT> __device__ __forceinline__ unsigned ldb(const uint8_t *p) {
    unsigned short v;
    if (HINT == 1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.u8 %0, [%1];" : "=h"(v) : "l"(p));
    else
        v = __ldcs(p);
    return v;
}

// 1 px per (thread, k), interleaved tiles, contiguous share per block
template <int KPX, int HINT>
__global__ void __launch_bounds__(256) v_interleaved(const float4 *sf, const float2 *fl, const float *a,
                                                     const float *b, const uint8_t *m0, const uint8_t *m1,
                                                     long long npx, unsigned *out) {
    const long long share = ((npx + gridDim.x - 1) / gridDim.x + 31) & ~31LL;
    const long long lo = blockIdx.x * share, hi = lo + share < npx ? lo + share : npx;
    unsigned acc = 0;
    for (long long base = lo; base < hi; base += 256 * KPX) {
        float4 s[KPX]; float2 f[KPX]; float x[KPX], y[KPX]; unsigned m[KPX];
#pragma unroll
        for (int k = 0; k < KPX; ++k) {
            long long i = base + k * 256 + threadIdx.x;
            i = i < hi ? i : hi - 1;
            s[k] = ld4<HINT>(sf + i); f[k] = ld2<HINT>(fl + i); x[k] = ld1<HINT>(a + i);
            y[k] = ld1<HINT>(b + i); m[k] = ldb<HINT>(m0 + i) + ldb<HINT>(m1 + i);
        }
#pragma unroll
        for (int k = 0; k < KPX; ++k)
            acc += (s[k].x + s[k].y + s[k].z + s[k].w + f[k].x + f[k].y + x[k] + y[k] > 1e30f) + m[k];
    }
    acc = __reduce_add_sync(0xffffffffu, acc);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

// 4 consecutive px per thread: sf 4x16B, flow 2x16B, d 16B each, masks u32 each
template <int HINT>
__global__ void __launch_bounds__(256) v_vec4(const float4 *sf, const float2 *fl, const float *a,
                                              const float *b, const uint8_t *m0, const uint8_t *m1,
                                              long long npx, unsigned *out) {
    const long long ng = npx / 4;
    unsigned acc = 0;
    for (long long g = blockIdx.x * 256LL + threadIdx.x; g < ng; g += gridDim.x * 256LL) {
        float4 s0 = ld4<HINT>(sf + 4 * g), s1 = ld4<HINT>(sf + 4 * g + 1), s2 = ld4<HINT>(sf + 4 * g + 2),
               s3 = ld4<HINT>(sf + 4 * g + 3);
        float4 f0 = ld4<HINT>(reinterpret_cast<const float4 *>(fl) + 2 * g),
               f1 = ld4<HINT>(reinterpret_cast<const float4 *>(fl) + 2 * g + 1);
        float4 x = ld4<HINT>(reinterpret_cast<const float4 *>(a) + g);
        float4 y = ld4<HINT>(reinterpret_cast<const float4 *>(b) + g);
        unsigned u0 = __ldcs(reinterpret_cast<const unsigned *>(m0) + g);
        unsigned u1 = __ldcs(reinterpret_cast<const unsigned *>(m1) + g);
        float t = s0.x + s1.y + s2.z + s3.w + f0.x + f1.w + x.y + y.z;
        acc += (t > 1e30f) + __popc(u0 ^ u1);
    }
    acc = __reduce_add_sync(0xffffffffu, acc);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

// pure float4 stream of the same byte count (upper bound)
__global__ void __launch_bounds__(256) v_copyread(const float4 *p, long long n4, unsigned *out) {
    unsigned acc = 0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += gridDim.x * 256LL) {
        float4 v = __ldcs(p + i);
        acc += (v.x + v.y + v.z + v.w > 1e30f);
    }
    acc = __reduce_add_sync(0xffffffffu, acc);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

int main() {
    const long long npx = 8LL * 465750;
    float4 *sf; float2 *fl; float *a, *b; uint8_t *m0, *m1; unsigned *out; char *flush;
    CK(cudaMalloc(&sf, npx * 16)); CK(cudaMalloc(&fl, npx * 8)); CK(cudaMalloc(&a, npx * 4));
    CK(cudaMalloc(&b, npx * 4)); CK(cudaMalloc(&m0, npx)); CK(cudaMalloc(&m1, npx));
    CK(cudaMalloc(&out, 4)); CK(cudaMalloc(&flush, 256 << 20));
    float4 *big; CK(cudaMalloc(&big, npx * 34 + 64)); CK(cudaMemset(big, 0, npx * 34 + 64));
    CK(cudaMemset(sf, 0, npx * 16)); CK(cudaMemset(fl, 0, npx * 8)); CK(cudaMemset(a, 0, npx * 4));
    CK(cudaMemset(b, 0, npx * 4)); CK(cudaMemset(m0, 0, npx)); CK(cudaMemset(m1, 0, npx));
    const double bytes = npx * 34.0;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](const char *name, auto launch) {
        float best = 1e9, tot = 0; int reps = 20;
        for (int r = 0; r < reps + 3; ++r) {
            cudaMemsetAsync(flush, r, 256 << 20);
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 3) { tot += ms; best = ms < best ? ms : best; }
        }
        printf("%-28s avg %7.2f us  best %7.2f us  %6.0f GB/s (avg)\n", name, 1e3 * tot / reps, 1e3 * best,
               bytes / (tot / reps * 1e-3) / 1e9);
    };
    for (int bps : {4, 8}) {
        const int grid = 148 * bps;
        char nm[64];
        snprintf(nm, 64, "interleaved k4 h0 g%d", grid);
        timeit(nm, [&] { v_interleaved<4, 0><<<grid, 256>>>(sf, fl, a, b, m0, m1, npx, out); });
        snprintf(nm, 64, "interleaved k4 h1 g%d", grid);
        timeit(nm, [&] { v_interleaved<4, 1><<<grid, 256>>>(sf, fl, a, b, m0, m1, npx, out); });
        snprintf(nm, 64, "interleaved k8 h1 g%d", grid);
        timeit(nm, [&] { v_interleaved<8, 1><<<grid, 256>>>(sf, fl, a, b, m0, m1, npx, out); });
        snprintf(nm, 64, "interleaved k2 h1 g%d", grid);
        timeit(nm, [&] { v_interleaved<2, 1><<<grid, 256>>>(sf, fl, a, b, m0, m1, npx, out); });
        snprintf(nm, 64, "vec4 h0 g%d", grid);
        timeit(nm, [&] { v_vec4<0><<<grid, 256>>>(sf, fl, a, b, m0, m1, npx, out); });
        snprintf(nm, 64, "vec4 h1 g%d", grid);
        timeit(nm, [&] { v_vec4<1><<<grid, 256>>>(sf, fl, a, b, m0, m1, npx, out); });
        snprintf(nm, 64, "copyread g%d", grid);
        timeit(nm, [&] { v_copyread<<<grid, 256>>>(big, (long long)(bytes / 16), out); });
    }
    timeit("vec4 h1 g4736", [&] { v_vec4<1><<<148 * 32, 256>>>(sf, fl, a, b, m0, m1, npx, out); });
    timeit("copyread g4736", [&] { v_copyread<<<148 * 32, 256>>>(big, (long long)(bytes / 16), out); });
    timeit("empty launch", [&] { v_copyread<<<1, 32>>>(sf, 0, out); });
    return 0;
}
