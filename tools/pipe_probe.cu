// Throughput microbenchmark: which instructions share a pipe on sm_100a.
// 32 warps/block, 8 independent chains per thread; reports warp-instructions per
// cycle per SMSP for each op alone and for 1:1 mixes.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define ITER 2048
template <int OP>
__device__ __forceinline__ unsigned op(unsigned a, unsigned b) {
    if (OP == 0) return __vminu2(a, b);                         // VIMNMX.U16x2
    if (OP == 1) return __viaddmin_u16x2(a, 0x00070007u, b);      // VIADDMNMX
    if (OP == 2) { __half2 x = *(__half2 *)&a, y = *(__half2 *)&b; __half2 r = __hmin2(x, y); return *(unsigned *)&r; }
    if (OP == 3) { __half2 x = *(__half2 *)&a, y = *(__half2 *)&b; __half2 r = __hadd2(x, y); return *(unsigned *)&r; }
    if (OP == 4) return a * 3u + b;                              // IMAD
    if (OP == 5) return __byte_perm(a, b, 0x5432);              // PRMT
    if (OP == 6) return a + b;                                   // IADD3 / IMAD.IADD
    if (OP == 7) return a ^ b;                                   // LOP3
    if (OP == 8) return min(a, b);                               // IMNMX
    if (OP == 9) return __popc(a) + b;                           // POPC (+add)
    if (OP == 10) { float x = __uint_as_float(a), y = __uint_as_float(b); return __float_as_uint(fminf(x, y)); }
    if (OP == 11) return __vadd2(a, b);                          // VIADD.16x2
    return a;
}
template <int OPA, int OPB>
__global__ void k(unsigned *out, long long *cyc, unsigned s) {
    unsigned v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = threadIdx.x * (j + 1) + s;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = (j & 1) ? op<OPB>(v[j], v[(j + 3) & 7]) : op<OPA>(v[j], v[(j + 5) & 7]);
    }
    __syncthreads();
    long long t1 = clock64();
    unsigned acc = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc ^= v[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
const char *names[] = {"VIMNMX.U16x2", "VIADDMNMX", "HMNMX2", "HADD2", "IMAD", "PRMT", "IADD", "LOP3", "IMNMX", "POPC+IADD", "FMNMX", "VIADD.16x2"};
unsigned *o; long long *c;
template <int A, int B>
void run() {
    k<A, B><<<1, 1024>>>(o, c, 5); cudaDeviceSynchronize();
    k<A, B><<<1, 1024>>>(o, c, 5); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double instr_per_smsp = 8.0 * ITER * 32 / 4;   // warp-instrs per SMSP (8 warps x 8 chains x ITER)
    printf("%-14s + %-14s : %.3f warp-inst/cycle/SMSP\n", names[A], names[B], instr_per_smsp / h);
}
int main() {
    cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 64);
    run<0, 0>(); run<1, 1>(); run<2, 2>(); run<3, 3>(); run<4, 4>(); run<5, 5>(); run<6, 6>();
    run<7, 7>(); run<8, 8>(); run<9, 9>(); run<10, 10>(); run<11, 11>();
    run<0, 2>(); run<0, 3>(); run<0, 4>(); run<0, 6>(); run<1, 2>(); run<2, 3>(); run<0, 5>(); run<2, 4>(); run<0, 10>();
    return 0;
}
