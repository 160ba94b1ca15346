// evaluate.cu -- KITTI scene-flow outlier counts (Table 1
// semantics P:130-155, density P:159; outlier rule SPEC E-1 / S:467).
//
// A pure HBM-bound reduction: every pixel is read once (35 bytes with gt_valid,
// 34 without) and turned into 12 one-bit votes {n_gt, n_eval, d1, d2, fl, sf} x
// {Occ, Noc}.  Each thread handles kPx pixels of a block tile with all loads
// issued before any arithmetic, votes are summed per warp with REDUX, per block in
// shared memory and per quad with 64-bit global atomics (integer sums: the result
// is independent of the schedule).  The float32 decisions use separately rounded
// operations (__fsub_rn / __fmul_rn / __fadd_rn / __fsqrt_rn) so that they are the
// ones a plain C program takes without contraction.
#include "sgm_internal.cuh"

namespace sgm {
namespace {

constexpr int kEvalBlock = 256;
constexpr int kPx = 4;                       // pixels per thread per tile
constexpr int kTile = kEvalBlock * kPx;

__device__ __forceinline__ unsigned outlier(float err, float mag, float tau_abs, float tau_rel) {
    return (err > tau_abs && err > __fmul_rn(tau_rel, mag)) ? 1u : 0u;
}

__device__ __forceinline__ float norm2(float a, float b) {
    return __fsqrt_rn(__fadd_rn(__fmul_rn(a, a), __fmul_rn(b, b)));
}

__global__ void __launch_bounds__(kEvalBlock) eval_kernel(const EvalParams p) {
    __shared__ unsigned blk[12];
    if (threadIdx.x < 12) blk[threadIdx.x] = 0;
    __syncthreads();
    const long long npx = (long long)p.W * p.H;
    const long long q = blockIdx.y;
    const float4 *sf = reinterpret_cast<const float4 *>(p.sf) + q * npx;
    const float2 *gfl = reinterpret_cast<const float2 *>(p.gt_flow) + q * npx;
    const float *gd0 = p.gt_d0 + q * npx, *gd1 = p.gt_d1 + q * npx;
    const uint8_t *vsf = p.valid_sf + q * npx, *noc = p.gt_noc + q * npx;
    const uint8_t *gv = p.gt_valid ? p.gt_valid + q * npx : nullptr;

    unsigned c[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) c[k] = 0;
    for (long long base = (long long)blockIdx.x * kTile; base < npx;
         base += (long long)gridDim.x * kTile) {
        float4 s[kPx]; float2 f[kPx]; float a[kPx], b[kPx];
        unsigned m[kPx];                      // bit0 gt valid, bit1 est valid, bit2 noc
#pragma unroll
        for (int k = 0; k < kPx; ++k) {
            const long long i = base + k * kEvalBlock + threadIdx.x;
            const long long j = i < npx ? i : npx - 1;
            s[k] = __ldcs(sf + j);
            f[k] = __ldcs(gfl + j);
            a[k] = __ldcs(gd0 + j);
            b[k] = __ldcs(gd1 + j);
            const unsigned g = gv ? unsigned(__ldcs(gv + j) != 0) : 1u;
            m[k] = (i < npx ? g : 0u) | (unsigned(__ldcs(vsf + j) != 0) << 1) |
                   (unsigned(__ldcs(noc + j) != 0) << 2);
        }
#pragma unroll
        for (int k = 0; k < kPx; ++k) {
            const unsigned gt = m[k] & 1u;
            const unsigned ev = gt & (m[k] >> 1);
            const unsigned nc = gt & (m[k] >> 2);
            const unsigned o1 = outlier(fabsf(__fsub_rn(s[k].z, a[k])), fabsf(a[k]), p.tau_abs, p.tau_rel);
            const unsigned o2 = outlier(fabsf(__fsub_rn(s[k].w, b[k])), fabsf(b[k]), p.tau_abs, p.tau_rel);
            const unsigned of = outlier(norm2(__fsub_rn(s[k].x, f[k].x), __fsub_rn(s[k].y, f[k].y)),
                                        norm2(f[k].x, f[k].y), p.tau_abs, p.tau_rel);
            const unsigned osf = o1 | o2 | of;
            c[0] += gt; c[1] += ev; c[2] += ev & o1; c[3] += ev & o2; c[4] += ev & of; c[5] += ev & osf;
            const unsigned en = ev & nc;
            c[6] += nc; c[7] += en; c[8] += en & o1; c[9] += en & o2; c[10] += en & of; c[11] += en & osf;
        }
    }
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const unsigned w = __reduce_add_sync(0xffffffffu, c[k]);
        if ((threadIdx.x & 31) == 0 && w) atomicAdd(&blk[k], w);
    }
    __syncthreads();
    if (threadIdx.x < 12 && blk[threadIdx.x])
        atomicAdd(reinterpret_cast<unsigned long long *>(p.counts) + q * 12 + threadIdx.x,
                  (unsigned long long)blk[threadIdx.x]);
}

}  // namespace

cudaError_t launch_evaluate(const EvalParams &p, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(p.counts, 0, sizeof(unsigned long long) * 12 * p.nquads, st);
    if (e != cudaSuccess) return e;
    const long long npx = (long long)p.W * p.H;
    const long long tiles = (npx + kTile - 1) / kTile;
    // ~4 resident 256-thread blocks per SM over the whole batch.
    long long bx = (148LL * 8 + p.nquads - 1) / p.nquads;
    if (bx > tiles) bx = tiles;
    if (bx < 1) bx = 1;
    eval_kernel<<<dim3(unsigned(bx), unsigned(p.nquads)), kEvalBlock, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace sgm
