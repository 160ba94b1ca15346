// evaluate.cu -- KITTI scene-flow outlier counts (Table 1
// semantics P:130-155, density P:159; outlier rule SPEC E-1 / S:467).
//
// A pure HBM-bound reduction: every pixel is read once (35 bytes with gt_valid,
// 34 without) and turned into 12 one-bit votes {n_gt, n_eval, d1, d2, fl, sf} x
// {Occ, Noc}.  One wave of resident blocks; the blocks of a quad grid-stride over
// it together.  Vector path: a thread reads 4 consecutive pixels per iteration
// (sf 4 x 16 B, gt_flow 2 x 16 B, gt_d0/gt_d1 16 B each, masks 4 B each); the <= 3
// pixels before the first 16-byte-aligned group of a quad and after its last one are
// done by the scalar vote of block 0.  Scalar path (any base misaligned): one pixel
// per thread per load.  Votes are summed per warp with REDUX and per block in shared
// memory; the last block to finish (atomic ticket) adds the block partials per quad
// in a fixed order and overwrites the counts -- one launch, no memset, integer sums
// independent of the schedule.  The float32 decisions use separately rounded
// operations (__fsub_rn / __fmul_rn / __fadd_rn / __fsqrt_rn) so that they are the
// ones a plain C program takes without contraction.
#include "sgm_internal.cuh"

namespace sgm {
namespace {

constexpr int kEvalBlock = 256;

__device__ __forceinline__ unsigned outlier(float err, float mag, float tau_abs, float tau_rel) {
    return (err > tau_abs && err > __fmul_rn(tau_rel, mag)) ? 1u : 0u;
}

__device__ __forceinline__ float norm2(float a, float b) {
    return __fsqrt_rn(__fadd_rn(__fmul_rn(a, a), __fmul_rn(b, b)));
}

__device__ __forceinline__ float4 ld_stream(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ unsigned ld_stream(const unsigned *p) {
    unsigned v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// One pixel's votes.  gt, est, noc are 0/1.
__device__ __forceinline__ void vote(unsigned (&c)[12], const EvalParams &p, float4 s, float fu,
                                     float fv, float a, float b, unsigned gt, unsigned est,
                                     unsigned noc) {
    const unsigned ev = gt & est;
    const unsigned nc = gt & noc;
    const unsigned o1 = outlier(fabsf(__fsub_rn(s.z, a)), fabsf(a), p.tau_abs, p.tau_rel);
    const unsigned o2 = outlier(fabsf(__fsub_rn(s.w, b)), fabsf(b), p.tau_abs, p.tau_rel);
    const unsigned of = outlier(norm2(__fsub_rn(s.x, fu), __fsub_rn(s.y, fv)), norm2(fu, fv),
                                p.tau_abs, p.tau_rel);
    const unsigned osf = o1 | o2 | of;
    c[0] += gt; c[1] += ev; c[2] += ev & o1; c[3] += ev & o2; c[4] += ev & of; c[5] += ev & osf;
    const unsigned en = ev & nc;
    c[6] += nc; c[7] += en; c[8] += en & o1; c[9] += en & o2; c[10] += en & of; c[11] += en & osf;
}

__device__ __forceinline__ void vote_pixel(unsigned (&c)[12], const EvalParams &p, long long i) {
    const float4 s = reinterpret_cast<const float4 *>(p.sf)[i];
    const float2 f = reinterpret_cast<const float2 *>(p.gt_flow)[i];
    const unsigned g = p.gt_valid ? unsigned(p.gt_valid[i] != 0) : 1u;
    vote(c, p, s, f.x, f.y, p.gt_d0[i], p.gt_d1[i], g, unsigned(p.valid_sf[i] != 0),
         unsigned(p.gt_noc[i] != 0));
}

__device__ __forceinline__ unsigned nz_byte(unsigned w, int k) {
    return unsigned(((w >> (8 * k)) & 0xffu) != 0);
}

// Four consecutive pixels: sf 4 x 16 B, gt_flow 2 x 16 B, gt_d0/gt_d1 16 B, masks 4 B.
struct Group {
    float4 s[4], f01, f23, a, b;
    unsigned vw, nw, gw;
    __device__ __forceinline__ void load(const float4 *sf4, const float4 *fl4, const float4 *a4,
                                         const float4 *b4, const unsigned *v4, const unsigned *n4,
                                         const unsigned *g4, long long g) {
#pragma unroll
        for (int k = 0; k < 4; ++k) s[k] = ld_stream(sf4 + 4 * g + k);
        f01 = ld_stream(fl4 + 2 * g); f23 = ld_stream(fl4 + 2 * g + 1);
        a = ld_stream(a4 + g); b = ld_stream(b4 + g);
        vw = ld_stream(v4 + g); nw = ld_stream(n4 + g);
        gw = g4 ? ld_stream(g4 + g) : 0x01010101u;
    }
    __device__ __forceinline__ void votes(unsigned (&c)[12], const EvalParams &p) const {
        vote(c, p, s[0], f01.x, f01.y, a.x, b.x, nz_byte(gw, 0), nz_byte(vw, 0), nz_byte(nw, 0));
        vote(c, p, s[1], f01.z, f01.w, a.y, b.y, nz_byte(gw, 1), nz_byte(vw, 1), nz_byte(nw, 1));
        vote(c, p, s[2], f23.x, f23.y, a.z, b.z, nz_byte(gw, 2), nz_byte(vw, 2), nz_byte(nw, 2));
        vote(c, p, s[3], f23.z, f23.w, a.w, b.w, nz_byte(gw, 3), nz_byte(vw, 3), nz_byte(nw, 3));
    }
};

template <bool VEC>
__global__ void __launch_bounds__(kEvalBlock) eval_kernel(const EvalParams p) {
    __shared__ unsigned blk[12];
    __shared__ bool last;
    if (threadIdx.x < 12) blk[threadIdx.x] = 0;
    __syncthreads();
    const long long npx = (long long)p.W * p.H;
    const long long q0 = blockIdx.y * npx;           // first flat pixel of this quad

    unsigned c[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) c[k] = 0;
    if (VEC) {
        // groups of 4 flat pixels fully inside the quad, 16-byte aligned for every array
        const long long g0 = (q0 + 3) >> 2, g1 = (q0 + npx) >> 2;
        const long long ng = g1 > g0 ? g1 - g0 : 0;
        const long long hi = g0 + ng;
        const float4 *sf4 = reinterpret_cast<const float4 *>(p.sf);
        const float4 *fl4 = reinterpret_cast<const float4 *>(p.gt_flow);
        const float4 *a4 = reinterpret_cast<const float4 *>(p.gt_d0);
        const float4 *b4 = reinterpret_cast<const float4 *>(p.gt_d1);
        const unsigned *v4 = reinterpret_cast<const unsigned *>(p.valid_sf);
        const unsigned *n4 = reinterpret_cast<const unsigned *>(p.gt_noc);
        const unsigned *g4 = reinterpret_cast<const unsigned *>(p.gt_valid);
        // grid-stride: the blocks of a quad sweep one compact window of every array
        // (better DRAM row locality than one contiguous share per block)
        for (long long g = g0 + (long long)blockIdx.x * kEvalBlock + threadIdx.x; g < hi;
             g += (long long)gridDim.x * kEvalBlock) {
            Group cur;
            cur.load(sf4, fl4, a4, b4, v4, n4, g4, g);
            cur.votes(c, p);
        }
        // ragged ends of the quad: [q0, 4*g0) and [4*g1, q0+npx) (or the whole quad if tiny)
        if (blockIdx.x == 0 && threadIdx.x < 8) {
            if (ng == 0) {
                for (long long i = q0 + threadIdx.x; i < q0 + npx; i += 8) vote_pixel(c, p, i);
            } else {
                const long long i = threadIdx.x < 4 ? q0 + threadIdx.x : 4 * g1 + (threadIdx.x - 4);
                const bool in = threadIdx.x < 4 ? i < 4 * g0 : i < q0 + npx;
                if (in) vote_pixel(c, p, i);
            }
        }
    } else {
        const long long share = ((npx + gridDim.x - 1) / gridDim.x + 31) & ~31LL;
        const long long lo = (long long)blockIdx.x * share;
        const long long hi = lo + share < npx ? lo + share : npx;
        for (long long i = lo + threadIdx.x; i < hi; i += kEvalBlock) vote_pixel(c, p, q0 + i);
    }
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const unsigned w = __reduce_add_sync(0xffffffffu, c[k]);
        if ((threadIdx.x & 31) == 0 && w) atomicAdd(&blk[k], w);
    }
    __syncthreads();
    // Block partials -> scratch; the last block to finish (ticket) sums them per quad in
    // a fixed order and overwrites `counts`.
    const unsigned nblk = gridDim.x * gridDim.y;
    const unsigned bid = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x < 12) p.part[bid * 12 + threadIdx.x] = blk[threadIdx.x];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(p.ticket, 1u) == nblk - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (unsigned j = threadIdx.x; j < 12u * gridDim.y; j += blockDim.x) {
        const unsigned qq = j / 12, k = j % 12;
        const volatile unsigned *src = p.part + (qq * gridDim.x) * 12 + k;
        unsigned long long sum = 0;
        for (unsigned bx = 0; bx < gridDim.x; ++bx) sum += src[bx * 12];
        p.counts[qq * 12 + k] = sum;
    }
    if (threadIdx.x == 0) *p.ticket = 0;
}

int g_eval_blocks[2] = {0, 0};   // resident blocks on the device (SMs x occupancy)

bool aligned(const void *ptr, unsigned a) { return (reinterpret_cast<uintptr_t>(ptr) & (a - 1)) == 0; }

template <bool VEC>
cudaError_t launch(const EvalParams &p, cudaStream_t st) {
    int &nb = g_eval_blocks[VEC];
    if (nb == 0) {
        int dev = 0, sms = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, eval_kernel<VEC>, kEvalBlock, 0);
        const int b = sms * (occ < 1 ? 1 : occ);
        nb = b < evaluate_max_blocks() ? b : evaluate_max_blocks();
    }
    const long long npx = (long long)p.W * p.H;
    // one wave of resident blocks over the whole batch, split evenly over the quads
    long long bx = nb / p.nquads;
    const long long cap = VEC ? (npx / 4 + kEvalBlock - 1) / kEvalBlock : (npx + 31) / 32;
    if (bx > cap) bx = cap;
    if (bx < 1) bx = 1;
    eval_kernel<VEC><<<dim3(unsigned(bx), unsigned(p.nquads)), kEvalBlock, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace

int evaluate_max_blocks() { return 148 * 8; }

cudaError_t launch_evaluate(const EvalParams &p, cudaStream_t st) {
    const bool vec = aligned(p.sf, 16) && aligned(p.gt_flow, 16) && aligned(p.gt_d0, 16) &&
                     aligned(p.gt_d1, 16) && aligned(p.valid_sf, 16) && aligned(p.gt_noc, 16) &&
                     (!p.gt_valid || aligned(p.gt_valid, 16));
    return vec ? launch<true>(p, st) : launch<false>(p, st);
}

}  // namespace sgm
