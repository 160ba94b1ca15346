// sweep_common.cuh -- device building blocks of the SGM sweep kernels (sweep.cu,
// sweep_stair.cu): vector I/O, the DPX path update, mbarrier / cp.async / L2 helpers.
// Nothing here is shared with oracle/ (the CPU oracle).
#pragma once

#include "sgm_internal.cuh"

namespace sgm {
namespace sweep_detail {

// ---------------------------------------------------------------- small helpers
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <int R>
struct VecIO;

template <>
struct VecIO<1> {
    static __device__ __forceinline__ void ld(const uint16_t *p, uint32_t (&v)[1]) {
        v[0] = *reinterpret_cast<const uint32_t *>(p);
    }
    static __device__ __forceinline__ void st(uint16_t *p, const uint32_t (&v)[1]) {
        *reinterpret_cast<uint32_t *>(p) = v[0];
    }
};
template <>
struct VecIO<2> {
    static __device__ __forceinline__ void ld(const uint16_t *p, uint32_t (&v)[2]) {
        uint2 t = *reinterpret_cast<const uint2 *>(p);
        v[0] = t.x; v[1] = t.y;
    }
    static __device__ __forceinline__ void st(uint16_t *p, const uint32_t (&v)[2]) {
        *reinterpret_cast<uint2 *>(p) = make_uint2(v[0], v[1]);
    }
};
template <>
struct VecIO<3> {
    static __device__ __forceinline__ void ld(const uint16_t *p, uint32_t (&v)[3]) {
        const uint32_t *q = reinterpret_cast<const uint32_t *>(p);
        v[0] = q[0]; v[1] = q[1]; v[2] = q[2];
    }
    static __device__ __forceinline__ void st(uint16_t *p, const uint32_t (&v)[3]) {
        uint32_t *q = reinterpret_cast<uint32_t *>(p);
        q[0] = v[0]; q[1] = v[1]; q[2] = v[2];
    }
};
template <>
struct VecIO<4> {
    static __device__ __forceinline__ void ld(const uint16_t *p, uint32_t (&v)[4]) {
        uint4 t = *reinterpret_cast<const uint4 *>(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
    static __device__ __forceinline__ void st(uint16_t *p, const uint32_t (&v)[4]) {
        *reinterpret_cast<uint4 *>(p) = make_uint4(v[0], v[1], v[2], v[3]);
    }
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ int ld_relaxed_gpu(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Drop a 128-byte line from L2 without writing it back (PTX discard.global.L2): the band
// handoff rows are read exactly once, by the next band, right after they are written; once
// they sit in the consumer's shared memory their dirty L2 lines would otherwise be written
// back to DRAM for nothing (~0.7 GB per sweep launch on 8 Driving quads).
__device__ __forceinline__ void discard_l2(const void *p) {
    asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(p) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(int *p, int v) {
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

#ifndef SGM_UR_MB
#define SGM_UR_MB 0
#endif

// Integer multiply-add on the FMA pipe.  `one` is a runtime 1 (kernel parameter), so
// ptxas cannot fold a*one+c into an ALU-pipe IADD3: the min-plus work saturates the
// half-rate ALU pipe (VIMNMX / VIADDMNMX / PRMT / LOP3 all issue there), while IMAD
// issues on the otherwise idle FMA pipe.
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// One semi-global path update for the CPL cells a lane holds, on path vectors
// carried with a +P1 bias (Lb = L + P1, u16x2 pairs):
//   t  = min(L(d-1) + P1, L(d+1) + P1, L(d), m + P2)      (exactly the recursion's min term)
//      = VIMNMX3(Lb(d-1), Lb(d+1), VIADDMNMX(Lb(d), -P1, m + P2))
//   Lb'(d) = C(d) + t - m + P1,   m = min_k L(p - r, k) = min_k Lb - P1.
// The bias turns the three min operations per pair of the plain form into two (the +P1
// of the neighbours is already in their stored value).  A path start is the vector P1
// (L = 0, m = 0), which returns Lb' = C + P1.
//
// Folded disparity layout: register r of lane l holds the pair k = R*l + r, i.e. the
// disparities (k, Dp-1-k) in its (low, high) halves.  The d-1 / d+1 neighbours of both
// halves of pair k are then the halves of pairs k-1 and k+1, aligned: no byte permutes,
// one SHFL each way per path.  Two lanes need care:
//   * pair 0 (lane 0, reg 0) has no pair -1 (d = 0 has no d-1, d = Dp-1 no d+1); the
//     clamped SHFL returns the lane's own reg R-1, which is pair 1 -- a duplicate of the
//     other neighbour, hence harmless (G7) -- for R <= 2; for R > 2 it is forced to 0xFFFF.
//   * pair Dp/2-1 (lane 31, reg R-1) is the fold (Dp/2-1, Dp/2): its "pair k+1" is itself
//     with the halves swapped -- one PRMT with a per-lane selector (sel_fold).
template <int R>
__device__ __forceinline__ void path_update(const uint32_t (&prev)[R], const uint32_t (&C)[R],
                                            uint32_t (&out)[R], uint32_t negp1x2, uint32_t p2mp1x2,
                                            uint32_t twop1x2, uint32_t sel_fold, uint32_t ff_lane0,
                                            uint32_t k10001 = 0x10001u, uint32_t kneg10001 = 0xFFFEFFFFu) {
    // mb = min_k Lb(p - r, k): min over the lane's pairs, then over the two halves (the
    // high half is brought down with IMAD.HI on the FMA pipe), then over the warp
    uint32_t v = prev[0];
#pragma unroll
    for (int r = 1; r < R; ++r) v = __vminu2(v, prev[r]);
    v = __vminu2(v, __umulhi(v, 0x10000u));           // lo = min(lo, hi), hi = 0
    const uint32_t mb = __reduce_min_sync(0xffffffffu, v);
#if SGM_UR_MB == 2
    // plain expressions: the compiler may keep both in the uniform datapath (mb is the
    // CREDUX result in a uniform register, the constants are uniform)
    const uint32_t mP2 = mb * 0x10001u + p2mp1x2;
    const uint32_t K = twop1x2 - mb * 0x10001u;
#elif SGM_UR_MB
    // mb lives in a uniform register (CREDUX): as IMAD's B operand it needs no move to a
    // vector register; the multipliers are runtime registers (k10001 = 0x10001, kneg = -0x10001)
    const uint32_t mP2 = imad(k10001, mb, p2mp1x2);
    const uint32_t K = imad(kneg10001, mb, twop1x2);
#else
    const uint32_t mP2 = imad(mb, 0x10001u, p2mp1x2);  // m + P2 = mb - P1 + P2, both halves
    const uint32_t K = imad(mb, 0xFFFEFFFFu, twop1x2); // 2 P1 - mb in both halves (mod 2^32)
#endif
    // neighbour pairs k-1 (of reg 0) and k+1 (of reg R-1)
    uint32_t up = __shfl_up_sync(0xffffffffu, prev[R - 1], 1);
    if (R > 2) up |= ff_lane0;
    const uint32_t dn = __byte_perm(__shfl_down_sync(0xffffffffu, prev[0], 1), prev[R - 1], sel_fold);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t centre = __viaddmin_u16x2(prev[r], negp1x2, mP2);   // min(L(d), m + P2)
        const uint32_t t = __vimin3_u16x2(r == 0 ? up : prev[r - 1], r == R - 1 ? dn : prev[r + 1], centre);
        // C + t - m + P1: exact mod 2^32, every half's result lies in [P1, 2^16)
        out[r] = t + C[r] + K;
    }
}

__device__ __forceinline__ unsigned smem_addr(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(b)) : "memory");
}
// mbarrier wait: try_wait without a suspend-time hint (the hardware's default window).
// Measured against a 20 us suspend hint (7.17 ms per step; the hinted form compiles to a
// TRYWAIT + NANOSLEEP.SYNCS loop that woke ~70 times per wait) and a test_wait spin
// (7.27 ms): the plain form is fastest (7.16 ms).
#ifndef SGM_MBAR_HINT
#define SGM_MBAR_HINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
#if SGM_MBAR_HINT
    asm volatile(
        "{\n .reg .pred P1;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_addr(b)),
        "r"(parity), "n"(SGM_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n .reg .pred P1;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
#endif
}

// One mbarrier test (no retry loop): true once the phase with `parity` has completed.
__device__ __forceinline__ bool mbar_test(uint64_t *b, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred P1;\n"
        " mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        " selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
    return ok != 0;
}

}  // namespace sweep_detail
}  // namespace sgm
