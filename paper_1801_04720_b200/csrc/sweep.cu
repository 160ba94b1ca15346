// sweep.cu -- fused matching cost + semi-global aggregation + WTA for sm_100a.
//
// What it computes: for every view-cell (x, y, d)
//   C(x,y,d)  = popcount(census_ref(x,y) ^ census_match(x - d, y))     (C_max outside)
//   L_r(p,d)  = C(p,d) + min(L_r(p-r,d), L_r(p-r,d+-1)+P1, min_k L_r(p-r,k)+P2)
//               - min_k L_r(p-r,k)                                      (8 directions r)
//   S(p,d)    = sum_r L_r(p,d);  d* = smallest argmin_d S;  parabola sub-pixel.
// The right-reference view (match at x + d, G12) is run as a left-reference view
// in mirrored x coordinates, which is bit-identical (S:148 S-5).
//
// Design:
//  * Two sweeps.  The forward sweep walks rows top->bottom, each row left->right, and
//    evaluates the 4 paths whose predecessor is already visited: r = (1,0) (->),
//    (0,1) (down), (1,1) and (-1,1) (diagonals).  It writes S_fwd = sum of those 4
//    path costs as uint16 [H][W][Dp] -- the only W x H x D array that touches HBM,
//    written once, in 64*CPL-byte coalesced chunks.  The backward sweep walks
//    bottom->top, right->left, evaluates the mirrored 4 paths, adds S_fwd and does WTA
//    + parabola in registers; only int16 / float32 disparities leave the SM.
//  * One warp owns one image row; the disparities are folded into pairs k = (k, Dp-1-k)
//    and lane l holds pairs R*l .. R*l+R-1 (R = CPL/2) as packed u16x2 registers (see
//    path_update).  A path update is DPX min-plus: VIADDMNMX.U16x2 / VIMNMX3.U16x2, the
//    d+-1 neighbours are the sibling registers or one SHFL each way, min over d by
//    VIMNMX + CREDUX.MIN (__reduce_min_sync), and the normalisation "+C - m" is a single
//    IADD3 with a two's-complement constant.
//  * The cost C is recomputed on the fly from the census windows (never stored); the
//    two windows of census_match values (low / high halves) slide one position per
//    step by one SHFL each.
//  * Rows of a CTA run as a skewed wavefront: row w+1 consumes row w's path vectors
//    through a shared-memory ring of position slots with full / empty mbarriers
//    (synchronised in groups of positions).  CTAs own bands of up to NW rows (height
//    chosen per call on the host); the band's last row hands its vectors to the next
//    band's CTA through global memory with a progress flag published by a separate
//    warp, prefetched by cp.async.  CTAs take tickets (atomicAdd) so a band only ever
//    waits for an already-running band.
#include <type_traits>

#include "sweep_common.cuh"

// Row -> row ring synchronisation: 1 (default) = one named barrier per warp pair (ids 0..15:
// the producer row's index), met once per position group as a rendezvous -- bar.sync blocks
// in hardware, so a waiting row spends no issue slots; 0 = full / empty mbarriers per ring
// group (the waiting row spins on try_wait: ncu counted ~89 try_wait retries per group wait,
// ~20 % of the sweeps' issued instructions).  Measured (1x B200, same box): 64 quads 49.29 ->
// 47.81 ms, 8 Driving 6.75 -> 6.55, 8 Wide 11.26 -> 10.69, 4 HighRes 20.32 -> 19.65; a producer
// one group further ahead (SGM_NAMED_LEAD=1) was slower (48.48 ms).
#ifndef SGM_NAMED_RING
#define SGM_NAMED_RING 1
#endif
#ifndef SGM_TAIL_SPLIT
#define SGM_TAIL_SPLIT 1
#endif
#ifndef SGM_SLOT_BASE
#define SGM_SLOT_BASE 1
#endif
#ifndef SGM_FINE_PUB
#define SGM_FINE_PUB 0
#endif
#ifndef SGM_FINE_ALL
#define SGM_FINE_ALL 0
#endif
#ifndef SGM_WTA_SHFL
#define SGM_WTA_SHFL 0
#endif
#ifndef SGM_CONST_PARAMS
#define SGM_CONST_PARAMS 1
#endif
#ifndef SGM_PUB_SLEEP
#define SGM_PUB_SLEEP 0
#endif
#ifndef SGM_NAMED_LEAD
#define SGM_NAMED_LEAD 0
#endif
// backward sweep: the sub-pixel / store block (one pixel per lane, every kWtaPeriod positions)
// is only reachable at the last position of an unrolled block when CPL divides the period:
// 1 = test for it there only.  Without it every position carried a BSSY / BRA / BSYNC region
// that also fenced the scheduler: 8 Driving quads backward sweep 2.912 -> 2.714 ms, 64 quads
// 21.19 -> 19.63 ms, 8 Wide quads 5.28 -> 5.06 ms (bit-identical).  For 6 cells per lane the
// period is 30 positions (SGM_PER30; lanes 30, 31 hold no pixel).
#ifndef SGM_FIN_LAST
#define SGM_FIN_LAST 1
#endif
// band input (gbuf rows of the band above): L2 prefetch this many positions ahead (0 = off).
// Measured slower at 16 / 32 / 64 positions alike (64 quads forward sweep 20.88 -> 21.39 ms, 8
// Driving quads 2.90 -> 2.96 ms): the extra code costs more than the latency it hides.
#ifndef SGM_GIN_L2PF
#define SGM_GIN_L2PF 0
#endif
#ifndef SGM_REFILL_FIRST
#define SGM_REFILL_FIRST 0
#endif
#ifndef SGM_PER30
#define SGM_PER30 1
#endif
// backward sweep: L2 prefetch of the S_fwd row this many positions ahead, per cells-per-lane
// (0 = off).  Measured with SGM_FIN_LAST: 8 Wide quads (CPL 8) 5.06 -> 4.44 ms with 16; 4
// HighRes quads (CPL 6) 9.75 -> 9.33 ms with 16 (32: 9.42); 8 Driving quads (CPL 4) 2.714 ->
// 2.775 ms with 16 (off).
#ifndef SGM_L2PF_BULK
#define SGM_L2PF_BULK 0
#endif
#ifndef SGM_L2PF_PH
#define SGM_L2PF_PH 0
#endif
#ifndef SGM_L2PF4
#define SGM_L2PF4 0
#endif
#ifndef SGM_L2PF6
#define SGM_L2PF6 16
#endif
#ifndef SGM_L2PF8
#define SGM_L2PF8 16
#endif
// backward sweep: S_fwd register prefetch depth (positions) for 6 / 8 cells per lane.
// Measured, 4 HighRes quads (CPL = 6) before the L2 prefetch: depth 2 9.75 ms, 3 10.32 ms, 6
// 9.44 ms; with the L2 prefetch and the 30-position WTA period: depth 2 8.80 ms (kept), 6 8.92
// ms.  8 Wide quads (CPL = 8): depth 2 4.45 ms (kept), 4 4.49 ms.  Outputs bit-identical.
// Measured (64 quads, backward sweep): two blocks with the prefetch 8 deep 19.64 -> 19.75 ms,
// two blocks with the prefetch 4 deep 24.45 ms (the 24 KB loop body no longer fits the
// instruction cache); in latency mode (1 Driving quad) 8 deep is faster: 1.098 -> 1.056 ms.
#ifndef SGM_UR_TICKET
#define SGM_UR_TICKET 0
#endif
#ifndef SGM_BWD4_UNROLL
#define SGM_BWD4_UNROLL 1
#endif
#ifndef SGM_BWD4_UNROLL_FINE
#define SGM_BWD4_UNROLL_FINE 2
#endif
#ifndef SGM_PF4U
#define SGM_PF4U 8
#endif
#ifndef SGM_PF4
#define SGM_PF4 4
#endif
#ifndef SGM_PF6
#define SGM_PF6 2
#endif
#ifndef SGM_PF8
#define SGM_PF8 2
#endif

namespace sgm {
namespace {
using namespace sweep_detail;

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// GS: ring sync group (positions) for CPL <= 4; 0 = the default (kGroupWide, else CPL)
template <int CPL, bool C64, bool BWD, int NW, int GS = 0>
struct Sweep {
    static constexpr int R = CPL / 2;
    static constexpr int DP = 32 * CPL;
    static constexpr int VEC = 3 * DP;             // u16 per ring slot (3 path vectors)
    // Row->row handoff: a ring of RS position slots per warp, synchronised in groups of G
    // consecutive positions (one full-wait / empty-release per group).  The consumer of
    // group g needs the producer to have finished position (g+1)G, and the producer may
    // run at most ~RS-G positions ahead; RS = 16 needs 16 x 3 x Dp x 2 bytes per warp.
    static constexpr int RS = (CPL <= 4) ? kRingWide : kRing;
    // groups align with the unrolled block; CPL > 4 (8 ring slots): 2-position groups
    // (lead window [3, 6]) instead of per-position sync: Wide 15.6 -> 11.5 ms
    static constexpr int G = GS ? GS : ((CPL <= 4) ? (kGroupWide ? kGroupWide : CPL) : 2);
    static constexpr int RG = RS / G;              // groups per ring
    // band-input ring of warp 0 (positions) and census prefetch entries per warp: trimmed
    // for 8 cells per lane so that 17-row bands fit the 227 KB of shared memory
    static constexpr int RING0 = (CPL <= 6) ? kRing0 : kRing0 / 2;
    static constexpr int CEN = BWD ? 0 : 64;       // the backward sweep reads no census

    static constexpr size_t smem_bytes() {
        size_t b = 0;
        b += size_t(NW - 1) * RS * VEC * 2;         // ring (the band's last row writes none)
        b += size_t(RING0) * VEC * 2;               // band input ring
        b += size_t(NW) * 2 * CEN * 8;              // census prefetch (ref, fresh)
        if (BWD) {
            b += size_t(NW) * (DP + 4) * 2;         // WTA scratch (S(d) at index d + 2)
        }
        b += size_t(2) * NW * RG * 8;               // full / empty mbarriers
        b += size_t(2) * kPubDepth * 8;             // publisher mbarriers
        return b;
    }
};

// SOUT (backward sweep only): write S(d) of view 0 (sgm_aggregate, debug) instead of WTA
template <int CPL, bool C64, bool BWD, int NW, bool PAD, bool SOUT, int GS>
__global__ void __launch_bounds__((NW + 1) * 32, kSweepCtasPerSm) sweep_kernel(const SweepParams p) {
    using SW = Sweep<CPL, C64, BWD, NW, GS>;
    static_assert(!SGM_NAMED_RING || NW <= 17, "named ring barriers: ids 0..NW-2 must be < 16");
    // block-relative ring slots (needs the loop split into whole CPL blocks)
    // positions per unrolled block of the row loop (the backward sweep with 4 cells per lane
    // may unroll two CPL blocks, so that its S_fwd register prefetch can run 8 positions deep)
    constexpr int U = (BWD && CPL == 4 && SGM_TAIL_SPLIT) ? CPL * (GS ? SGM_BWD4_UNROLL_FINE : SGM_BWD4_UNROLL) : CPL;
    constexpr bool SB = SGM_SLOT_BASE && SGM_TAIL_SPLIT && (SW::RS % U == 0) && (SW::RING0 % U == 0);
    // band-handoff publication granularity (positions): measured best 8 for the forward
    // sweep, 4 for the backward sweep
    constexpr int PUB = (GS && SGM_FINE_PUB) ? SGM_FINE_PUB : (BWD ? 4 : kPublish);
    constexpr int R = SW::R;
    constexpr int DP = SW::DP;
    constexpr int VEC = SW::VEC;
    constexpr int RS = SW::RS;
    constexpr int G = SW::G;
    constexpr int RG = SW::RG;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint16_t *ring = reinterpret_cast<uint16_t *>(smem_raw);
    uint16_t *in0 = ring + size_t(NW - 1) * RS * VEC;
    constexpr int RING0 = SW::RING0;
    uint64_t *cbuf = reinterpret_cast<uint64_t *>(in0 + size_t(RING0) * VEC);
    uint16_t *wsc = reinterpret_cast<uint16_t *>(cbuf + size_t(NW) * 2 * SW::CEN);
    uint64_t *bars = reinterpret_cast<uint64_t *>(wsc + (BWD ? size_t(NW) * (DP + 4) : 0));
    // full[w][s]: slot s of warp w's ring holds complete data (32 producer lanes arrive)
    // empty[w][s]: the consumer (warp w+1) is done with slot s (32 consumer lanes arrive)
    // pub_full[k] / pub_empty[k]: band producer -> publisher warp handoff (kPubDepth deep)
    uint64_t *pub_full = bars + 2 * NW * RG;
    uint64_t *pub_empty = pub_full + kPubDepth;

    // Zero the path-vector rings: a zero vector with m = 0 makes the recursion return
    // L = C, i.e. every slot nobody writes acts as a path start.
    {
        uint4 *z = reinterpret_cast<uint4 *>(smem_raw);
        const int n16 = int((size_t(NW - 1) * RS + RING0) * VEC * 2 / 16);
        const uint32_t ps = uint32_t(p.P1) * 0x10001u;     // biased path-start vector
        for (int k = threadIdx.x; k < n16; k += (NW + 1) * 32) z[k] = make_uint4(ps, ps, ps, ps);
    }
    __shared__ int s_ticket;
    if (threadIdx.x < 2 * NW * RG) mbar_init(bars + threadIdx.x, 32);
    if (threadIdx.x < kPubDepth) {
        mbar_init(pub_full + threadIdx.x, 32);
        mbar_init(pub_empty + threadIdx.x, 1);
    }
    if (threadIdx.x == 0) s_ticket = atomicAdd(p.ticket, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    // Programmatic dependent launch: the backward sweep's CTAs may be scheduled once every
    // forward CTA has started (so they never hold an SM a forward CTA still needs); they
    // then wait per view on fwd_done, not for the whole forward grid.
    if (!BWD) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    // ticket -> (band, view): views in groups of p.vgroup, band-major inside a group, so
    // that band b+1 of a view starts about one band lag after band b (its handoff rows are
    // read while still in L2) and never before it (a band only waits for a running band)
#if SGM_UR_TICKET
    // through a warp reduction, so that the compiler knows band / view / row are warp-uniform
    const int ticket = int(__reduce_min_sync(0xffffffffu, unsigned(s_ticket)));
#else
    const int ticket = s_ticket;
#endif
    const int grp = ticket / (p.vgroup * p.nbands);
    const int v0 = grp * p.vgroup;
    const int gv = min(p.vgroup, p.nviews - v0);
    const int rem = ticket - v0 * p.nbands;
    const int band = rem / gv;
    const int view = v0 + rem - band * gv;

    // warp index through a warp reduction: the compiler then keeps it (and everything
    // derived from it) in uniform registers and emits uniform branches.
    const int wid = int(__reduce_min_sync(0xffffffffu, threadIdx.x >> 5));
    // row of the band this warp computes: the band's first (upstream) row runs on the
    // highest compute-warp id (the warp arbiter favours high warp ids, so upstream rows win
    // ties and downstream rows find their inputs ready: 6.79 -> 6.67 ms on 8 Driving quads).
    // For 8 cells per lane the same mapping behind a runtime-opaque select (p.one == 1)
    // compiles to a faster backward sweep (8 Wide quads 11.91 -> 11.34 ms; code generation,
    // measured: tools/ab_flags.sh)
    const int warp = (CPL == 8) ? ((wid == NW || p.one == 0) ? wid : NW - 1 - wid)
                                : (wid == NW ? wid : NW - 1 - wid);
    const int lane = lane_id();
    const int W = p.W, H = p.H;
    if (warp == NW) {
        // Publisher warp: turns the band producer's completed position groups into the
        // gpu-scope progress flag the next band polls.  The gpu-scope fence (a round trip
        // to L2) runs here, off the producer's critical path.  Causality: producer lanes'
        // gbuf stores -> mbarrier arrive (release.cta) -> wait here (acquire.cta) ->
        // fence.acq_rel.gpu -> flag store (cumulative release).
        // It also drops this band's consumed INPUT handoff lines from L2 (discard, no
        // write-back): once the band's last row has passed position q, warp 0 has long
        // copied input q into shared memory.  (Done here, off the compute warps: issued by
        // warp 0 itself the discards cost 1-12 % of the sweep.)
        if (band + 1 < p.nbands && !(p.debug_flags & 3)) {
            int *prog = p.progress + view * p.nbands + band;
            const char *gin_b = (band > 0 && !(p.debug_flags & 16)) ? reinterpret_cast<const char *>(
                                               p.gbuf + (long long)(view * p.nbands + band - 1) * W * (3 * DP))
                                         : nullptr;
            constexpr int kLinesPerPos = 3 * DP * 2 / 128;
            const int ngroups = (W + PUB - 1) / PUB;
            for (int k = 0; k < ngroups; ++k) {
#if SGM_PUB_SLEEP
                // back off between tests: a spinning publisher takes issue slots from the
                // compute warps of its SM sub-partition
                while (!mbar_test(pub_full + (k % kPubDepth), unsigned(k / kPubDepth) & 1u))
                    __nanosleep(SGM_PUB_SLEEP);
#else
                mbar_wait(pub_full + (k % kPubDepth), unsigned(k / kPubDepth) & 1u);
#endif
                asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
                if (lane == 0) {
                    st_relaxed_gpu(prog, min((k + 1) * PUB, W));
                    mbar_arrive(pub_empty + (k % kPubDepth));
                }
                if (gin_b != nullptr) {
                    const int q0 = k * PUB, nl = (min(q0 + PUB, W) - q0) * kLinesPerPos;
                    const char *g0 = gin_b + (long long)q0 * (3 * DP * 2);
                    for (int c = lane; c < nl; c += 32) discard_l2(g0 + 128 * c);
                }
                __syncwarp();
            }
        }
        return;
    }
    // this band's rows (runtime height <= NW, see band_geometry in api.cu)
    const int hb = p.band_q + (band < p.band_r ? 1 : 0);
    const int j = band * p.band_q + min(band, p.band_r) + warp;   // iteration row
    if (warp >= hb) return;                         // rows past the band
    const bool has_row_below = (warp < hb - 1) && !(p.debug_flags & 1);
    const int y = BWD ? (H - 1 - j) : j;
    // Bounded cross-CTA waits: a wait that times out (a scheduling or logic error, or the
    // debug flag 4) stores its fault code into p.err -- the next entry point of the handle
    // then fails with SGM_ERR_CUDA -- and the row runs to completion (so that every other
    // warp's waits still complete); that call's results are invalid.
    // (every lane stores the same code: a lane-0-only store would make the compiler treat
    // the warp as possibly diverged and wrap the later SHFL / CREDUX in WARPSYNC; nothing
    // of this state may stay live through the row loop: on 8 cells per lane the backward
    // sweep spills, 5.85 -> 7.06 ms on 8 Wide quads)
    const bool force_timeout = (p.debug_flags & 4) != 0;
    auto fault = [&](int code) {
        if (p.err != nullptr) *reinterpret_cast<volatile int *>(p.err) = code;
    };
    if (BWD) {
        // the view's forward sweep must be complete before this row reads S_fwd (the
        // S_fwd prefetch below runs before any other synchronisation)
        // every lane polls (one request per poll): a lane-0-only loop made the compiler
        // treat the warp as possibly diverged and wrap every later SHFL / CREDUX in
        // WARPSYNC (backward sweep 3.36 -> 4.85 ms)
        const int need = force_timeout ? H + 1 : H;
        bool done = false;
#pragma unroll 1
        for (int spins = 0; spins < (force_timeout ? (1 << 9) : (1 << 26)); ++spins) {
            done = __all_sync(0xffffffffu, ld_acquire_gpu(p.fwd_done + view) >= need);
            if (done) break;
            __nanosleep(256);
        }
        if (!done) fault(kFaultFwdDone);
    }

    const uint64_t *ref, *match;
    int mirror;
    if (p.explicit_mode) {
        ref = p.ref0; match = p.match0; mirror = p.mirror0;
    } else {
        const int pair = view >> 1, side = view & 1;
        const uint64_t *a = p.cen + (long long)(2 * pair) * p.cen_img_stride;
        const uint64_t *b = a + p.cen_img_stride;
        ref = side ? b : a;
        match = side ? a : b;
        mirror = side;
    }
    const long long yrow = (long long)y * W;
    const uint64_t *ref_row = ref + yrow;
    const uint64_t *match_row = match + yrow;
    auto X = [&](int xv) { return mirror ? (W - 1 - xv) : xv; };   // view x' -> image x
    auto xview = [&](int i) { return BWD ? (W - 1 - i) : i; };      // iteration i -> x'
    // S_fwd row in view coordinates; the backward sweep walks it from the right end
    uint16_t *sfwd_row = p.sfwd + (long long)view * p.sfwd_view_stride + yrow * DP + CPL * lane;
    const long long sstep = BWD ? -DP : DP;
    uint16_t *sfwd_ptr = sfwd_row + (BWD ? (long long)(W - 1) * DP : 0);

    // per-lane constants
    const uint32_t one = uint32_t(p.one);
    const uint32_t k10001 = one * 0x10001u, kneg10001 = one * 0xFFFEFFFFu;   // (SGM_UR_MB)
    // the forward sweep takes the u16x2 constants as kernel-parameter operands (c[] bank:
    // forward sweep 21.38 -> 21.03 ms on 64 quads); the backward sweep computes them into
    // registers (as parameters it measured slower: 21.32 -> 21.46 ms, Wide 5.29 -> 5.87 ms)
    constexpr bool kcp = SGM_CONST_PARAMS && !BWD;
    const uint32_t p1x2 = kcp ? p.k_p1x2 : uint32_t(p.P1) * 0x10001u;
    const uint32_t negp1x2 = kcp ? p.k_negp1x2 : (uint32_t(0x10000 - p.P1) & 0xFFFFu) * 0x10001u;   // -P1 per half
    const uint32_t p2mp1x2 = kcp ? p.k_p2mp1x2 : uint32_t(p.P2 - p.P1) * 0x10001u;                  // P2 - P1
    const uint32_t twop1x2 = kcp ? p.k_twop1x2 : 2u * p1x2;
    const uint32_t negb4 = kcp ? p.k_negb4 : 0u - 4u * p1x2;    // removes the 4 path biases from S
    const int dbase = CPL * lane;                  // the lane's u16 offset inside a vector
    // folded layout (path_update): register r holds disparities dlo + r (low half) and
    // dhi - r (high half)
    const int dlo = R * lane, dhi = DP - 1 - R * lane;
    constexpr bool has_pad = PAD;                  // D < Dp (template: no padding work otherwise)
    const uint32_t sel_fold = lane == 31 ? 0x5476u : 0x3210u;    // swap the halves at the fold
    const uint32_t ff_lane0 = lane == 0 ? 0xffffffffu : 0u;      // pair -1 does not exist
    uint32_t pad[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        pad[r] = (dlo + r >= p.D ? 0x1000u : 0u) | (dhi - r >= p.D ? 0x10000000u : 0u);
    }
    uint32_t dcode[R];   // bytes: d_lo, d_hi, 0, 0 (WTA keys)
#pragma unroll
    for (int r = 0; r < R; ++r) dcode[r] = uint32_t(dlo + r) | (uint32_t(dhi - r) << 8);

    // Ring layout (consumer-centric): slot s of a warp's ring holds, for the position q
    // with q & (kRing-1) == s, the three row-above vectors the consumer needs at q:
    //   v0 = L_down(q), v1 = L_diag(q-1) (predecessor of the (1,1) path),
    //   v2 = L_anti(q+1) (predecessor of the (-1,1) path).
    // The producer at position p writes v0 -> slot p, v1 -> slot p+1, v2 -> slot p-1, and
    // arrives on full[p-1] (its v2 is the last write into that slot).
    uint16_t *my_ring = ring + size_t(warp) * RS * VEC + dbase;
    const uint16_t *src_ring = (warp == 0 ? in0 : ring + size_t(warp - 1) * RS * VEC) + dbase;
    uint64_t *my_full = bars + size_t(warp) * RG;
    uint64_t *my_empty = bars + size_t(NW + warp) * RG;              // released by warp+1
    uint64_t *src_full = bars + size_t(warp - 1) * RG;               // (warp >= 1)
    uint64_t *src_empty = bars + size_t(NW + warp - 1) * RG;
    uint64_t *cref = cbuf + size_t(warp) * 128;
    uint64_t *cfresh = cref + 64;
    uint16_t *wta = wsc + size_t(warp) * (DP + 4);

    // band handoff (gbuf row has the same consumer-centric layout per position)
    const int nb_id = view * p.nbands + band;
    const bool has_consumer = band + 1 < p.nbands;
    const bool is_producer = (warp == hb - 1) && has_consumer && !(p.debug_flags & 3);
    uint16_t *gout = p.gbuf + (long long)nb_id * W * VEC + dbase;
    const uint16_t *gin = p.gbuf + (long long)(nb_id - 1) * W * VEC;
    // debug flag 4: poll a word nobody publishes (word 1 of the host-mapped fault block)
    const int *prog_in = (force_timeout && p.err != nullptr) ? p.err + 1 : p.progress + (nb_id - 1);
    const bool nodeps = (p.debug_flags & 1) != 0;
    const bool noband = (p.debug_flags & 2) != 0;   // debug: no inter-band handoff
    const bool band_input = (warp == 0) && band > 0 && !nodeps && !noband;
    const bool ring_input = warp > 0 && !nodeps;
    int known = 0;                                  // producer progress seen (warp 0)
    constexpr int kChunks = VEC * 2 / 16;           // 16-byte chunks per position

    // cp.async the band input of positions [hG, hG+G) (gbuf -> in0), one commit group
    // prefetch distance (groups): one group ahead in the forward sweep, two in the
    // backward sweep (measured: forward 3.29 -> 3.12 ms with 1; backward 3.36 -> 3.37)
    constexpr int LG = BWD ? ((RING0 / G - 1) > 2 ? 2 : (RING0 / G - 1)) : 1;
    auto issue_input = [&](int h) {
        const int q0 = h * G;
        if (q0 < W) {
            const int need = min(q0 + G + 1, W);    // gbuf[q] is complete once q+1 is done
            if (known < need) {
                int k, spins = 0;
                // bounded wait: a logic error must not hang the GPU (~>2 s of polling)
                const int cap = (p.debug_flags & 4) ? (1 << 8) : (1 << 25);
                while ((k = ld_relaxed_gpu(prog_in)) < need && ++spins < cap) __nanosleep(32);
                asm volatile("fence.acq_rel.gpu;\n" ::: "memory");   // acquire what k covers
                // a time-out stops all later waits and is reported after the row (reporting
                // it here, or raising `need` for the forced test, made the compiler wrap the
                // forward sweep's loop in 23 more convergence barriers: 3.12 -> 3.31 ms)
                known = __any_sync(0xffffffffu, k < need) ? (1 << 30) : k;
            }
            const char *g = reinterpret_cast<const char *>(gin + (long long)q0 * VEC) + 16 * lane;
#pragma unroll 1
            for (int q = q0; q < q0 + G && q < W; ++q, g += 2 * VEC) {
                char *sm = reinterpret_cast<char *>(in0 + size_t(q & (RING0 - 1)) * VEC) + 16 * lane;
#pragma unroll
                for (int c = 0; c < kChunks; c += 32)
                    if (c + lane < kChunks) cp_async16(sm + 16 * c, g + 16 * c);
            }
        }
        cp_async_commit();
    };

    // census prefetch: positions 0..63 (forward sweep only: the backward sweep reads the
    // matching cost the forward sweep packed into S_fwd)
    for (int k = lane; k < 64 && !BWD; k += 32) {
        if (k < W) {
            const int xv = xview(k);
            int xm = xv - (BWD ? DP - 1 : 0);
            xm = xm < 0 ? 0 : xm;
            cref[k] = __ldg(ref_row + X(xv));
            cfresh[k] = __ldg(match_row + X(xm));
        }
    }
    uint64_t stage_ref = 0, stage_fresh = 0;

    if (band_input) {
#pragma unroll 1
        for (int h = 0; h < LG; ++h) issue_input(h);
    }

    // state
    uint32_t Lh[R];
#pragma unroll
    for (int r = 0; r < R; ++r) Lh[r] = p1x2;                // path start (biased zero)
    using CW = typename std::conditional<C64, uint64_t, uint32_t>::type;
    // census windows of the two halves' disparity chains: lw[] holds census_match(x - d)
    // for d = dlo + r, hw[] for d = dhi - r (rotating slot indices, see the slide below)
    CW lw[R], hw[R];
#pragma unroll
    for (int k = 0; k < R; ++k) { lw[k] = 0; hw[k] = 0; }
    // BWD: S_fwd register prefetch PF positions ahead (slot = position mod PF must be a
    // compile-time index, so PF divides the unroll CPL)
    constexpr int PF = (CPL == 4) ? (U > CPL ? SGM_PF4U : SGM_PF4) : (CPL == 6) ? SGM_PF6 : (CPL == 8) ? SGM_PF8 : 2;
    static_assert(U % PF == 0, "the prefetch depth must divide the unrolled block");
    uint32_t pf[PF][R];
#pragma unroll
    for (int k = 0; k < PF; ++k)
#pragma unroll
        for (int r = 0; r < R; ++r) pf[k][r] = 0;
    if (BWD) {
#pragma unroll
        for (int k = 0; k < PF; ++k)
            if (k < W) VecIO<R>::ld(sfwd_ptr + k * sstep, pf[k]);
    }
    // BWD: WTA record of position (i - i mod kWtaPeriod) + lane, finished every kWtaPeriod positions
    constexpr int kWtaPeriod = (SGM_PER30 && SGM_TAIL_SPLIT && CPL == 6) ? 30 : 32;
    int pbase = 0;                                   // i0 mod kWtaPeriod (kWtaPeriod != 32 only)
    uint32_t rec_key = 0, rec_ac = 0;
    constexpr bool do_wta = BWD && !SOUT;
    constexpr bool do_sout = BWD && SOUT;
    int16_t *dint_row = do_wta ? p.dint + (long long)view * p.disp_view_stride + yrow : nullptr;
    float *dsub_row = do_wta ? p.dsub + (long long)view * p.disp_view_stride + yrow : nullptr;
    const int Dm1 = p.D - 1;
    __syncwarp();
    unsigned long long *trace = p.trace ? p.trace + (size_t(ticket) * (NW + 1) + warp) * 4 : nullptr;
    if (trace && lane == 0) {
        unsigned long long t;
        unsigned sm;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        trace[0] = t;
        trace[2] = sm;
    }

#if SGM_TAIL_SPLIT
    // one position of the row (ph = i mod CPL is a compile-time constant after unrolling)
    auto position = [&](const int i0, const int ph, const bool tail) {
        {
            const int i = i0 + ph;
#else
    constexpr bool tail = true;
#pragma unroll 1
    for (int i0 = 0; i0 < W; i0 += CPL) {
#pragma unroll
        for (int ph = 0; ph < CPL; ++ph) {
            const int i = i0 + ph;
            if (i >= W) break;
#endif
            const int xv = xview(i);
            // --- inputs of the row above
            if (band_input) {
                if (SGM_GIN_L2PF > 0 && ph == 0 && i + SGM_GIN_L2PF + CPL <= W) {
                    // the band above finished these handoff rows long ago (band-major tickets)
                    // and at large batches they have left L2: pull them back ahead of the
                    // cp.async that needs them
                    constexpr int kL = CPL * VEC * 2 / 128;
                    const char *a = reinterpret_cast<const char *>(gin + (long long)(i + SGM_GIN_L2PF) * VEC);
#pragma unroll
                    for (int c = 0; c < kL; c += 32)
                        if (c + lane < kL) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a + 128 * (c + lane)));
                }
                if ((ph % G) == 0) {                   // group start: keep LG groups in flight
                    issue_input(i / G + LG);
                    cp_async_wait<LG>();
                    __syncwarp();
                }
            } else if (ring_input && (ph % G) == 0) {
                const int g = i / G;                       // group start: wait for slots
                if (SGM_NAMED_RING == 2) {
                    // blocking wait for the producer's arrival g, then tell it sync g passed
                    named_sync(warp - 1, 64);
                    mbar_arrive(src_empty);
                } else if (SGM_NAMED_RING) {
                    named_sync(warp - 1, 64);                  // rendezvous g
                }
                else mbar_wait(src_full + (g % RG), unsigned(g / RG) & 1u);
            }
            // --- census prefetch refill (i0 is a multiple of CPL: with CPL | 16 only the first
            // position of a block can be a refill point)
            constexpr bool rf_first = SGM_REFILL_FIRST && (16 % CPL == 0);
            if (BWD) {
            } else if ((!rf_first || ph == 0) && (i & 31) == 0) {
                const int q = min(i + 32 + lane, W - 1);   // clamped: keeps the loads unpredicated
                {
                    const int xq = xview(q);
                    int xm = xq - (BWD ? DP - 1 : 0);
                    xm = xm < 0 ? 0 : xm;
                    stage_ref = __ldg(ref_row + X(xq));
                    stage_fresh = __ldg(match_row + X(xm));
                }
            } else if ((!rf_first || ph == 0) && (i & 31) == 16) {
                const int q = i + 16 + lane;
                if (q < W) {
                    cref[q & 63] = stage_ref;
                    cfresh[q & 63] = stage_fresh;
                }
                __syncwarp();
            }
            // --- slide the census windows by one position: cell d takes cell d-1's value.
            // Low chain (d = dlo + r, logical r in slot (r - ph) mod R): enters at r = 0
            // from lane l-1 (lane 0: the fresh census), leaves at r = R-1.  High chain
            // (d = dhi - r, logical r in slot (r + ph) mod R): enters at r = R-1 from lane
            // l+1 (lane 31: its own low chain's outgoing d = Dp/2-1), leaves at r = 0.
            if (!BWD) {
                const uint64_t fresh = cfresh[i & 63];
                const int ql = (2 * R - ph) % R;
                const int qh = (ph + R - 1) % R;
                const CW out_lo = lw[ql];
                const CW vl = __shfl_up_sync(0xffffffffu, out_lo, 1);
                const CW vh = __shfl_down_sync(0xffffffffu, hw[qh], 1);
                lw[ql] = lane == 0 ? CW(fresh) : vl;
                hw[qh] = lane == 31 ? out_lo : vh;
            }
            // --- matching cost C(x', d) for the lane's CPL cells.  The forward sweep
            // computes it from the census window; the backward sweep unpacks it from the
            // S_fwd word the forward sweep stored: word = S_fwd << 6 | C (S_fwd <= 4 *
            // (C_max + P2) <= 1020 < 2^10, C <= C_max <= 63 < 2^6; sgm_create enforces both).
            uint32_t C[R], craw[R], Sf[R];
            if (BWD) {
                const int slot = ph % PF;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    craw[r] = pf[slot][r] & 0x003F003Fu;
                    Sf[r] = (pf[slot][r] >> 6) & 0x03FF03FFu;
                    C[r] = PAD ? craw[r] + pad[r] : craw[r];
                }
                // unconditional load: a predicated load would make the compiler copy the
                // result into the slot at once and stall on it.  Past the row's end it reads
                // the row before (or the allocation's front guard); the value is never used.
                VecIO<R>::ld(sfwd_ptr + PF * sstep, pf[slot]);
                constexpr int L2PF = (CPL == 4) ? SGM_L2PF4 : (CPL == 6) ? SGM_L2PF6 : (CPL == 8) ? SGM_L2PF8 : 0;
                // once per block: lanes 0 .. (lines per block - 1) pull the block SGM_L2PF
                // positions ahead into L2 (past the row's start it touches the row before or
                // the front guard: harmless)
                if (L2PF > 0 && ph % CPL == SGM_L2PF_PH) {
#if SGM_L2PF_BULK
                    // one bulk prefetch (a single lane's instruction) for the whole block
                    const char *a = reinterpret_cast<const char *>(sfwd_ptr - CPL * lane + (L2PF + CPL - 1) * sstep);
                    if (lane == 0)
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a), "n"(CPL * DP * 2));
#else
                    constexpr int kLines = CPL * DP * 2 / 128;
                    const char *a = reinterpret_cast<const char *>(sfwd_ptr - CPL * lane + L2PF * sstep) +
                                    (BWD ? -128 * lane + (DP * 2 - 128) : 128 * lane);
                    if (lane < kLines) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a));
#endif
                }
                sfwd_ptr += sstep;
            } else {
                const uint64_t rv = cref[i & 63];
                uint32_t c[CPL];                           // c[2r]: d = dlo + r, c[2r+1]: d = dhi - r
#pragma unroll
                for (int jj = 0; jj < CPL; ++jj) {
                    const int r = jj >> 1;
                    const CW w = (jj & 1) ? hw[(r + ph) % R] : lw[(r - ph + 2 * R) % R];
                    if (C64) {
                        const uint64_t x = rv ^ uint64_t(w);
                        c[jj] = imad(uint32_t(__popc(uint32_t(x))), one, uint32_t(__popc(uint32_t(x >> 32))));
                    } else {
                        c[jj] = __popc(uint32_t(rv) ^ uint32_t(w));
                    }
                }
                if (xv < Dm1) {                            // border: x' - d < 0 -> C_max
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        if (dlo + r > xv) c[2 * r] = uint32_t(p.cmax);
                        if (dhi - r > xv) c[2 * r + 1] = uint32_t(p.cmax);
                    }
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    craw[r] = imad(c[2 * r + 1], 0x10000u, c[2 * r]);
                    C[r] = PAD ? craw[r] + pad[r] : craw[r];
                }
            }
            // --- row-above predecessors: all three live in slot i
            uint32_t pv[3][R];
            {
                // block-relative slots (SB): i0 is a multiple of CPL and CPL divides the ring
                const int msk = band_input || warp == 0 ? RING0 - 1 : RS - 1;
                const uint16_t *src = src_ring + size_t(SB ? (i0 & msk) + ph : (i & msk)) * VEC;
#pragma unroll
                for (int v = 0; v < 3; ++v) VecIO<R>::ld(src + v * DP, pv[v]);
            }
            if (!SGM_NAMED_RING && ring_input && (ph % G) == G - 1) {   // group end: release its slots
                __syncwarp();
                mbar_arrive(src_empty + ((i / G) % RG));
            }
            // --- the four path updates (->, down, two diagonals)
            uint32_t S[R];
            {
                uint32_t nL[R];
                path_update<R>(Lh, C, nL, negp1x2, p2mp1x2, twop1x2, sel_fold, ff_lane0, k10001, kneg10001);
#pragma unroll
                for (int r = 0; r < R; ++r) { Lh[r] = nL[r]; S[r] = nL[r]; }
            }
            uint32_t nv[3][R];
#pragma unroll
            for (int v = 0; v < 3; ++v)
                path_update<R>(pv[v], C, nv[v], negp1x2, p2mp1x2, twop1x2, sel_fold, ff_lane0, k10001, kneg10001);
            // S = sum of the four unbiased path costs: the -4 P1 rides in IADD3's third slot
#pragma unroll
            for (int r = 0; r < R; ++r) S[r] = (S[r] + nv[0][r] + nv[1][r]) + (nv[2][r] + negb4);
            // --- hand the three vectors to the row below
            if (has_row_below) {
                if (!SGM_NAMED_RING && (ph % G) == G - 1) {   // next group's slots free again?
                    const int h = i / G + 1;
                    if (h >= RG) mbar_wait(my_empty + (h % RG), unsigned(h / RG - 1) & 1u);
                }
                {
                    const int sb = i0 & (RS - 1);
                    const int s0 = SB ? sb + ph : (i & (RS - 1));
                    const int s1 = SB ? ((ph == U - 1) ? ((i0 + U) & (RS - 1)) : sb + ph + 1) : ((i + 1) & (RS - 1));
                    const int s2 = SB ? ((ph == 0) ? ((i0 - 1) & (RS - 1)) : sb + ph - 1) : ((i - 1) & (RS - 1));
                    VecIO<R>::st(my_ring + size_t(s0) * VEC, nv[0]);
                    VecIO<R>::st(my_ring + size_t(s1) * VEC + DP, nv[1]);
                    VecIO<R>::st(my_ring + size_t(s2) * VEC + 2 * DP, nv[2]);
                }
                if (SGM_NAMED_RING == 2) {
                    // arrival n = i/G - 1 once position (n + 1) G is stored, after the consumer
                    // passed its sync n - 1 (at most one arrival pending per barrier id)
                    if ((ph % G) == 0 && i >= G) {
                        const int n = i / G - 1;
                        if (n >= 1) mbar_wait(my_empty, unsigned(n - 1) & 1u);
                        named_arrive(warp, 64);
                    }
                } else if (SGM_NAMED_RING) {
                    // rendezvous n = i/G - 1 - lead once position (n + 1 + lead) G is stored
                    if ((ph % G) == 0 && i >= (1 + SGM_NAMED_LEAD) * G) named_sync(warp, 64);
                } else if ((ph % G) == 0 && i > 0) {
                    mbar_arrive(my_full + ((i / G - 1) % RG));   // group done
                }
            } else if (is_producer) {
                uint16_t *g = gout + (long long)i * VEC;
                uint32_t zero[R];
#pragma unroll
                for (int r = 0; r < R; ++r) zero[r] = p1x2;        // biased path start
                VecIO<R>::st(g, nv[0]);
                if (i + 1 < W) VecIO<R>::st(g + VEC + DP, nv[1]);
                if (i > 0) VecIO<R>::st(g - VEC + 2 * DP, nv[2]);
                if (i == 0) VecIO<R>::st(g + DP, zero);            // no (i-1) predecessor
                if (i == W - 1) VecIO<R>::st(g + 2 * DP, zero);    // no (i+1) predecessor
                if ((i + 1) % PUB == 0 || i == W - 1) {            // hand group k to the publisher
                    const int k = i / PUB;
                    if (k >= kPubDepth)
                        mbar_wait(pub_empty + (k % kPubDepth), unsigned(k / kPubDepth - 1) & 1u);
                    mbar_arrive(pub_full + (k % kPubDepth));
                }
            }
            // --- sweep output
            if (!BWD) {
                uint32_t w[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    // padded disparities (d >= D) carry huge sums: saturate them to 10 bits,
                    // the backward sweep re-applies the padding cost anyway
                    const uint32_t sv = has_pad ? __vminu2(S[r], 0x03FF03FFu) : S[r];
                    w[r] = imad(sv, 64u, craw[r]);
                }
                VecIO<R>::st(sfwd_ptr, w);
                sfwd_ptr += sstep;
            } else {
                uint32_t St[R];
#pragma unroll
                for (int r = 0; r < R; ++r) St[r] = S[r] + Sf[r];
                if (do_sout) {
                    const int x = X(xv);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        uint16_t *o = p.sout + ((long long)y * W + x) * p.D;
                        if (dlo + r < p.D) o[dlo + r] = uint16_t(St[r] & 0xffffu);
                        if (dhi - r < p.D) o[dhi - r] = uint16_t(St[r] >> 16);
                    }
                }
                if (do_wta) {
                    // smallest-index argmin via min of (S << 8 | d) (G10)
                    uint32_t best = 0xffffffffu;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const uint32_t k0 = __byte_perm(St[r], dcode[r], 0x6104);
                        const uint32_t k1 = __byte_perm(St[r], dcode[r], 0x7325);
                        best = min(best, min(k0, k1));
                    }
                    const uint32_t bkey = __reduce_min_sync(0xffffffffu, best);
                    const int dstar = int(bkey & 0xffu);
#if SGM_WTA_SHFL
                    // S(d*-1), S(d*+1) straight from the registers of the lanes holding them:
                    // d lies in pair k = min(d, Dp-1-d) (low half iff d < Dp/2), register k mod
                    // R of lane k / R (values at d* = 0 / Dp-1 are never used)
                    auto s_at = [&](int d) -> uint32_t {
                        const bool lo = d < DP / 2;
                        const int k = lo ? d : DP - 1 - d;
                        const int kl = k / R, kr = k - kl * R;
                        uint32_t v = St[0];
#pragma unroll
                        for (int r = 1; r < R; ++r) v = (kr == r) ? St[r] : v;
                        v = __shfl_sync(0xffffffffu, v, kl & 31);
                        return lo ? (v & 0xffffu) : (v >> 16);
                    };
                    const uint32_t sa = s_at(dstar - 1);
                    const uint32_t sc = s_at(dstar + 1);
#else
                    __syncwarp();                                // previous reads of wta done
#pragma unroll
                    for (int r = 0; r < R; ++r) {           // natural disparity order
                        wta[2 + dlo + r] = uint16_t(St[r]);
                        wta[2 + dhi - r] = uint16_t(__umulhi(St[r], 0x10000u));
                    }
                    __syncwarp();
                    // S(d*-1), S(d*+1): one guard entry each side, no clamping (unused at
                    // d* = 0 / Dp-1)
                    const uint32_t sa = wta[dstar + 1];
                    const uint32_t sc = wta[dstar + 3];
#endif
                    // WTA record slot of this position: i mod kWtaPeriod (pbase = i0 mod period)
                    const int sl = (kWtaPeriod == 32) ? (i & 31) : pbase + ph;
                    if (lane == sl) { rec_key = bkey; rec_ac = sa | (sc << 16); }
                    // every 32 positions each lane finishes one pixel: the parabola
                    // sub-pixel (one IEEE division per lane) and the stores
                    // (whole blocks with CPL | 32: only their last position can be one)
                    constexpr bool fin_last = SGM_FIN_LAST && SGM_TAIL_SPLIT && (kWtaPeriod % U == 0);
                    if ((!fin_last || tail || ph == U - 1) && (sl == kWtaPeriod - 1 || i == W - 1)) {
                        if (lane <= sl) {
                            const int d = int(rec_key & 0xffu);
                            const int b = int(rec_key >> 8);
                            const int a = int(rec_ac & 0xffffu), c = int(rec_ac >> 16);
                            float sub = float(d);
                            if (d > 0 && d < Dm1) {
                                const int den = 2 * (a + c - 2 * b);
                                float off = 0.f;
                                if (den != 0) off = __fdiv_rn(float(a - c), float(den));
                                off = fminf(fmaxf(off, -0.5f), 0.5f);
                                sub = __fadd_rn(float(d), off);
                            }
                            const int xo = X(xview((i - sl) + lane));
                            dint_row[xo] = int16_t(d);
                            dsub_row[xo] = sub;
                        }
                    }
                }
            }
        }
    }
#if SGM_TAIL_SPLIT
    ;
    // whole CPL-position blocks without a per-position bound check, then the tail
    const int Wfull = W - W % U;
#pragma unroll 1
    for (int i0 = 0; i0 < Wfull; i0 += U) {
#pragma unroll
        for (int ph = 0; ph < U; ++ph) position(i0, ph, false);
        if (BWD && kWtaPeriod != 32) pbase = (pbase + CPL == kWtaPeriod) ? 0 : pbase + CPL;
    }
    if (Wfull < W) {
#pragma unroll
        for (int ph = 0; ph < U - 1; ++ph)
            if (Wfull + ph < W) position(Wfull, ph, true);
    }
#endif
    if (has_row_below) {
        // position W lies outside the image: the (-1,1) path of the row below starts at
        // x' = W-1, so that slot's v2 must read as zero; then release slot W-1.
        uint32_t zero[R];
#pragma unroll
        for (int r = 0; r < R; ++r) zero[r] = p1x2;                // biased path start
        VecIO<R>::st(my_ring + size_t((W - 1) & (RS - 1)) * VEC + 2 * DP, zero);
        if (SGM_NAMED_RING == 2) {
            const int ng = (W + G - 1) / G;
            for (int n = (W - 1) / G; n < ng; ++n) {
                if (n >= 1) mbar_wait(my_empty, unsigned(n - 1) & 1u);
                named_arrive(warp, 64);
            }
        } else if (SGM_NAMED_RING) {
            // the consumer meets ceil(W / G) rendezvous; the loop made floor((W-1)/G) - lead
            const int ng = (W + G - 1) / G;
            int done = (W - 1) / G - SGM_NAMED_LEAD;
            for (done = done < 0 ? 0 : done; done < ng; ++done) named_sync(warp, 64);
        } else {
            mbar_arrive(my_full + (((W - 1) / G) % RG));
        }
    }
    if (band_input) cp_async_wait<0>();
    if (band_input && known >= (1 << 30)) fault(kFaultBandInput);
    if (!BWD) {                                     // this row's S_fwd is complete
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAdd(p.fwd_done + view, 1);
        }
    }
    if (trace && lane == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        trace[1] = t;
    }
}

// The two sweeps of one call.  Sync buffer (zeroed once, before the forward launch):
//   [ticket, progress[nviews*nbands]] forward, the same for the backward sweep, fwd_done[nviews]
// and the band-handoff buffer is split in two, so that the backward sweep (launched with
// programmatic stream serialisation) can overlap the forward sweep's last wave.
template <int CPL, bool C64, int NW, bool PAD, int GS>
cudaError_t launch_pair(const SweepParams &p, bool debug_s, cudaStream_t st, cudaEvent_t ev_mid_a,
                        cudaEvent_t ev_mid_b, int *launches, int *sync_buf, size_t sync_bytes) {
    (void)debug_s;
    const dim3 grid(p.nviews * p.nbands), block((NW + 1) * 32);
    const size_t per = 1 + size_t(p.nviews) * p.nbands;
    SweepParams pf = p, pb = p;
    pf.ticket = sync_buf; pf.progress = sync_buf + 1;
    pb.ticket = sync_buf + per; pb.progress = sync_buf + per + 1;
    pf.fwd_done = pb.fwd_done = sync_buf + 2 * per;
    pb.gbuf = p.gbuf + size_t(p.nviews) * p.nbands * size_t(p.W) * 3 * p.Dp;
    cudaError_t e;
    if ((e = cudaMemsetAsync(sync_buf, 0, sync_bytes, st)) != cudaSuccess) return e;
    {
        constexpr size_t sm = Sweep<CPL, C64, false, NW, GS>::smem_bytes();
        auto k = sweep_kernel<CPL, C64, false, NW, PAD, false, GS>;
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm))) != cudaSuccess) return e;
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) != cudaSuccess) return e;
        k<<<grid, block, sm, st>>>(pf);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (launches) ++*launches;
    }
    if (ev_mid_a) cudaEventRecord(ev_mid_a, st);    // (timing mode: no overlap)
    if (ev_mid_b) cudaEventRecord(ev_mid_b, st);
    {
        constexpr size_t sm = Sweep<CPL, C64, true, NW, GS>::smem_bytes();   // same for PAD
        // the backward sweep keeps the general (padded) cost unpack: specialising it for
        // D = Dp measured slower (3.78 -> 3.94 ms on 8 Driving quads; code scheduling)
        auto k = p.sout ? sweep_kernel<CPL, C64, true, NW, true, true, GS> : sweep_kernel<CPL, C64, true, NW, true, false, GS>;
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm))) != cudaSuccess) return e;
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) != cudaSuccess) return e;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = block;
        cfg.dynamicSmemBytes = sm;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if ((e = cudaLaunchKernelEx(&cfg, k, pb)) != cudaSuccess) return e;
        if (launches) ++*launches;
    }
    return cudaSuccess;
}

}  // namespace

int sweep_warps_for(int cpl) { (void)cpl; return kBandRowsMax; }
// [ticket, progress[nviews*nbands]] x 2 sweeps, fwd_done[nviews]
size_t sweep_sync_ints(int nviews, int nbands) { return 2 * (1 + size_t(nviews) * nbands) + size_t(nviews); }

cudaError_t launch_sweeps(const SweepParams &p, int cpl, bool c64, int nw, bool debug_s,
                          cudaStream_t st, cudaEvent_t mid_ev_a, cudaEvent_t mid_ev_b,
                          int *launches) {
    // the call's sync buffer starts at p.ticket (layout: launch_pair)
    int *sync_buf = p.ticket;
    const size_t sync_bytes = sizeof(int) * sweep_sync_ints(p.nviews, p.nbands);
    if (nw != sweep_warps_for(cpl)) return cudaErrorInvalidValue;
#define SGM_PAIR(CPL_, C64_, PAD_, GS_)                                                        \
    launch_pair<CPL_, C64_, kBandRowsMax, PAD_, GS_>(p, debug_s, st, mid_ev_a, mid_ev_b, launches, \
                                                   sync_buf, sync_bytes)
    // latency mode (fewer than two waves of CTAs: each view's band chain is the critical
    // path): CPL <= 4 rows meet every kFineGroup positions instead of every CPL (a shorter
    // row-to-row lag shortens the chain)
#define SGM_CASE(CPL_, C64_)                                                                   \
    if (cpl == CPL_ && c64 == C64_) {                                                          \
        constexpr int gf = (CPL_ <= 4 || SGM_FINE_ALL) ? kFineGroup : 0;                       \
        if (p.D < 32 * CPL_)                                                                   \
            return p.fine_sync && gf ? SGM_PAIR(CPL_, C64_, true, gf) : SGM_PAIR(CPL_, C64_, true, 0); \
        return p.fine_sync && gf ? SGM_PAIR(CPL_, C64_, false, gf) : SGM_PAIR(CPL_, C64_, false, 0);   \
    }
    SGM_CASE(2, false) SGM_CASE(2, true) SGM_CASE(4, false) SGM_CASE(4, true)
    SGM_CASE(6, false) SGM_CASE(6, true) SGM_CASE(8, false) SGM_CASE(8, true)
#undef SGM_PAIR
#undef SGM_CASE
    return cudaErrorInvalidValue;
}

}  // namespace sgm
