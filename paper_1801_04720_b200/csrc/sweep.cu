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
//  * One warp owns one image row; lane l owns the contiguous disparities
//    d = CPL*l .. CPL*l+CPL-1 as CPL/2 packed u16x2 registers.  A path update is
//    DPX min-plus: VIMNMX.U16x2 / VIADDMNMX.U16x2, neighbours d+-1 by PRMT plus one
//    SHFL each way, min over d by VIMNMX + CREDUX.MIN (__reduce_min_sync), and the
//    normalisation "+C - m" is a single IADD3 with a two's-complement constant.
//  * The cost C is recomputed on the fly from the census windows (never stored); the
//    window of census_match values slides one position per step by one SHFL.
//  * Rows of a CTA run as a skewed wavefront: warp w processes position t - 2w at
//    lockstep step t, so its three row-above predecessors (x-1, x, x+1) were produced
//    at least one step earlier.  Row-above path vectors pass through a 4-slot shared
//    memory ring per warp pair.  CTAs own bands of NW rows; the band's last row hands
//    its vectors to the next band's CTA through global memory with a progress flag
//    (release/acquire at gpu scope), prefetched by cp.async 8 positions ahead.  CTAs
//    take tickets (atomicAdd) so a band only ever waits for an already-running band.
#include <type_traits>

#include "sgm_internal.cuh"

namespace sgm {
namespace {

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
__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu(int *p, int v) {
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// One semi-global path update for the CPL cells a lane holds.
//   prev: L_r(p - r, .) (u16x2 pairs), C: C(p, .), out: L_r(p, .).
template <int R>
__device__ __forceinline__ void path_update(const uint32_t (&prev)[R], const uint32_t (&C)[R],
                                            uint32_t (&out)[R], uint32_t p1x2, uint32_t p2x2,
                                            int lane) {
    // m = min_k L_r(p - r, k), broadcast as m * 0x10001
    uint32_t v = prev[0];
#pragma unroll
    for (int r = 1; r < R; ++r) v = __vminu2(v, prev[r]);
    v = __vminu2(v, __byte_perm(v, 0, 0x1032));
    const uint32_t mm = __reduce_min_sync(0xffffffffu, v);
    const uint32_t mP2 = mm + p2x2;      // m + P2 in both halves
    const uint32_t K = 0u - mm;          // adds -m to both halves (carry-exact)
    // neighbours d-1 / d+1
    uint32_t up = __shfl_up_sync(0xffffffffu, prev[R - 1], 1);
    uint32_t dn = __shfl_down_sync(0xffffffffu, prev[0], 1);
    up = lane == 0 ? kSent : up;
    dn = lane == 31 ? kSent : dn;
    uint32_t nb[R + 1];
    nb[0] = __byte_perm(up, prev[0], 0x5432);
#pragma unroll
    for (int r = 1; r < R; ++r) nb[r] = __byte_perm(prev[r - 1], prev[r], 0x5432);
    nb[R] = __byte_perm(prev[R - 1], dn, 0x5432);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        uint32_t t = __vminu2(nb[r], nb[r + 1]);       // min(L(d-1), L(d+1))
        t = __viaddmin_u16x2(t, p1x2, prev[r]);        // min(.. + P1, L(d))
        t = __vminu2(t, mP2);                          // min(.., m + P2)
        out[r] = t + C[r] + K;                         // + C - m
    }
}

template <int CPL, bool C64, bool BWD, int NW>
struct Sweep {
    static constexpr int R = CPL / 2;
    static constexpr int DP = 32 * CPL;
    static constexpr int VEC = 3 * DP;             // u16 per ring slot (3 path vectors)

    static constexpr size_t smem_bytes() {
        size_t b = 0;
        b += size_t(NW) * kRing * VEC * 2;          // ring
        b += size_t(kRing0) * VEC * 2;              // band input ring
        b += size_t(NW) * 2 * 64 * 8;               // census prefetch (ref, fresh)
        if (BWD) {
            b += size_t(NW) * DP * 2;               // WTA scratch
        }
        return b;
    }
};

template <int CPL, bool C64, bool BWD, int NW>
__global__ void __launch_bounds__(NW * 32, 1) sweep_kernel(const SweepParams p) {
    using SW = Sweep<CPL, C64, BWD, NW>;
    constexpr int R = SW::R;
    constexpr int DP = SW::DP;
    constexpr int VEC = SW::VEC;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint16_t *ring = reinterpret_cast<uint16_t *>(smem_raw);
    uint16_t *in0 = ring + size_t(NW) * kRing * VEC;
    uint64_t *cbuf = reinterpret_cast<uint64_t *>(in0 + size_t(kRing0) * VEC);
    uint16_t *wsc = reinterpret_cast<uint16_t *>(cbuf + size_t(NW) * 2 * 64);

    __shared__ int s_ticket;
    if (threadIdx.x == 0) s_ticket = atomicAdd(p.ticket, 1);
    __syncthreads();
    const int ticket = s_ticket;
    const int band = ticket / p.nviews;
    const int view = ticket - band * p.nviews;

    const int warp = threadIdx.x >> 5;
    const int lane = lane_id();
    const int W = p.W, H = p.H;
    const int j = band * NW + warp;                 // iteration row
    const bool row_ok = j < H;
    const int y = BWD ? (H - 1 - j) : j;

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
    const long long yrow = (long long)(row_ok ? y : 0) * W;
    const uint64_t *ref_row = ref + yrow;
    const uint64_t *match_row = match + yrow;
    uint16_t *sfwd_row = p.sfwd + (long long)view * p.sfwd_view_stride + yrow * DP;
    auto X = [&](int xv) { return mirror ? (W - 1 - xv) : xv; };   // view x' -> image x
    auto xview = [&](int i) { return BWD ? (W - 1 - i) : i; };      // iteration i -> x'

    // per-lane constants
    const uint32_t p1x2 = uint32_t(p.P1) * 0x10001u;
    const uint32_t p2x2 = uint32_t(p.P2) * 0x10001u;
    const int dbase = CPL * lane;
    uint32_t pad[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        pad[r] = (dbase + 2 * r >= p.D ? 0x1000u : 0u) | (dbase + 2 * r + 1 >= p.D ? 0x10000000u : 0u);
    }
    uint32_t dcode[R];   // bytes: d_lo, d_hi, 0, 0 (WTA keys)
#pragma unroll
    for (int r = 0; r < R; ++r) dcode[r] = uint32_t(dbase + 2 * r) | (uint32_t(dbase + 2 * r + 1) << 8);

    // shared-memory views of this warp
    uint16_t *my_ring = ring + size_t(warp) * kRing * VEC;
    const uint16_t *src_ring = warp == 0 ? in0 : ring + size_t(warp - 1) * kRing * VEC;
    const int src_mask = warp == 0 ? (kRing0 - 1) : (kRing - 1);
    const bool have_above = j > 0;                  // row j-1 exists in the view
    uint64_t *cref = cbuf + size_t(warp) * 128;
    uint64_t *cfresh = cref + 64;
    uint16_t *wta = wsc + size_t(warp) * DP;

    // band handoff
    const int nb_id = view * p.nbands + band;
    const bool has_consumer = band + 1 < p.nbands;
    const bool is_producer = (warp == NW - 1) && has_consumer;
    uint16_t *gout = p.gbuf + (long long)nb_id * W * VEC;
    const uint16_t *gin = p.gbuf + (long long)(nb_id - 1) * W * VEC;
    int *prog_out = p.progress + nb_id;
    const int *prog_in = p.progress + (nb_id - 1);
    const bool band_input = (warp == 0) && band > 0;
    int known = 0;                                  // producer progress seen (warp 0)
    constexpr int kChunks = VEC * 2 / 16;           // 16-byte chunks per position

    auto issue_input = [&](int q) {                 // cp.async position q of the row above
        if (q < W) {
            if (known < q + 1) {
                int k, spins = 0;
                // bounded wait: a logic error must not hang the GPU (~>2 s of polling)
                while ((k = ld_acquire_gpu(prog_in)) < q + 1 && ++spins < (1 << 25)) __nanosleep(64);
                known = k;
            }
            const char *g = reinterpret_cast<const char *>(gin + (long long)q * VEC);
            char *s = reinterpret_cast<char *>(in0 + size_t(q & (kRing0 - 1)) * VEC);
#pragma unroll
            for (int c = lane; c < kChunks; c += 32) cp_async16(s + 16 * c, g + 16 * c);
        }
        cp_async_commit();
    };

    // census prefetch: positions 0..63
    auto census_fill = [&](int i0, int n) {
        for (int k = lane; k < n; k += 32) {
            const int i = i0 + k;
            if (i < W) {
                const int xv = xview(i);
                int xm = xv - (BWD ? DP - 1 : 0);
                xm = xm < 0 ? 0 : xm;
                cref[i & 63] = __ldg(ref_row + X(xv));
                cfresh[i & 63] = __ldg(match_row + X(xm));
            }
        }
    };
    if (row_ok) census_fill(0, 64);
    uint64_t stage_ref = 0, stage_fresh = 0;

    if (band_input) {
#pragma unroll 1
        for (int q = 0; q < kLook; ++q) issue_input(q);
    }

    // state
    uint32_t Lh[R];
#pragma unroll
    for (int r = 0; r < R; ++r) Lh[r] = 0;
    using CW = typename std::conditional<C64, uint64_t, uint32_t>::type;
    CW win[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) win[k] = 0;
    uint32_t pf[2][R];                               // BWD: S_fwd prefetch (2 positions)
#pragma unroll
    for (int r = 0; r < R; ++r) { pf[0][r] = 0; pf[1][r] = 0; }
    if (BWD && row_ok) {
        VecIO<R>::ld(sfwd_row + (long long)xview(0) * DP + dbase, pf[0]);
        if (W > 1) VecIO<R>::ld(sfwd_row + (long long)xview(1) * DP + dbase, pf[1]);
    }
    int od = 0;
    float os = 0.f;
    const bool do_wta = BWD && p.dint != nullptr;
    const bool do_sout = BWD && p.sout != nullptr;
    int16_t *dint_row = do_wta ? p.dint + (long long)view * p.disp_view_stride + yrow : nullptr;
    float *dsub_row = do_wta ? p.dsub + (long long)view * p.disp_view_stride + yrow : nullptr;

    __syncwarp();
    __syncthreads();

    const int T = W + 2 * (NW - 1);
#pragma unroll 1
    for (int t0 = 0; t0 < T; t0 += CPL) {
#pragma unroll
        for (int ph = 0; ph < CPL; ++ph) {
            const int t = t0 + ph;
            const int i = t - 2 * warp;
            const bool active = row_ok && i >= 0 && i < W;

            // --- band output publication (producer warp, before this step's stores)
            if (is_producer) {
                const int c = t - 2 * (NW - 1);
                if (c >= 1 && c <= W && ((c % kPublish) == 0 || c == W)) {
                    __threadfence();
                    if (lane == 0) st_relaxed_gpu(prog_out, c);
                }
            }
            if (active) {
                const int xv = xview(i);
                // --- band input: keep cp.async kLook positions ahead
                if (band_input) {
                    issue_input(i + kLook);
                    cp_async_wait<kLook - 1>();
                    __syncwarp();
                }
                // --- census prefetch refill
                if ((i & 31) == 0) {
                    const int q = i + 32 + lane;
                    if (q < W) {
                        const int xq = xview(q);
                        int xm = xq - (BWD ? DP - 1 : 0);
                        xm = xm < 0 ? 0 : xm;
                        stage_ref = __ldg(ref_row + X(xq));
                        stage_fresh = __ldg(match_row + X(xm));
                    }
                } else if ((i & 31) == 16) {
                    const int q = i + 16 + lane;
                    if (q < W) {
                        cref[q & 63] = stage_ref;
                        cfresh[q & 63] = stage_fresh;
                    }
                    __syncwarp();
                }
                // --- BWD window initialisation (logical j <-> cm(W - d) before rotation)
                if (BWD && i == 0) {
#pragma unroll
                    for (int jj = 0; jj < CPL; ++jj) {
                        int xm = W - (dbase + jj);
                        xm = xm < 0 ? 0 : (xm > W - 1 ? W - 1 : xm);
                        const uint64_t v = __ldg(match_row + X(xm));
                        win[(jj + ph - 1 + CPL) % CPL] = CW(v);
                    }
                }
                // --- slide the census window by one position
                {
                    const uint64_t fresh = cfresh[i & 63];
                    if (!BWD) {
                        const int q = (CPL - ph) % CPL;       // outgoing logical CPL-1
                        CW v = __shfl_up_sync(0xffffffffu, win[q], 1);
                        win[q] = lane == 0 ? CW(fresh) : v;
                    } else {
                        const int q = (ph - 1 + CPL) % CPL;   // outgoing logical 0
                        CW v = __shfl_down_sync(0xffffffffu, win[q], 1);
                        win[q] = lane == 31 ? CW(fresh) : v;
                    }
                }
                // --- matching cost C(x', d) for the lane's CPL cells
                uint32_t C[R];
                {
                    const uint64_t rv = cref[i & 63];
                    uint32_t c[CPL];
#pragma unroll
                    for (int jj = 0; jj < CPL; ++jj) {
                        const int phys = BWD ? (jj + ph) % CPL : (jj - ph + CPL) % CPL;
                        if (C64) c[jj] = __popcll(rv ^ uint64_t(win[phys]));
                        else c[jj] = __popc(uint32_t(rv) ^ uint32_t(win[phys]));
                    }
                    if (xv < p.D - 1) {                        // border: x' - d < 0 -> C_max
#pragma unroll
                        for (int jj = 0; jj < CPL; ++jj)
                            if (dbase + jj > xv) c[jj] = uint32_t(p.cmax);
                    }
#pragma unroll
                    for (int r = 0; r < R; ++r) C[r] = __byte_perm(c[2 * r], c[2 * r + 1], 0x5410) | pad[r];
                }
                // --- horizontal path (registers)
                uint32_t S[R];
                {
                    uint32_t nL[R];
                    path_update<R>(Lh, C, nL, p1x2, p2x2, lane);
#pragma unroll
                    for (int r = 0; r < R; ++r) { Lh[r] = nL[r]; S[r] = nL[r]; }
                }
                // --- vertical + diagonal paths from the row above
                uint16_t *dst = nullptr;
                if (warp < NW - 1) dst = my_ring + size_t(i & (kRing - 1)) * VEC;
                else if (is_producer) dst = gout + (long long)i * VEC;
#pragma unroll
                for (int v = 0; v < 3; ++v) {
                    // v = 0: down (row above at i), 1: diagonal from (i-1), 2: diagonal from (i+1)
                    const int q = i + (v == 1 ? -1 : (v == 2 ? 1 : 0));
                    uint32_t prev[R];
                    if (have_above && q >= 0 && q < W) {
                        VecIO<R>::ld(src_ring + size_t(q & src_mask) * VEC + v * DP + dbase, prev);
                    } else {
#pragma unroll
                        for (int r = 0; r < R; ++r) prev[r] = 0;
                    }
                    uint32_t nL[R];
                    path_update<R>(prev, C, nL, p1x2, p2x2, lane);
#pragma unroll
                    for (int r = 0; r < R; ++r) S[r] += nL[r];
                    if (dst) VecIO<R>::st(dst + v * DP + dbase, nL);
                }
                // --- sweep output
                if (!BWD) {
                    VecIO<R>::st(sfwd_row + (long long)xv * DP + dbase, S);
                } else {
                    uint32_t St[R];
                    const int slot = ph & 1;
#pragma unroll
                    for (int r = 0; r < R; ++r) St[r] = S[r] + pf[slot][r];
                    if (i + 2 < W) VecIO<R>::ld(sfwd_row + (long long)xview(i + 2) * DP + dbase, pf[slot]);
                    const int x = X(xv);
                    if (do_sout) {
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            const int d0 = dbase + 2 * r;
                            uint16_t *o = p.sout + ((long long)y * W + x) * p.D;
                            if (d0 < p.D) o[d0] = uint16_t(St[r] & 0xffffu);
                            if (d0 + 1 < p.D) o[d0 + 1] = uint16_t(St[r] >> 16);
                        }
                    }
                    if (do_wta) {
                        uint32_t best = 0xffffffffu;
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            const uint32_t k0 = __byte_perm(St[r], dcode[r], 0x6104);
                            const uint32_t k1 = __byte_perm(St[r], dcode[r], 0x7325);
                            best = min(best, min(k0, k1));
                        }
                        const uint32_t bkey = __reduce_min_sync(0xffffffffu, best);
                        const int dstar = int(bkey & 0xffu);
                        const int sb = int(bkey >> 8);
                        VecIO<R>::st(wta + dbase, St);
                        __syncwarp();
                        float sub = float(dstar);
                        if (dstar > 0 && dstar < p.D - 1) {
                            const int sa = wta[dstar - 1];
                            const int sc = wta[dstar + 1];
                            const int den = 2 * (sa + sc - 2 * sb);
                            float off = 0.f;
                            if (den != 0) off = __fdiv_rn(float(sa - sc), float(den));
                            off = fminf(fmaxf(off, -0.5f), 0.5f);
                            sub = __fadd_rn(float(dstar), off);
                        }
                        __syncwarp();
                        const int sl = i & 31;
                        if (lane == sl) { od = dstar; os = sub; }
                        if (sl == 31 || i == W - 1) {
                            const int pos = (i & ~31) + lane;
                            if (lane <= sl) {
                                const int xo = X(xview(pos));
                                dint_row[xo] = int16_t(od);
                                dsub_row[xo] = os;
                            }
                        }
                    }
                }
            }
            __syncthreads();
        }
    }
    if (is_producer) {
        __threadfence();
        if (lane == 0) st_relaxed_gpu(prog_out, W);
    }
    if (band_input) cp_async_wait<0>();
}

template <int CPL, bool C64, int NW>
cudaError_t launch_pair(const SweepParams &p, bool debug_s, cudaStream_t st, cudaEvent_t ev_mid_a,
                        cudaEvent_t ev_mid_b, int *launches, int *sync_buf, size_t sync_bytes) {
    (void)debug_s;
    const dim3 grid(p.nviews * p.nbands), block(NW * 32);
    cudaError_t e;
    {
        constexpr size_t sm = Sweep<CPL, C64, false, NW>::smem_bytes();
        auto k = sweep_kernel<CPL, C64, false, NW>;
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm))) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(sync_buf, 0, sync_bytes, st)) != cudaSuccess) return e;
        k<<<grid, block, sm, st>>>(p);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (launches) ++*launches;
    }
    if (ev_mid_a) cudaEventRecord(ev_mid_a, st);
    if (ev_mid_b) cudaEventRecord(ev_mid_b, st);
    {
        constexpr size_t sm = Sweep<CPL, C64, true, NW>::smem_bytes();
        auto k = sweep_kernel<CPL, C64, true, NW>;
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm))) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(sync_buf, 0, sync_bytes, st)) != cudaSuccess) return e;
        k<<<grid, block, sm, st>>>(p);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (launches) ++*launches;
    }
    return cudaSuccess;
}

}  // namespace

int sweep_warps_for(int cpl) { return cpl <= 4 ? 16 : 8; }

cudaError_t launch_sweeps(const SweepParams &p, int cpl, bool c64, int nw, bool debug_s,
                          cudaStream_t st, cudaEvent_t mid_ev_a, cudaEvent_t mid_ev_b,
                          int *launches) {
    // ticket + progress live at p.ticket (ticket first, then progress[nviews*nbands])
    int *sync_buf = p.ticket;
    const size_t sync_bytes = sizeof(int) * (1 + size_t(p.nviews) * p.nbands);
    if (nw != sweep_warps_for(cpl)) return cudaErrorInvalidValue;
#define SGM_CASE(CPL_, C64_)                                                                   \
    if (cpl == CPL_ && c64 == C64_)                                                            \
        return launch_pair<CPL_, C64_, (CPL_ <= 4 ? 16 : 8)>(p, debug_s, st, mid_ev_a, mid_ev_b, \
                                                             launches, sync_buf, sync_bytes);
    SGM_CASE(2, false) SGM_CASE(2, true) SGM_CASE(4, false) SGM_CASE(4, true)
    SGM_CASE(6, false) SGM_CASE(6, true) SGM_CASE(8, false) SGM_CASE(8, true)
#undef SGM_CASE
    return cudaErrorInvalidValue;
}

}  // namespace sgm
