// flow.cu -- the optical-flow core of the method ("Optical
// Flow from Flow Fields+"; SPEC flow-fields S:189-292) for sm_100a.
//
// Everything is exact integer arithmetic (readings FF1-FF10): flow
// vectors in 1/8 px, the patch data term as an integer SAD with bilinear weights in
// 1/64 steps, WHT descriptors as exact integer sums, kNN distances exact in fp64.  So
// every accept / reject decision equals the CPU oracle's, whatever the summation order.
//
// Kernels
//   ff_downsample_kernel  2x2 box pyramid level (thread per output pixel)
//   ff_wht_kernel         16 lowest-sequency WHT coefficients (thread per pixel)
//   ff_knn_kernel         exhaustive k nearest descriptors of the 16x16 window (thread per
//                         query; the database streams through shared memory in tiles;
//                         strict-< insertion in index order reproduces the "ties to the
//                         smaller index" rule); windows up to 8x8 run on the tensor cores
//                         (knn_tc.cu: tcgen05.mma into TMEM, exact limb arithmetic)
//   ff_init_kernel        best of the k candidates by data term (thread per pixel)
//   ff_prop_kernel        one propagation sweep: a persistent wavefront, one warp per
//                         image row, the row's pixels in scan order; the warp's 32 lanes
//                         split the (2r+1)^2 samples of both candidates (left/up, or
//                         right/down) and sum them with REDUX; rows hand their vectors to the
//                         next row through a shared-memory ring, bands of NW rows through a
//                         global row buffer, both as tagged 64-bit words polled directly (no
//                         fences); CTAs take tickets so a band only waits for an
//                         already-running band
//                         the random search after each sweep is fused in: once a row's
//                         propagation is done its warp searches the row (lane per pixel)
//   ff_lift_kernel        x2 vectors, nearest-neighbour upsampling, costs recomputed
//   ff_consistency_kernel two-inverse-field check (thread per pixel)
#include "sgm_internal.cuh"

namespace sgm {
namespace {

constexpr int FQ = 8;
constexpr int FQ2 = FQ * FQ;
constexpr int kRowRing = 128;    // row -> next-row handoff ring (positions) per warp

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Quad image (FF4 helper, exact): Q(x, y) packs the four bilinear taps B(x, y), B(x+1, y),
// B(x, y+1), B(x+1, y+1) (coordinates clamped) into one 32-bit word, so a sample is one
// load and one DP4A against the packed weights.
// Bilinear setup of one candidate vector (fu, fv): every sample of the patch has the same
// fractional part, so the weights and the integer offset are computed once.  Sample at
// pixel (sx, sy) reads Q at (sx + qx, sy + qy); it lies inside [0, (W-1) Q] x [0, (H-1) Q]
// iff 0 <= sx + qx <= ixmax and 0 <= sy + qy <= iymax (a clamped tap has weight 0).
struct Cand {
    int qx, qy, ixmax, iymax;
    unsigned wpack;
    __device__ __forceinline__ Cand(int fu, int fv, int W, int H) {
        qx = fu >> 3; qy = fv >> 3;                    // floor (arithmetic shift)
        const int fx = fu & 7, fy = fv & 7;
        wpack = unsigned((FQ - fx) * (FQ - fy)) | (unsigned(fx * (FQ - fy)) << 8) |
                (unsigned((FQ - fx) * fy) << 16) | (unsigned(fx * fy) << 24);
        ixmax = W - 1 - (fx ? 1 : 0); iymax = H - 1 - (fy ? 1 : 0);
    }
    // |Q^2 a - b| at B position (ix, iy) = sample + (qx, qy), or pen64 outside
    __device__ __forceinline__ int cost(const uint32_t *__restrict__ QB, int W, int ix, int iy, int a,
                                        int pen64) const {
        const bool in = (ix | iy) >= 0 && ix <= ixmax && iy <= iymax;
        const unsigned t = __ldg(QB + (in ? iy * W + ix : 0));   // images < 2^31 pixels
        const int b = int(__dp4a(t, wpack, 0u));
        return in ? abs(FQ2 * a - b) : pen64;
    }
};

// Candidate setup for the warp-cooperative evaluation at pixel (x, y): per-lane sample k is
// the pixel (x + sdx[k], y + sdy[k]); its B position (bx + sdx[k], by + sdy[k]) is inside
// iff both unsigned coordinates are <= (ux, uy) (ux = 0 with bx pushed far negative when no
// column can be inside, W = 1 with a fractional part); offsets are 32-bit.
struct CandW {
    int base, bx, by;
    unsigned ux, uy, wpack;
    __device__ __forceinline__ CandW(int fu, int fv, int x, int y, int W, int H) {
        const int fx = fu & 7, fy = fv & 7;
        wpack = unsigned((FQ - fx) * (FQ - fy)) | (unsigned(fx * (FQ - fy)) << 8) |
                (unsigned((FQ - fx) * fy) << 16) | (unsigned(fx * fy) << 24);
        const int ixmax = W - 1 - (fx ? 1 : 0), iymax = H - 1 - (fy ? 1 : 0);
        bx = ixmax >= 0 ? x + (fu >> 3) : -(1 << 29);
        by = iymax >= 0 ? y + (fv >> 3) : -(1 << 29);
        ux = ixmax >= 0 ? unsigned(ixmax) : 0u;
        uy = iymax >= 0 ? unsigned(iymax) : 0u;
        base = by * W + bx;
    }
    __device__ __forceinline__ int cost(const uint32_t *__restrict__ QB, int dx, int dy, int soff, int a,
                                        int pen64) const {
        const bool in = unsigned(bx + dx) <= ux && unsigned(by + dy) <= uy;
        const unsigned t = __ldg(QB + (in ? base + soff : 0));
        const int b = int(__dp4a(t, wpack, 0u));
        return in ? abs(FQ2 * a - b) : pen64;
    }
    // every sample of the (2r+1)^2 patch inside (the common case away from the borders):
    // then no sample needs the bounds test or the penalty (same integers as cost())
    __device__ __forceinline__ bool interior(int r) const {
        return bx - r >= 0 && unsigned(bx + r) <= ux && by - r >= 0 && unsigned(by + r) <= uy;
    }
    __device__ __forceinline__ int cost_in(const uint32_t *__restrict__ QB, int soff, int a64) const {
        const unsigned t = __ldg(QB + base + soff);
        return abs(a64 - int(__dp4a(t, wpack, 0u)));
    }
};

// The whole data term by one thread, sample order irrelevant (integers).  The
// row loop is unrolled over the widest supported patch (15) with a predicate, so the
// loads of a row's samples are in flight together.
__device__ __forceinline__ int patch_cost_thread(const uint8_t *__restrict__ A, const uint32_t *__restrict__ QB,
                                                 int W, int H, int x, int y, int fu, int fv, int r, int pen64) {
    const Cand c(fu, fv, W, H);
    int s = 0;
    // the whole patch inside both images (the common case): no clamping, no bounds tests
    if (x - r >= 0 && x + r < W && y - r >= 0 && y + r < H && x - r + c.qx >= 0 && x + r + c.qx <= c.ixmax &&
        y - r + c.qy >= 0 && y + r + c.qy <= c.iymax) {
        const uint8_t *arow = A + (y - r) * W + x;
        const uint32_t *brow = QB + (y - r + c.qy) * W + x + c.qx;
        for (int dy = -r; dy <= r; ++dy, arow += W, brow += W) {
#pragma unroll
            for (int k = 0; k < 15; ++k) {
                const int dx = k - r;
                if (dx <= r) {
                    const int a = __ldg(arow + dx);
                    s += abs(FQ2 * a - int(__dp4a(__ldg(brow + dx), c.wpack, 0u)));
                }
            }
        }
        return s;
    }
    for (int dy = -r; dy <= r; ++dy) {
        const uint8_t *arow = A + clampi(y + dy, 0, H - 1) * W;
        const int iy = y + dy + c.qy;
#pragma unroll
        for (int k = 0; k < 15; ++k) {
            const int dx = k - r;
            if (dx <= r) {
                const int a = __ldg(arow + clampi(x + dx, 0, W - 1));
                s += c.cost(QB, W, x + dx + c.qx, iy, a, pen64);
            }
        }
    }
    return s;
}

__global__ void ff_quad_kernel(const uint8_t *__restrict__ src, long long src_stride, int W, int H, int nimg,
                               uint32_t *__restrict__ dst, long long dst_stride) {
    const long long per = (long long)W * H, total = per * nimg;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int k = int(t / per);
        const long long q = t - k * per;
        const int y = int(q / W), x = int(q - (long long)y * W);
        const uint8_t *s0 = src + k * src_stride + (long long)y * W;
        const uint8_t *s1 = src + k * src_stride + (long long)min(y + 1, H - 1) * W;
        const int x1 = min(x + 1, W - 1);
        dst[k * dst_stride + q] = unsigned(s0[x]) | (unsigned(s0[x1]) << 8) | (unsigned(s1[x]) << 16) |
                                  (unsigned(s1[x1]) << 24);
    }
}

__device__ __forceinline__ uint64_t splitmix(uint64_t seed, int level, int sweep, int x, int y) {
    uint64_t z = seed ^ (uint64_t(level & 0xff) << 56) ^ (uint64_t(sweep & 0xff) << 48) ^
                 (uint64_t(y & 0xffffff) << 24) ^ uint64_t(x & 0xffffff);
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// ------------------------------------------------------------------ pyramid (FF2)
__global__ void ff_downsample_kernel(const uint8_t *__restrict__ src, long long src_stride, int W, int H,
                                     uint8_t *__restrict__ dst, long long dst_stride, int nimg) {
    const int W2 = (W + 1) / 2, H2 = (H + 1) / 2;
    const long long per = (long long)W2 * H2, total = per * nimg;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int k = int(i / per);
        const long long q = i - k * per;
        const int y = int(q / W2), x = int(q - (long long)y * W2);
        const uint8_t *s = src + k * src_stride;
        const int x0 = min(2 * x, W - 1), x1 = min(2 * x + 1, W - 1);
        const int y0 = min(2 * y, H - 1), y1 = min(2 * y + 1, H - 1);
        const int sum = s[(long long)y0 * W + x0] + s[(long long)y0 * W + x1] + s[(long long)y1 * W + x0] +
                        s[(long long)y1 * W + x1];
        dst[k * dst_stride + q] = uint8_t((sum + 2) >> 2);
    }
}

// ------------------------------------------------------------------ WHT (FF3)
// Sequency-ordered Walsh function value w_k(i) for length N: the Sylvester row with k
// sign changes is the one whose index is the bit-reversed Gray code of k.
__device__ __forceinline__ int walsh(int k, int i, int logn) {
    const int g = k ^ (k >> 1);                       // Gray code
    const int rrow = __brev(unsigned(g)) >> (32 - logn);   // bit reversal
    return (__popc(rrow & i) & 1) ? -1 : 1;
}

__global__ void ff_wht_kernel(const uint8_t *__restrict__ img, long long img_stride, int W, int H,
                              int win, int nimg, int32_t *__restrict__ desc) {
    const int logn = win == 4 ? 2 : (win == 8 ? 3 : 4);
    const long long per = (long long)W * H, total = per * nimg;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int k = int(t / per);
        const long long q = t - k * per;
        const int y = int(q / W), x = int(q - (long long)y * W);
        const uint8_t *s = img + k * img_stride;
        const int o = win / 2 - 1;
        // row transform: R[j][u] = sum_i P(i, j) w_u(i), u < 4; then columns
        int acc[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[c] = 0;
        for (int j = 0; j < win; ++j) {
            const uint8_t *row = s + (long long)clampi(y - o + j, 0, H - 1) * W;
            int R[4] = {0, 0, 0, 0};
            for (int i = 0; i < win; ++i) {
                const int pv = row[clampi(x - o + i, 0, W - 1)];
#pragma unroll
                for (int u = 0; u < 4; ++u) R[u] += pv * walsh(u, i, logn);
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int wv = walsh(v, j, logn);
#pragma unroll
                for (int u = 0; u < 4; ++u) acc[v * 4 + u] += R[u] * wv;
            }
        }
        int4 *out = reinterpret_cast<int4 *>(desc + t * 16);
#pragma unroll
        for (int c = 0; c < 4; ++c) out[c] = make_int4(acc[4 * c], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
    }
}

// ------------------------------------------------------------------ kNN (FF5)
constexpr int kKnnMax = 8;
constexpr int kKnnTile = 128;

// desc [2 npairs][n][16] (image 2k = A_k, 2k+1 = B_k); problem p takes its queries from
// image p and its database from image p ^ 1 (A_k -> B_k, B_k -> A_k); nn [nprob][n][knn]
__global__ void __launch_bounds__(128) ff_knn_kernel(const int32_t *__restrict__ desc, int n, int knn,
                                                     int32_t *__restrict__ nn) {
    __shared__ double tile[kKnnTile][16];
    const int prob = blockIdx.y;
    const int qi = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = qi < n;
    const int32_t *dq = desc + (long long)prob * n * 16;
    const int32_t *dd = desc + (long long)(prob ^ 1) * n * 16;
    double q[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) q[c] = active ? double(dq[(long long)qi * 16 + c]) : 0.0;
    double bd[kKnnMax];
    int bi[kKnnMax];
#pragma unroll
    for (int k = 0; k < kKnnMax; ++k) { bd[k] = 1e300; bi[k] = 0x7fffffff; }
    double thr = active ? 1e300 : -1.0;           // k-th best distance so far (inactive: never)
    int thr_i = 0x7fffffff;                        // and its index
    // Tiles are visited nearest-first around the block's own image position (small motions
    // find good matches early, so the DC bound prunes most of the database).  Entries are
    // ranked by (distance, index) lexicographically, so the visiting order does not change
    // the result: it equals the index-order scan of the oracle with ties to the smaller index.
    const int ntiles = (n + kKnnTile - 1) / kKnnTile;
    const int t0 = min(int((long long)blockIdx.x * blockDim.x / kKnnTile), ntiles - 1);
    for (int it = 0; it < ntiles; ++it) {
        // t0, t0+1, t0-1, t0+2, t0-2, ... clipped to [0, ntiles)
        const int up = ntiles - 1 - t0, dn = t0;
        int t;
        const int h = (it + 1) / 2;
        if (it == 0) t = t0;
        else if (h <= min(up, dn)) t = (it & 1) ? t0 + h : t0 - h;
        else t = up > dn ? t0 + (it - dn) : t0 - (it - up);
        const int base = t * kKnnTile;
        __syncthreads();
        for (int u = threadIdx.x; u < kKnnTile * 16; u += blockDim.x) {
            const int e = base + u / 16;
            tile[u / 16][u & 15] = e < n ? double(dd[(long long)e * 16 + (u & 15)]) : 0.0;
        }
        __syncthreads();
        const int lim = min(kKnnTile, n - base);
        for (int e = 0; e < lim; ++e) {
            // the DC term alone bounds the distance from below: when it exceeds the k-th
            // best for every lane, the entry cannot enter any list (exact pruning)
            const double t0d = q[0] - tile[e][0];
            double d = t0d * t0d;
            if (!__any_sync(0xffffffffu, d <= thr)) continue;
#pragma unroll
            for (int c = 1; c < 16; ++c) {
                const double tc = q[c] - tile[e][c];
                d = fma(tc, tc, d);
            }
            // exact: every term and partial sum is an integer < 2^53
            const int idx = base + e;
            if (d < thr || (d == thr && idx < thr_i)) {
                int ci = idx;
                double dv = d;
                bool ins = false;
#pragma unroll
                for (int k = 0; k < kKnnMax; ++k) {      // sorted insertion by (d, index)
                    if (k < knn && (ins || dv < bd[k] || (dv == bd[k] && ci < bi[k]))) {
                        const double td = bd[k]; const int ti = bi[k];
                        bd[k] = dv; bi[k] = ci; dv = td; ci = ti;
                        ins = true;
                    }
                }
#pragma unroll
                for (int k = 0; k < kKnnMax; ++k)
                    if (k == knn - 1) { thr = bd[k]; thr_i = bi[k]; }
            }
        }
    }
    if (active)
        for (int k = 0; k < knn; ++k) nn[((long long)prob * n + qi) * knn + k] = bi[k];
}
// ------------------------------------------------------------------ fields
// A field f of a batch: pair k = f / fpp, kind = f % fpp; kind 0 matches A_k -> B_k,
// kinds 1, 2 match B_k -> A_k (the two inverse fields, F-5).
struct FieldSet {
    int W, H, fpp, nfields;
    const uint8_t *A, *B;          // level images, pair k at + k * img_stride
    long long img_stride;
    const uint32_t *QA, *QB;       // their quad images, pair k at + k * img_stride
    int radius[3];
    uint64_t seed[3];
    int pen64;
    int32_t *flow;                 // [nfields][H][W][2]
    int32_t *cost;                 // [nfields][H][W]
    // source image and the quad image of the target of field f
    __device__ __forceinline__ void images(int f, const uint8_t *&src, const uint32_t *&qdst) const {
        const int k = f / fpp, kind = f - k * fpp;
        src = (kind == 0 ? A : B) + k * img_stride;
        qdst = (kind == 0 ? QB : QA) + k * img_stride;
    }
    __device__ __forceinline__ int kind(int f) const { return f % fpp; }
    // selects instead of indexing: a runtime index into the by-value parameter arrays
    // would copy them to local memory
    __device__ __forceinline__ int rad(int k) const { return k == 0 ? radius[0] : (k == 1 ? radius[1] : radius[2]); }
    __device__ __forceinline__ uint64_t sd(int k) const { return k == 0 ? seed[0] : (k == 1 ? seed[1] : seed[2]); }
};

// best of the k candidates (FF5): nn lists per (pair, direction): direction 0 = A->B
__global__ void ff_init_kernel(FieldSet fs, const int32_t *__restrict__ nn, int knn) {
    const long long per = (long long)fs.W * fs.H, total = per * fs.nfields;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int f = int(t / per);
        const long long p = t - f * per;
        const int y = int(p / fs.W), x = int(p - (long long)y * fs.W);
        const uint8_t *src;
        const uint32_t *dst;
        fs.images(f, src, dst);
        const int kind = fs.kind(f), pair = f / fs.fpp;
        const int dir = kind == 0 ? 0 : 1;
        const int32_t *cand = nn + ((long long)(2 * pair + dir) * per + p) * knn;
        int best = 0x7fffffff, bu = 0, bv = 0;
        for (int k = 0; k < knn; ++k) {
            const int q = cand[k];
            if (q < 0 || q >= per) continue;        // fewer database pixels than knn
            const int yb = q / fs.W, xb = q - yb * fs.W;
            const int fu = (xb - x) * FQ, fv = (yb - y) * FQ;
            const int c = patch_cost_thread(src, dst, fs.W, fs.H, x, y, fu, fv, fs.rad(kind), fs.pen64);
            if (c < best) { best = c; bu = fu; bv = fv; }
        }
        fs.flow[2 * t] = bu;
        fs.flow[2 * t + 1] = bv;
        fs.cost[t] = best;
    }
}

// lift (FF8): coarse [nfields][Hc][Wc][2] -> fine
__global__ void ff_lift_kernel(FieldSet fs, const int32_t *__restrict__ coarse, int Wc, int Hc) {
    const long long per = (long long)fs.W * fs.H, total = per * fs.nfields;
    const long long cper = (long long)Wc * Hc;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int f = int(t / per);
        const long long p = t - f * per;
        const int y = int(p / fs.W), x = int(p - (long long)y * fs.W);
        const long long c = f * cper + (long long)min(y >> 1, Hc - 1) * Wc + min(x >> 1, Wc - 1);
        const int fu = 2 * coarse[2 * c], fv = 2 * coarse[2 * c + 1];
        const uint8_t *src;
        const uint32_t *dst;
        fs.images(f, src, dst);
        fs.flow[2 * t] = fu;
        fs.flow[2 * t + 1] = fv;
        fs.cost[t] = patch_cost_thread(src, dst, fs.W, fs.H, x, y, fu, fv, fs.rad(fs.kind(f)), fs.pen64);
    }
}

// 1: warp-uniform decisions of the pixel loop are taken through votes and the lane-0 store
// block is executed by every lane (same values, same addresses), so the compiler emits uniform
// branches and no reconvergence regions: propagation 46.7 -> 45.3 ms per 8 Driving pairs,
// output digest identical.  2: also the warp index and the polling loops.
// (2: 45.3 -> 40.9 ms.)  3: also the interior tests and the band-handoff polling loop.
#ifndef FF_UNIFORM
#define FF_UNIFORM 2
#endif
#ifndef FF_APRE
#define FF_APRE 0
#endif
// ------------------------------------------------------------------ propagation (FF7)
struct PropParams {
    FieldSet fs;
    int sweep;
    int level;                    // RNG stream of the fused random search
    int R0;                       // random-search radius of sweep 0 (px); 0 = no search
    int nbands;
    int *ticket;                  // zeroed before the launch
    unsigned long long *hand;     // [nfields][nbands][W] band handoff rows, zeroed before the launch
};

// Row-to-row handoff entries: one 64-bit word = vector (2 x 20-bit two's complement, 1/8 px)
// + tag (24 bits, position + 1, 0 = empty).  A 64-bit store / load is single-copy atomic,
// so the consumer polls the entry itself: no fence and no separate progress flag.
__device__ __forceinline__ unsigned long long pack_hand(int u, int v, int tag) {
    return (unsigned long long)(unsigned(u) & 0xFFFFFu) | ((unsigned long long)(unsigned(v) & 0xFFFFFu) << 20) |
           ((unsigned long long)unsigned(tag) << 40);
}
__device__ __forceinline__ int hand_tag(unsigned long long e) { return int(e >> 40); }
__device__ __forceinline__ int2 hand_vec(unsigned long long e) {
    const int u = int(unsigned(e) << 12) >> 12;                     // sign-extend 20 bits
    const int v = int(unsigned(e >> 20) << 12) >> 12;
    return make_int2(u, v);
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}

// One row of one field in scan order (the body of ff_prop_kernel); NK = samples per lane
// ((2r+1)^2 <= 32 NK), so every lane's A and B loads of a pixel are issued together.
template <int NW, int NK, int RC>   // RC >= 0: the patch radius as a compile-time constant
__device__ __forceinline__ void prop_row(const PropParams &pp, volatile unsigned long long *sring,
                                         volatile int *sprog, int f, int band, int warp, int lane, int j) {
    const FieldSet &fs = pp.fs;
    const int W = fs.W, H = fs.H;
    const bool fwd = (pp.sweep & 1) == 0;
    const int y = fwd ? j : H - 1 - j;
    const uint8_t *src;
    const uint32_t *dst;
    fs.images(f, src, dst);
    const int kind = fs.kind(f);
    const int r = RC >= 0 ? RC : fs.rad(kind), side = 2 * r + 1, ns = side * side;
    const long long per = (long long)W * H;
    int32_t *flow = fs.flow + 2 * f * per;
    int32_t *cost = fs.cost + f * per;
    const bool has_above = j > 0;                   // previous row in scan order exists
    const bool above_in_cta = warp > 0;
    const bool has_below_in_cta = warp + 1 < NW && j + 1 < H;
    // band handoff rows: [nfields][nbands][W], zeroed before the launch
    const unsigned long long *hin = pp.hand + ((long long)f * pp.nbands + band - 1) * W;
    unsigned long long *hout = pp.hand + ((long long)f * pp.nbands + band) * W;
    const bool publish = warp == NW - 1 && band + 1 < pp.nbands;
    volatile unsigned long long *ring_in = sring + (size_t)(warp - 1) * kRowRing;
    volatile unsigned long long *ring_out = sring + (size_t)warp * kRowRing;
    // this lane's samples: (dx, dy) of sample lane + 32 k, valid iff < ns
    int sdx[NK], sdy[NK];
    bool sok[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        const int sidx = lane + 32 * k;
        sok[k] = sidx < ns;
        const int q = sok[k] ? sidx : 0;
        sdy[k] = q / side - r;
        sdx[k] = q - (q / side) * side - r;
    }
    int aoff[NK], soff[NK];                         // A row / B offset of this lane's samples
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        aoff[k] = clampi(y + sdy[k], 0, H - 1) * W;
        soff[k] = sdy[k] * W + sdx[k];
    }
    int2 hv = make_int2(0, 0);                      // vector of the previous pixel in scan order
    unsigned long long hbuf = 0ull;                 // band handoff entries of the chunk (lane l)
    // The incumbents (vector + cost) of 32 positions are loaded per chunk, lane l holding
    // position 32c + l, one chunk ahead: no global load latency on the row's chain.
    auto chunk_px = [&](int i) { return y * W + (fwd ? i : W - 1 - i); };   // < 2^31 per field
    int cu_l = 0, cv_l = 0, cc_l = 0, nu_l = 0, nv_l = 0, nc_l = 0;
    if (lane < W) { const int q = chunk_px(lane); cu_l = flow[2 * q]; cv_l = flow[2 * q + 1]; cc_l = cost[q]; }
    if (32 + lane < W) { const int q = chunk_px(32 + lane); nu_l = flow[2 * q]; nv_l = flow[2 * q + 1]; nc_l = cost[q]; }
    for (int i = 0; i < W; ++i) {
        const int x = fwd ? i : W - 1 - i;
        const int p = y * W + x;
        if ((i & 31) == 0 && i > 0) {               // next chunk: rotate and prefetch
            cu_l = nu_l; cv_l = nv_l; cc_l = nc_l;
            if (i + 32 + lane < W) {
                const int q = chunk_px(i + 32 + lane);
                nu_l = flow[2 * q]; nv_l = flow[2 * q + 1]; nc_l = cost[q];
            }
        }
#if FF_APRE
        // A samples of this pixel: independent of the candidates, so they are issued before
        // the wait for the row above (their latency leaves the pixel-to-pixel chain)
        int a[NK];
#pragma unroll
        for (int k = 0; k < NK; ++k)
            a[k] = __ldg(src + aoff[k] + clampi(x + sdx[k], 0, W - 1));
#endif
        int cu = __shfl_sync(0xffffffffu, cu_l, i & 31);
        int cv = __shfl_sync(0xffffffffu, cv_l, i & 31);
        int cc = __shfl_sync(0xffffffffu, cc_l, i & 31);
        // vertical candidate: the finished vector of (x, row above in scan order)
        int2 vv = make_int2(0, 0);
        if (has_above) {
            unsigned long long e;
            if (above_in_cta) {
                // back off while waiting: spinning warps would take the issue slots of the
                // warps that have work
#if FF_UNIFORM >= 2
                while (__any_sync(0xffffffffu, hand_tag(e = ring_in[i & (kRowRing - 1)]) != i + 1)) __nanosleep(20);
#else
                while (hand_tag(e = ring_in[i & (kRowRing - 1)]) != i + 1) __nanosleep(20);
#endif
            } else {
                // band handoff through L2: the 32 positions of a chunk are fetched in one
                // round trip (lane l holds position 32c + l); a position not yet published
                // re-fetches the chunk, so the band runs one position behind its producer
                if ((i & 31) == 0) hbuf = i + lane < W ? ld_relaxed_u64(hin + i + lane) : 0ull;
                e = __shfl_sync(0xffffffffu, hbuf, i & 31);
#if FF_UNIFORM >= 3
                while (__any_sync(0xffffffffu, hand_tag(e) != i + 1)) {
#else
                while (hand_tag(e) != i + 1) {
#endif
                    __nanosleep(64);
                    const int q = (i & ~31) + lane;
                    hbuf = q < W ? ld_relaxed_u64(hin + q) : 0ull;
                    e = __shfl_sync(0xffffffffu, hbuf, i & 31);
                }
            }
            vv = hand_vec(e);
        }
        // candidates in order: horizontal (previous pixel), vertical; skip ones equal to
        // the incumbent (their data term equals the incumbent's: never strictly better)
#if FF_UNIFORM
        // (the values are warp-uniform; the votes tell the compiler so: uniform branches, no
        // reconvergence regions around the candidate evaluation)
        const bool eh = __any_sync(0xffffffffu, i > 0 && (hv.x != cu || hv.y != cv));
        const bool ev = __any_sync(0xffffffffu, has_above && (vv.x != cu || vv.y != cv) &&
                                                    (!eh || vv.x != hv.x || vv.y != hv.y));
#else
        const bool eh = i > 0 && (hv.x != cu || hv.y != cv);
        const bool ev = has_above && (vv.x != cu || vv.y != cv) && (!eh || vv.x != hv.x || vv.y != hv.y);
#endif
#if !FF_APRE
        int a[NK];                                  // A samples, loaded only when needed
        if (eh || ev) {
#pragma unroll
            for (int k = 0; k < NK; ++k)
                a[k] = __ldg(src + aoff[k] + clampi(x + sdx[k], 0, W - 1));
        }
#endif
        if (eh && ev) {                             // both candidates: loads in flight together
            const CandW C0(hv.x, hv.y, x, y, W, H), C1(vv.x, vv.y, x, y, W, H);
            int s0 = 0, s1 = 0;
#if FF_UNIFORM >= 3
            if (__all_sync(0xffffffffu, C0.interior(r) && C1.interior(r))) {
#else
            if (C0.interior(r) && C1.interior(r)) {     // (warp-uniform) no bounds tests
#endif
#pragma unroll
                for (int k = 0; k < NK; ++k) {
                    const int a64 = FQ2 * a[k];
                    const int t0 = C0.cost_in(dst, soff[k], a64);
                    const int t1 = C1.cost_in(dst, soff[k], a64);
                    s0 += sok[k] ? t0 : 0;
                    s1 += sok[k] ? t1 : 0;
                }
            } else {
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                const int t0 = C0.cost(dst, sdx[k], sdy[k], soff[k], a[k], fs.pen64);
                const int t1 = C1.cost(dst, sdx[k], sdy[k], soff[k], a[k], fs.pen64);
                s0 += sok[k] ? t0 : 0;
                s1 += sok[k] ? t1 : 0;
            }
            }
            const int c0 = int(__reduce_add_sync(0xffffffffu, unsigned(s0)));
            const int c1 = int(__reduce_add_sync(0xffffffffu, unsigned(s1)));
            if (c0 < cc) { cc = c0; cu = hv.x; cv = hv.y; }
            if (c1 < cc) { cc = c1; cu = vv.x; cv = vv.y; }
        } else if (eh || ev) {                      // one candidate
            const int2 w = eh ? hv : vv;
            const CandW C0(w.x, w.y, x, y, W, H);
            int s0 = 0;
#if FF_UNIFORM >= 3
            if (__all_sync(0xffffffffu, C0.interior(r))) {
#else
            if (C0.interior(r)) {
#endif
#pragma unroll
                for (int k = 0; k < NK; ++k) {
                    const int t0 = C0.cost_in(dst, soff[k], FQ2 * a[k]);
                    s0 += sok[k] ? t0 : 0;
                }
            } else {
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                const int t0 = C0.cost(dst, sdx[k], sdy[k], soff[k], a[k], fs.pen64);
                s0 += sok[k] ? t0 : 0;
            }
            }
            const int c0 = int(__reduce_add_sync(0xffffffffu, unsigned(s0)));
            if (c0 < cc) { cc = c0; cu = w.x; cv = w.y; }
        }
#if FF_UNIFORM
        // every lane stores the same values to the same addresses (one transaction each): no
        // divergent lane-0 region in the pixel loop
        {
            if (has_below_in_cta) {
                if (i >= kRowRing)
                    while (__any_sync(0xffffffffu, sprog[warp + 1] < i - kRowRing + 1)) __nanosleep(20);
                ring_out[i & (kRowRing - 1)] = pack_hand(cu, cv, i + 1);
            }
#else
        if (lane == 0) {
            if (has_below_in_cta) {
                // ring slot reuse: the row below must have consumed position i - kRowRing
                if (i >= kRowRing)
                    while (sprog[warp + 1] < i - kRowRing + 1) __nanosleep(20);
                ring_out[i & (kRowRing - 1)] = pack_hand(cu, cv, i + 1);
            }
#endif
            if (publish) st_relaxed_u64(hout + i, pack_hand(cu, cv, i + 1));
            sprog[warp] = i + 1;
            flow[2 * p] = cu;
            flow[2 * p + 1] = cv;
            cost[p] = cc;
        }
        hv = make_int2(cu, cv);
        __syncwarp();
    }
    // Random search of this row (FF7, second half), fused into the sweep: it reads only each
    // pixel's own vector after the propagation, and the rows below take this row's
    // propagation results from the ring / handoff buffer, not from `flow`, so the order of
    // S:231 (whole sweep, then the search) is kept.  One lane per pixel.
    if (pp.R0 > 0) {
        const int R = max(pp.R0 >> pp.sweep, 1);
        const unsigned span = unsigned(2 * R * FQ + 1);
        const uint64_t seed = fs.sd(kind);
        for (int x = lane; x < W; x += 32) {
            const int p = y * W + x;
            const uint64_t z = splitmix(seed, pp.level, pp.sweep, x, y);
            const int fu = flow[2 * p] + int(unsigned(z) % span) - R * FQ;
            const int fv = flow[2 * p + 1] + int(unsigned(z >> 32) % span) - R * FQ;
            const int c = patch_cost_thread(src, dst, W, H, x, y, fu, fv, r, fs.pen64);
            if (c < cost[p]) {
                cost[p] = c;
                flow[2 * p] = fu;
                flow[2 * p + 1] = fv;
            }
        }
    }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32) ff_prop_kernel(const PropParams pp) {
    extern __shared__ __align__(16) unsigned char ff_smem[];
    volatile unsigned long long *sring = reinterpret_cast<volatile unsigned long long *>(ff_smem);   // [NW][kRowRing]
    volatile int *sprog = reinterpret_cast<volatile int *>(ff_smem + sizeof(unsigned long long) * NW * kRowRing);
    __shared__ int s_ticket;
    for (int t = threadIdx.x; t < NW * kRowRing; t += blockDim.x) sring[t] = 0ull;
    if (threadIdx.x < NW) sprog[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_ticket = atomicAdd(pp.ticket, 1);
    __syncthreads();
    const int ticket = s_ticket;
    // band-major tickets: the resident CTAs are the first bands of all fields, so a band's
    // predecessor (one ticket "row" earlier) has normally finished before it starts
    const int band = ticket / pp.fs.nfields, f = ticket - band * pp.fs.nfields;
#if FF_UNIFORM >= 2
    const int warp = int(__reduce_min_sync(0xffffffffu, threadIdx.x >> 5)), lane = threadIdx.x & 31;
#else
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#endif
    const int j = band * NW + warp;                 // iteration row
    if (j >= pp.fs.H) return;
    const int r = pp.fs.rad(pp.fs.kind(f));
    const int nk = ((2 * r + 1) * (2 * r + 1) + 31) / 32;
    // the default radii (r = 4 and the second inverse field's r + 2 = 6) get sample geometry
    // fixed at compile time
    if (r == 4) prop_row<NW, 3, 4>(pp, sring, sprog, f, band, warp, lane, j);
    else if (r == 6) prop_row<NW, 6, 6>(pp, sring, sprog, f, band, warp, lane, j);
    else if (nk <= 1) prop_row<NW, 1, -1>(pp, sring, sprog, f, band, warp, lane, j);
    else if (nk <= 3) prop_row<NW, 3, -1>(pp, sring, sprog, f, band, warp, lane, j);
    else if (nk <= 6) prop_row<NW, 6, -1>(pp, sring, sprog, f, band, warp, lane, j);
    else prop_row<NW, 8, -1>(pp, sring, sprog, f, band, warp, lane, j);
}

// ------------------------------------------------------------------ consistency (FF9)
__global__ void ff_consistency_kernel(const int32_t *__restrict__ F, const int32_t *__restrict__ G1,
                                      const int32_t *__restrict__ G2, long long fstride,
                                      long long gstride, int W, int H, int n, int thr_q,
                                      uint8_t *__restrict__ valid, float *__restrict__ fout) {
    const long long per = (long long)W * H, total = per * n;
    const long long lim = (long long)thr_q * FQ2;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int k = int(t / per);
        const long long p = t - k * per;
        const int y = int(p / W), x = int(p - (long long)y * W);
        const int32_t *f = F + k * fstride;
        const int fu = f[2 * p], fv = f[2 * p + 1];
        const int tx = x * FQ + fu, ty = y * FQ + fv;
        bool ok = tx >= 0 && ty >= 0 && tx <= (W - 1) * FQ && ty <= (H - 1) * FQ;
        for (int g = 0; g < 2 && ok; ++g) {
            const int32_t *G = (g == 0 ? G1 : G2) + k * gstride;
            const int ix = tx >> 3, fx = tx & 7, iy = ty >> 3, fy = ty & 7;
            const int ix1 = min(ix + 1, W - 1), iy1 = min(iy + 1, H - 1);
            const long long w00 = (FQ - fx) * (FQ - fy), w10 = fx * (FQ - fy);
            const long long w01 = (FQ - fx) * fy, w11 = fx * fy;
            const long long t00 = (long long)iy * W + ix, t10 = (long long)iy * W + ix1;
            const long long t01 = (long long)iy1 * W + ix, t11 = (long long)iy1 * W + ix1;
            const long long e0 = (long long)FQ2 * fu + w00 * G[2 * t00] + w10 * G[2 * t10] +
                                 w01 * G[2 * t01] + w11 * G[2 * t11];
            const long long e1 = (long long)FQ2 * fv + w00 * G[2 * t00 + 1] + w10 * G[2 * t10 + 1] +
                                 w01 * G[2 * t01 + 1] + w11 * G[2 * t11 + 1];
            ok = e0 * e0 + e1 * e1 <= lim * lim;
        }
        if (valid) valid[t] = uint8_t(ok);
        if (fout) {
            fout[2 * t] = float(fu) * (1.0f / FQ);       // exact: fu / 8
            fout[2 * t + 1] = float(fv) * (1.0f / FQ);
        }
    }
}

// data term of explicit queries (parity / debugging)
__global__ void ff_cost_query_kernel(const uint8_t *A, const uint32_t *QB, int W, int H, int r, int pen64,
                                     int nq, const int32_t *q, int32_t *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nq) out[i] = patch_cost_thread(A, QB, W, H, q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3], r, pen64);
}

int ff_grid(long long n, int block) {
    long long g = (n + block - 1) / block;
    const long long cap = 148LL * 32;
    return int(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

// ------------------------------------------------------------------ launchers
cudaError_t ff_launch_downsample(const uint8_t *src, long long src_stride, int W, int H, uint8_t *dst,
                                 long long dst_stride, int nimg, cudaStream_t st) {
    const long long n = (long long)((W + 1) / 2) * ((H + 1) / 2) * nimg;
    ff_downsample_kernel<<<ff_grid(n, 256), 256, 0, st>>>(src, src_stride, W, H, dst, dst_stride, nimg);
    return cudaGetLastError();
}

cudaError_t ff_launch_wht(const uint8_t *img, long long img_stride, int W, int H, int win, int nimg,
                          int32_t *desc, cudaStream_t st) {
    ff_wht_kernel<<<ff_grid((long long)W * H * nimg, 128), 128, 0, st>>>(img, img_stride, W, H, win, nimg, desc);
    return cudaGetLastError();
}

size_t ff_knn_scratch_bytes(long long entries) { return ff_knn_tc_scratch_bytes(entries); }

// k nearest descriptors of every entry of problem p (query image p) in image p ^ 1: windows
// up to 8x8 on the tensor cores (knn_tc.cu: coefficients < 2^14 split into exact limbs), the
// 16x16 window (coefficients up to 2^16) on the fp64 CUDA-core kernel
cudaError_t ff_launch_knn(const int32_t *desc, int n, int nprob, int knn, int win, int32_t *nn, void *scratch,
                          cudaStream_t st) {
    if (knn < 1 || knn > kKnnMax) return cudaErrorInvalidValue;
    if (win <= 8) return ff_launch_knn_tc(desc, n, nprob, knn, nn, scratch, st);
    dim3 grid((n + 127) / 128, nprob);
    ff_knn_kernel<<<grid, 128, 0, st>>>(desc, n, knn, nn);
    return cudaGetLastError();
}

static FieldSet make_fs(const FFFields &F) {
    FieldSet fs{};
    fs.W = F.W; fs.H = F.H; fs.fpp = F.fpp; fs.nfields = F.nfields;
    fs.A = F.A; fs.B = F.B; fs.img_stride = F.img_stride;
    fs.QA = F.QA; fs.QB = F.QB;
    for (int k = 0; k < 3; ++k) { fs.radius[k] = F.radius[k]; fs.seed[k] = F.seed[k]; }
    fs.pen64 = F.penalty * FQ2;
    fs.flow = F.flow; fs.cost = F.cost;
    return fs;
}

cudaError_t ff_launch_init(const FFFields &F, const int32_t *nn, int knn, cudaStream_t st) {
    const long long n = (long long)F.W * F.H * F.nfields;
    ff_init_kernel<<<ff_grid(n, 128), 128, 0, st>>>(make_fs(F), nn, knn);
    return cudaGetLastError();
}

cudaError_t ff_launch_lift(const FFFields &F, const int32_t *coarse, int Wc, int Hc, cudaStream_t st) {
    const long long n = (long long)F.W * F.H * F.nfields;
    ff_lift_kernel<<<ff_grid(n, 128), 128, 0, st>>>(make_fs(F), coarse, Wc, Hc);
    return cudaGetLastError();
}

// rows (warps) per propagation CTA; measured on the 8 bench pairs (propagation ms): 12 rows
// 52.2, 16 rows 40.9, 20 rows 46.1 (96 registers), 24 rows 50.3 (80 registers)
#ifndef FF_PROP_NW
#define FF_PROP_NW 16
#endif
constexpr int kPropNW = FF_PROP_NW;

size_t ff_prop_smem(int W) {
    (void)W;
    return size_t(kPropNW) * kRowRing * sizeof(unsigned long long) + 64 * sizeof(int);
}

cudaError_t ff_launch_sweep(const FFFields &F, int sweep, int level, int R0, int *sync, cudaStream_t st,
                            int *launches, FFTimer *timer) {
    PropParams pp{};
    pp.fs = make_fs(F);
    pp.sweep = sweep;
    pp.nbands = (F.H + kPropNW - 1) / kPropNW;
    pp.ticket = sync;
    pp.hand = reinterpret_cast<unsigned long long *>(sync + 4);
    const size_t hand_bytes = sizeof(unsigned long long) * size_t(F.nfields) * pp.nbands * F.W;
    cudaError_t e = cudaMemsetAsync(sync, 0, 4 * sizeof(int) + hand_bytes, st);
    if (e != cudaSuccess) return e;
    const size_t sm = ff_prop_smem(F.W);
    e = cudaFuncSetAttribute(ff_prop_kernel<kPropNW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    if (e != cudaSuccess) return e;
    pp.level = level;
    pp.R0 = R0;                               // the random search runs inside the sweep
    if (timer) timer->begin(0);
    ff_prop_kernel<kPropNW><<<F.nfields * pp.nbands, kPropNW * 32, sm, st>>>(pp);
    if (timer) timer->end();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (launches) *launches += 1;
    return cudaSuccess;
}

// ticket (+ padding to 16 bytes) and the band handoff rows of the largest level
long long ff_sync_ints(int nfields, int W, int H) {
    return 4 + 2LL * nfields * ((H + kPropNW - 1) / kPropNW) * W;
}

cudaError_t ff_launch_consistency(const int32_t *F, const int32_t *G1, const int32_t *G2, long long fstride,
                                  long long gstride, int W, int H, int n, int thr_q, uint8_t *valid,
                                  float *fout, cudaStream_t st) {
    ff_consistency_kernel<<<ff_grid((long long)W * H * n, 256), 256, 0, st>>>(F, G1, G2, fstride, gstride, W, H,
                                                                                n, thr_q, valid, fout);
    return cudaGetLastError();
}

cudaError_t ff_launch_cost_query(const uint8_t *A, const uint32_t *QB, int W, int H, int r, int penalty, int nq,
                                 const int32_t *q, int32_t *out, cudaStream_t st) {
    ff_cost_query_kernel<<<(nq + 127) / 128, 128, 0, st>>>(A, QB, W, H, r, penalty * FQ2, nq, q, out);
    return cudaGetLastError();
}

cudaError_t ff_launch_quad(const uint8_t *src, long long src_stride, int W, int H, int nimg, uint32_t *dst,
                           long long dst_stride, cudaStream_t st) {
    ff_quad_kernel<<<ff_grid((long long)W * H * nimg, 256), 256, 0, st>>>(src, src_stride, W, H, nimg, dst,
                                                                          dst_stride);
    return cudaGetLastError();
}

}  // namespace sgm
