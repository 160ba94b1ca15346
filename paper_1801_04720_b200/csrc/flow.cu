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
//   ff_knn_kernel         exhaustive k nearest descriptors (thread per query; the database
//                         streams through shared memory in tiles; strict-< insertion in
//                         index order reproduces the "ties to the smaller index" rule)
//   ff_init_kernel        best of the k candidates by data term (thread per pixel)
//   ff_prop_kernel        one propagation sweep: a persistent wavefront, one warp per
//                         image row, the row's pixels in scan order; the warp's 32 lanes
//                         split the (2r+1)^2 samples of both candidates (left/up, or
//                         right/down) and sum them with REDUX; rows hand their vectors to the
//                         next row through shared memory (per-pixel progress counter), bands
//                         of NW rows hand over through global memory (release/acquire
//                         progress flag every kPubFF pixels); CTAs take tickets so a band only
//                         waits for an already-running band
//   ff_search_kernel      the random search after each sweep (thread per pixel, counter RNG)
//   ff_lift_kernel        x2 vectors, nearest-neighbour upsampling, costs recomputed
//   ff_consistency_kernel two-inverse-field check (thread per pixel)
#include "sgm_internal.cuh"

namespace sgm {
namespace {

constexpr int FQ = 8;
constexpr int FQ2 = FQ * FQ;
constexpr int kPubFF = 8;        // band-handoff publication granularity (pixels)
constexpr int kNsMax = 8;        // samples per lane: (2r+1)^2 <= 256 -> r <= 7

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// |Q^2 a - bilinear B| of one sample, or the penalty outside B (FF4).
__device__ __forceinline__ int sample_cost(const uint8_t *__restrict__ B, int W, int H, int px, int py,
                                           int a, int pen64) {
    if (px < 0 || py < 0 || px > (W - 1) * FQ || py > (H - 1) * FQ) return pen64;
    const int ix = px >> 3, fx = px & 7, iy = py >> 3, fy = py & 7;
    const int ix1 = min(ix + 1, W - 1), iy1 = min(iy + 1, H - 1);
    const uint8_t *r0 = B + (long long)iy * W, *r1 = B + (long long)iy1 * W;
    const int b = (FQ - fx) * (FQ - fy) * int(__ldg(r0 + ix)) + fx * (FQ - fy) * int(__ldg(r0 + ix1)) +
                  (FQ - fx) * fy * int(__ldg(r1 + ix)) + fx * fy * int(__ldg(r1 + ix1));
    return abs(FQ2 * a - b);
}

// The whole data term by one thread, sample order irrelevant (integers).
__device__ int patch_cost_thread(const uint8_t *__restrict__ A, const uint8_t *__restrict__ B, int W,
                                 int H, int x, int y, int fu, int fv, int r, int pen64) {
    int s = 0;
    for (int dy = -r; dy <= r; ++dy) {
        const uint8_t *arow = A + (long long)clampi(y + dy, 0, H - 1) * W;
        const int py = (y + dy) * FQ + fv;
        for (int dx = -r; dx <= r; ++dx) {
            const int a = __ldg(arow + clampi(x + dx, 0, W - 1));
            s += sample_cost(B, W, H, (x + dx) * FQ + fu, py, a, pen64);
        }
    }
    return s;
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
    __shared__ int4 tile[kKnnTile * 4];
    const int prob = blockIdx.y;
    const int qi = blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t *dq = desc + (long long)prob * n * 16;
    const int32_t *dd = desc + (long long)(prob ^ 1) * n * 16;
    double q[16];
    if (qi < n) {
#pragma unroll
        for (int c = 0; c < 16; ++c) q[c] = double(dq[(long long)qi * 16 + c]);
    }
    double bd[kKnnMax];
    int bi[kKnnMax];
#pragma unroll
    for (int k = 0; k < kKnnMax; ++k) { bd[k] = 1e300; bi[k] = 0x7fffffff; }
    for (int base = 0; base < n; base += kKnnTile) {
        __syncthreads();
        for (int t = threadIdx.x; t < kKnnTile * 4; t += blockDim.x) {
            const int e = base + t / 4;
            tile[t] = e < n ? reinterpret_cast<const int4 *>(dd)[(long long)e * 4 + (t & 3)] : make_int4(0, 0, 0, 0);
        }
        __syncthreads();
        if (qi >= n) continue;
        const int lim = min(kKnnTile, n - base);
        for (int e = 0; e < lim; ++e) {
            double d = 0.0;
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
                const int4 v = tile[e * 4 + c4];
                double t0 = q[4 * c4] - double(v.x), t1 = q[4 * c4 + 1] - double(v.y);
                double t2 = q[4 * c4 + 2] - double(v.z), t3 = q[4 * c4 + 3] - double(v.w);
                d = fma(t0, t0, d); d = fma(t1, t1, d); d = fma(t2, t2, d); d = fma(t3, t3, d);
            }
            // exact: every term and partial sum is an integer < 2^53
            if (d < bd[knn - 1]) {
                int idx = base + e;
                double dv = d;
                bool ins = false;
#pragma unroll
                for (int k = 0; k < kKnnMax; ++k) {      // sorted insertion after equal keys;
                    if (k < knn && (ins || dv < bd[k])) {   // displaced entries shift down
                        const double td = bd[k]; const int ti = bi[k];
                        bd[k] = dv; bi[k] = idx; dv = td; idx = ti;
                        ins = true;
                    }
                }
            }
        }
    }
    if (qi < n)
        for (int k = 0; k < knn; ++k) nn[((long long)prob * n + qi) * knn + k] = bi[k];
}

// ------------------------------------------------------------------ fields
// A field f of a batch: pair k = f / fpp, kind = f % fpp; kind 0 matches A_k -> B_k,
// kinds 1, 2 match B_k -> A_k (the two inverse fields, F-5).
struct FieldSet {
    int W, H, fpp, nfields;
    const uint8_t *A, *B;          // level images, pair k at + k * img_stride
    long long img_stride;
    int radius[3];
    uint64_t seed[3];
    int pen64;
    int32_t *flow;                 // [nfields][H][W][2]
    int32_t *cost;                 // [nfields][H][W]
    __device__ __forceinline__ void images(int f, const uint8_t *&src, const uint8_t *&dst) const {
        const int k = f / fpp, kind = f - k * fpp;
        const uint8_t *a = A + k * img_stride, *b = B + k * img_stride;
        src = kind == 0 ? a : b;
        dst = kind == 0 ? b : a;
    }
    __device__ __forceinline__ int kind(int f) const { return f % fpp; }
};

// best of the k candidates (FF5): nn lists per (pair, direction): direction 0 = A->B
__global__ void ff_init_kernel(FieldSet fs, const int32_t *__restrict__ nn, int knn) {
    const long long per = (long long)fs.W * fs.H, total = per * fs.nfields;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int f = int(t / per);
        const long long p = t - f * per;
        const int y = int(p / fs.W), x = int(p - (long long)y * fs.W);
        const uint8_t *src, *dst;
        fs.images(f, src, dst);
        const int kind = fs.kind(f), pair = f / fs.fpp;
        const int dir = kind == 0 ? 0 : 1;
        const int32_t *cand = nn + ((long long)(2 * pair + dir) * per + p) * knn;
        int best = 0x7fffffff, bu = 0, bv = 0;
        for (int k = 0; k < knn; ++k) {
            const int q = cand[k];
            const int yb = q / fs.W, xb = q - yb * fs.W;
            const int fu = (xb - x) * FQ, fv = (yb - y) * FQ;
            const int c = patch_cost_thread(src, dst, fs.W, fs.H, x, y, fu, fv, fs.radius[kind], fs.pen64);
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
        const uint8_t *src, *dst;
        fs.images(f, src, dst);
        fs.flow[2 * t] = fu;
        fs.flow[2 * t + 1] = fv;
        fs.cost[t] = patch_cost_thread(src, dst, fs.W, fs.H, x, y, fu, fv, fs.radius[fs.kind(f)], fs.pen64);
    }
}

// random search (FF7, second half): reads only the pixel's own vector
__global__ void ff_search_kernel(FieldSet fs, int sweep, int level, int R0) {
    const long long per = (long long)fs.W * fs.H, total = per * fs.nfields;
    const int R = max(R0 >> sweep, 1);
    const unsigned span = unsigned(2 * R * FQ + 1);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int f = int(t / per);
        const long long p = t - f * per;
        const int y = int(p / fs.W), x = int(p - (long long)y * fs.W);
        const int kind = fs.kind(f);
        const uint64_t z = splitmix(fs.seed[kind], level, sweep, x, y);
        const int fu = fs.flow[2 * t] + int(unsigned(z) % span) - R * FQ;
        const int fv = fs.flow[2 * t + 1] + int(unsigned(z >> 32) % span) - R * FQ;
        const uint8_t *src, *dst;
        fs.images(f, src, dst);
        const int c = patch_cost_thread(src, dst, fs.W, fs.H, x, y, fu, fv, fs.radius[kind], fs.pen64);
        if (c < fs.cost[t]) {
            fs.cost[t] = c;
            fs.flow[2 * t] = fu;
            fs.flow[2 * t + 1] = fv;
        }
    }
}

// ------------------------------------------------------------------ propagation (FF7)
__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int *p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

struct PropParams {
    FieldSet fs;
    int sweep;
    int nbands;
    int *ticket;       // zeroed before the launch
    int *progress;     // [nfields][nbands], zeroed before the launch
};

template <int NW>
__global__ void __launch_bounds__(NW * 32) ff_prop_kernel(const PropParams pp) {
    const FieldSet &fs = pp.fs;
    const int W = fs.W, H = fs.H;
    extern __shared__ __align__(16) unsigned char ff_smem[];
    int2 *srow = reinterpret_cast<int2 *>(ff_smem);          // [NW][W]
    volatile int *sprog = reinterpret_cast<volatile int *>(srow + (size_t)NW * W);   // [NW]
    __shared__ int s_ticket;
    if (threadIdx.x < NW) sprog[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_ticket = atomicAdd(pp.ticket, 1);
    __syncthreads();
    const int ticket = s_ticket;
    const int f = ticket / pp.nbands, band = ticket - f * pp.nbands;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = band * NW + warp;                 // iteration row
    if (j >= H) return;
    const bool fwd = (pp.sweep & 1) == 0;
    const int y = fwd ? j : H - 1 - j;
    const uint8_t *src, *dst;
    fs.images(f, src, dst);
    const int kind = fs.kind(f);
    const int r = fs.radius[kind], side = 2 * r + 1, ns = side * side;
    const long long per = (long long)W * H;
    int32_t *flow = fs.flow + 2 * f * per;
    int32_t *cost = fs.cost + f * per;
    const bool has_above = j > 0;                   // previous row in scan order exists
    const bool above_in_cta = warp > 0;
    const int *prog_in = pp.progress + f * pp.nbands + band - 1;
    int *prog_out = pp.progress + f * pp.nbands + band;
    const bool publish = warp == NW - 1 && band + 1 < pp.nbands;
    const int yv = fwd ? y - 1 : y + 1;             // row of the vertical candidate
    int known = 0;
    int2 hv = make_int2(0, 0);                      // vector of the previous pixel in scan order
    for (int i = 0; i < W; ++i) {
        const int x = fwd ? i : W - 1 - i;
        const long long p = (long long)y * W + x;
        int cu = flow[2 * p], cv = flow[2 * p + 1], cc = cost[p];
        // vertical candidate: the finished vector of (x, yv)
        int2 vv = make_int2(0, 0);
        if (has_above) {
            if (above_in_cta) {
                while (sprog[warp - 1] < i + 1) { }
                const volatile int *sv = reinterpret_cast<const volatile int *>(srow + (size_t)(warp - 1) * W + x);
                vv = make_int2(sv[0], sv[1]);
            } else {
                if (known < i + 1) {
                    int k;
                    while ((k = ld_acquire_gpu(prog_in)) < min(i + 1, W)) __nanosleep(20);
                    known = k;
                }
                const long long q = (long long)yv * W + x;
                vv = make_int2(__ldcg(flow + 2 * q), __ldcg(flow + 2 * q + 1));
            }
        }
        // candidates in order: horizontal (previous pixel), vertical; skip ones equal to
        // the incumbent (their data term equals the incumbent's: never strictly better)
        const bool eh = i > 0 && (hv.x != cu || hv.y != cv);
        bool ev = has_above && (vv.x != cu || vv.y != cv) && (!eh || vv.x != hv.x || vv.y != hv.y);
        if (eh || ev) {
            int s0 = 0, s1 = 0;
            for (int k = 0; k < kNsMax; ++k) {
                const int sidx = lane + 32 * k;
                if (sidx < ns) {
                    const int dy = sidx / side - r, dx = sidx - (sidx / side) * side - r;
                    const int a = __ldg(src + (long long)clampi(y + dy, 0, H - 1) * W + clampi(x + dx, 0, W - 1));
                    const int bx = (x + dx) * FQ, by = (y + dy) * FQ;
                    if (eh) s0 += sample_cost(dst, W, H, bx + hv.x, by + hv.y, a, fs.pen64);
                    if (ev) s1 += sample_cost(dst, W, H, bx + vv.x, by + vv.y, a, fs.pen64);
                }
            }
            if (eh) {
                const int c0 = int(__reduce_add_sync(0xffffffffu, unsigned(s0)));
                if (c0 < cc) { cc = c0; cu = hv.x; cv = hv.y; }
            }
            if (ev) {
                const int c1 = int(__reduce_add_sync(0xffffffffu, unsigned(s1)));
                if (c1 < cc) { cc = c1; cu = vv.x; cv = vv.y; }
            }
        }
        if (lane == 0) {
            flow[2 * p] = cu;
            flow[2 * p + 1] = cv;
            cost[p] = cc;
            srow[(size_t)warp * W + x] = make_int2(cu, cv);
        }
        hv = make_int2(cu, cv);
        if (lane == 0) {
            __threadfence_block();
            sprog[warp] = i + 1;
            if (publish && ((i + 1) % kPubFF == 0 || i == W - 1)) st_release_gpu(prog_out, i + 1);
        }
        __syncwarp();
    }
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
__global__ void ff_cost_query_kernel(const uint8_t *A, const uint8_t *B, int W, int H, int r, int pen64,
                                     int nq, const int32_t *q, int32_t *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nq) out[i] = patch_cost_thread(A, B, W, H, q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3], r, pen64);
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

cudaError_t ff_launch_knn(const int32_t *desc, int n, int nprob, int knn, int32_t *nn, cudaStream_t st) {
    if (knn < 1 || knn > kKnnMax) return cudaErrorInvalidValue;
    dim3 grid((n + 127) / 128, nprob);
    ff_knn_kernel<<<grid, 128, 0, st>>>(desc, n, knn, nn);
    return cudaGetLastError();
}

static FieldSet make_fs(const FFFields &F) {
    FieldSet fs{};
    fs.W = F.W; fs.H = F.H; fs.fpp = F.fpp; fs.nfields = F.nfields;
    fs.A = F.A; fs.B = F.B; fs.img_stride = F.img_stride;
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

constexpr int kPropNW = 8;

size_t ff_prop_smem(int W) { return size_t(kPropNW) * W * sizeof(int2) + 64; }

cudaError_t ff_launch_sweep(const FFFields &F, int sweep, int level, int R0, int *sync, cudaStream_t st,
                            int *launches) {
    PropParams pp{};
    pp.fs = make_fs(F);
    pp.sweep = sweep;
    pp.nbands = (F.H + kPropNW - 1) / kPropNW;
    pp.ticket = sync;
    pp.progress = sync + 1;
    cudaError_t e = cudaMemsetAsync(sync, 0, sizeof(int) * (1 + size_t(F.nfields) * pp.nbands), st);
    if (e != cudaSuccess) return e;
    const size_t sm = ff_prop_smem(F.W);
    e = cudaFuncSetAttribute(ff_prop_kernel<kPropNW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    if (e != cudaSuccess) return e;
    ff_prop_kernel<kPropNW><<<F.nfields * pp.nbands, kPropNW * 32, sm, st>>>(pp);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const long long n = (long long)F.W * F.H * F.nfields;
    ff_search_kernel<<<ff_grid(n, 128), 128, 0, st>>>(pp.fs, sweep, level, R0);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (launches) *launches += 2;
    return cudaSuccess;
}

int ff_sync_ints(int nfields, int H) { return 1 + nfields * ((H + kPropNW - 1) / kPropNW); }

cudaError_t ff_launch_consistency(const int32_t *F, const int32_t *G1, const int32_t *G2, long long fstride,
                                  long long gstride, int W, int H, int n, int thr_q, uint8_t *valid,
                                  float *fout, cudaStream_t st) {
    ff_consistency_kernel<<<ff_grid((long long)W * H * n, 256), 256, 0, st>>>(F, G1, G2, fstride, gstride, W, H,
                                                                                n, thr_q, valid, fout);
    return cudaGetLastError();
}

cudaError_t ff_launch_cost_query(const uint8_t *A, const uint8_t *B, int W, int H, int r, int penalty, int nq,
                                 const int32_t *q, int32_t *out, cudaStream_t st) {
    ff_cost_query_kernel<<<(nq + 127) / 128, 128, 0, st>>>(A, B, W, H, r, penalty * FQ2, nq, q, out);
    return cudaGetLastError();
}

}  // namespace sgm
