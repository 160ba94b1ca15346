// small_kernels.cu -- the bandwidth-bound stages of the hot path (sm_100a):
//   cost_kernel     materialised matching cost (debug / parity path)
//   wta_kernel      WTA + parabola on a materialised S (stage-wise API)
//   lr_kernel       integer left-right check (G13)
//   combine_kernel  Eq. (4)/(5) warp of D1 through the flow + 3D
#include "sgm_internal.cuh"

namespace sgm {
namespace {

// ------------------------------------------------------------------ cost (debug path)
// One thread per (x, y, d); C = popcount(ref(x) ^ match(x + s d)), C_max outside.
__global__ void cost_kernel(const uint64_t *__restrict__ ref, const uint64_t *__restrict__ match,
                            int W, int H, int D, int s, int cmax, uint8_t *__restrict__ cost) {
    const long long n = (long long)W * H * D;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const int d = int(idx % D);
        const long long px = idx / D;
        const int x = int(px % W);
        const long long rowbase = px - x;
        const int xm = x + s * d;
        int c = cmax;
        if (xm >= 0 && xm < W) c = __popcll(ref[px] ^ match[rowbase + xm]);
        cost[idx] = uint8_t(c);
    }
}

// ------------------------------------------------------------------ WTA (stage-wise)
// One warp per pixel; key = S * 256 + d gives the smallest-index argmin (G10).
__global__ void wta_kernel(const uint16_t *__restrict__ agg, int W, int H, int D,
                           int16_t *__restrict__ dint, float *__restrict__ dsub) {
    const int lane = threadIdx.x & 31;
    const long long npx = (long long)W * H;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long p = warp; p < npx; p += nwarps) {
        const uint16_t *s = agg + p * D;
        unsigned best = 0xffffffffu;
        for (int d = lane; d < D; d += 32) best = min(best, (unsigned(s[d]) << 8) | unsigned(d));
        best = __reduce_min_sync(0xffffffffu, best);
        const int ds = int(best & 0xffu), sb = int(best >> 8);
        float sub = float(ds);
        if (ds > 0 && ds < D - 1) {
            const int sa = s[ds - 1], sc = s[ds + 1];
            const int den = 2 * (sa + sc - 2 * sb);
            float off = 0.f;
            if (den != 0) off = __fdiv_rn(float(sa - sc), float(den));
            off = fminf(fmaxf(off, -0.5f), 0.5f);
            sub = __fadd_rn(float(ds), off);
        }
        if (lane == 0) { dint[p] = int16_t(ds); dsub[p] = sub; }
    }
}

// ------------------------------------------------------------------ LR check
// grid (ceil(W / blockDim.x), H, pairs): no index division (a 64-bit division per pixel
// made these small kernels instruction-bound)
__global__ void lr_kernel(const LrParams p) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= p.W) return;
    const long long pair = blockIdx.z;
    const int px = int(blockIdx.y) * p.W + x;      // W * H < 2^31 (sgm_create)
    {
        const int16_t *dl = p.dl + pair * p.in_stride_l;
        const float *dls = p.dls + pair * p.in_stride_l;
        const int16_t *dr = p.dr + pair * p.in_stride_r;
        const int d = dl[px];
        const int xr = x - d;
        bool ok = false;
        if (xr >= 0 && xr < p.W) {
            const int e = dr[px - x + xr];
            ok = abs(d - e) <= p.T;
        }
        const long long o = pair * p.out_stride + px;
        if (p.out_int) p.out_int[o] = ok ? int16_t(d) : int16_t(p.invalid);
        if (p.out_sub) p.out_sub[o] = ok ? dls[px] : float(p.invalid);
        if (p.valid) p.valid[o] = ok ? 1 : 0;
    }
}

// ------------------------------------------------------------------ combination + 3D
// One thread per pixel, float4 stores.  Validity decisions are taken in float32 exactly
// like the oracle's (x' = (float)x + u, floor, fractional part, taps with nonzero weight).
//
// LRF (production path when the caller takes no disparity maps): the LR check (G13) is
// fused in -- validity and value of D0 at x and of D1 at the four taps are derived from the raw
// WTA maps on the fly (valid iff x - d_L >= 0 and |d_L - d_R(x - d_L)| <= T; an invalid tap's
// value is invalid_disp, exactly what lr_kernel would have stored), so the LR-checked maps are
// never written or read and the LR launch disappears.  Same arithmetic, same results.
template <bool LRF>
__global__ void combine_kernel(const CombineParams p) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= p.W) return;
    const int y = blockIdx.y;
    const long long q = blockIdx.z;
    const long long npx = (long long)p.W * p.H;
    const long long px = (long long)y * p.W + x, idx = q * npx + px;
    {
        const float2 uv = reinterpret_cast<const float2 *>(p.flow)[idx];
        const float *d0 = LRF ? nullptr : p.d0 + q * p.disp_stride;
        const float *d1 = LRF ? nullptr : p.d1 + q * p.disp_stride;
        const uint8_t *v0 = LRF ? nullptr : p.v0 + q * p.disp_stride;
        const uint8_t *v1 = LRF ? nullptr : p.v1 + q * p.disp_stride;
        // fused LR: raw maps of the left / right views of the two pairs of this quad
        const long long vw0 = LRF ? 2 * (q * p.pair_step) * p.view_stride : 0;
        const int16_t *l0 = LRF ? p.raw_int + vw0 : nullptr, *l1 = LRF ? l0 + 2 * p.view_stride : nullptr;
        const float *s0 = LRF ? p.raw_sub + vw0 : nullptr, *s1 = LRF ? s0 + 2 * p.view_stride : nullptr;
        auto lr_ok = [&](const int16_t *L, long long row, int xx) {
            const int d = L[row + xx];
            const int xr = xx - d;
            return xr >= 0 && xr < p.W && abs(d - int(L[p.view_stride + row + xr])) <= p.T;
        };
        bool ok = (p.flow_valid == nullptr || p.flow_valid[idx]) &&
                  (LRF ? lr_ok(l0, px - x, x) : bool(v0[px]));
        const float xp = __fadd_rn(float(x), uv.x), yp = __fadd_rn(float(y), uv.y);
        ok = ok && (xp >= 0.f && xp <= float(p.W - 1) && yp >= 0.f && yp <= float(p.H - 1));
        float d1w = 0.f, d0v = 0.f;
        if (ok) {
            const int x0 = int(floorf(xp)), y0 = int(floorf(yp));
            const float fx = __fsub_rn(xp, float(x0)), fy = __fsub_rn(yp, float(y0));
            const int x1 = min(x0 + 1, p.W - 1), y1 = min(y0 + 1, p.H - 1);
            const long long q00 = (long long)y0 * p.W + x0, q10 = (long long)y0 * p.W + x1;
            const long long q01 = (long long)y1 * p.W + x0, q11 = (long long)y1 * p.W + x1;
            bool t00, t10, t01, t11;
            if (LRF) {
                const long long r0 = (long long)y0 * p.W, r1 = (long long)y1 * p.W;
                t00 = lr_ok(l1, r0, x0); t10 = lr_ok(l1, r0, x1);
                t01 = lr_ok(l1, r1, x0); t11 = lr_ok(l1, r1, x1);
            } else {
                t00 = v1[q00]; t10 = v1[q10]; t01 = v1[q01]; t11 = v1[q11];
            }
            bool tv;
            if (p.rule == 1) {
                tv = t00 && t10 && t01 && t11;
            } else {
                tv = t00 && (fx == 0.f || t10) && (fy == 0.f || t01) && (fx == 0.f || fy == 0.f || t11);
            }
            ok = tv;
            if (ok) {
                // Eq. (5) in the paper's term order; zero-weight taps contribute exactly 0
                // (their values are finite: invalid disparities are -1, never NaN, G14).
                const float ax = fx, ay = fy, bx = 1.f - fx, by = 1.f - fy;
                const float e00 = LRF ? s1[q00] : d1[q00];
                const float e10 = LRF ? (t10 ? s1[q10] : p.invalid) : d1[q10];
                const float e01 = LRF ? (t01 ? s1[q01] : p.invalid) : d1[q01];
                const float e11 = LRF ? (t11 ? s1[q11] : p.invalid) : d1[q11];
                float acc = __fmul_rn(__fmul_rn(e00, bx), by);
                acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(e10, ax), by));
                acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(e01, bx), ay));
                acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(e11, ax), ay));
                d1w = acc;
                d0v = LRF ? s0[px] : d0[px];
            }
        }
        float4 s = ok ? make_float4(uv.x, uv.y, d0v, d1w) : make_float4(0.f, 0.f, 0.f, 0.f);
        reinterpret_cast<float4 *>(p.sf)[idx] = s;
        p.valid_sf[idx] = ok ? 1 : 0;
        if (p.dp != nullptr) {
            const bool ok3 = ok && d0v > 0.f && d1w > 0.f;
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
            if (ok3) {
                const float Z0 = __fdiv_rn(p.fB, d0v);
                const float X0 = __fdiv_rn(__fmul_rn(__fsub_rn(float(x), p.cx), Z0), p.f);
                const float Y0 = __fdiv_rn(__fmul_rn(__fsub_rn(float(y), p.cy), Z0), p.f);
                const float Z1 = __fdiv_rn(p.fB, d1w);
                const float X1 = __fdiv_rn(__fmul_rn(__fsub_rn(xp, p.cx), Z1), p.f);
                const float Y1 = __fdiv_rn(__fmul_rn(__fsub_rn(yp, p.cy), Z1), p.f);
                a = make_float4(X0, Y0, Z0, 0.f);
                b = make_float4(__fsub_rn(X1, X0), __fsub_rn(Y1, Y0), __fsub_rn(Z1, Z0), 0.f);
            }
            if (p.p0 != nullptr) reinterpret_cast<float4 *>(p.p0)[idx] = a;
            reinterpret_cast<float4 *>(p.dp)[idx] = b;
            p.valid_3d[idx] = ok3 ? 1 : 0;
        }
    }
}

// ------------------------------------------------------------------ re-pitch (host entry)
// Dense [rows][W] uint8 -> [rows][pitch]: host images arrive by one 1D copy (a pitched
// 2D copy of 1242-byte rows runs at ~9 GB/s on PCIe, a 1D copy at ~54 GB/s).
__global__ void repitch_kernel(const uint8_t *__restrict__ src, uint8_t *__restrict__ dst, int W,
                               long long pitch, long long rows) {
    const long long n = rows * W;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long r = idx / W;
        dst[r * pitch + (idx - r * W)] = src[idx];
    }
}

int grid_for(long long n, int block) {
    long long g = (n + block - 1) / block;
    const long long cap = 148LL * 16;
    return int(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

cudaError_t launch_cost(const uint64_t *ref, const uint64_t *match, int W, int H, int D, int s,
                        int cmax, uint8_t *cost, cudaStream_t st) {
    const long long n = (long long)W * H * D;
    cost_kernel<<<grid_for(n, 256), 256, 0, st>>>(ref, match, W, H, D, s, cmax, cost);
    return cudaGetLastError();
}

cudaError_t launch_wta(const uint16_t *agg, int W, int H, int D, int16_t *dint, float *dsub,
                       cudaStream_t st) {
    const long long n = (long long)W * H * 32;
    wta_kernel<<<grid_for(n, 256), 256, 0, st>>>(agg, W, H, D, dint, dsub);
    return cudaGetLastError();
}

cudaError_t launch_repitch(const uint8_t *src, uint8_t *dst, int W, long long pitch, long long rows,
                           cudaStream_t st) {
    repitch_kernel<<<grid_for(rows * W, 256), 256, 0, st>>>(src, dst, W, pitch, rows);
    return cudaGetLastError();
}

cudaError_t launch_lr(const LrParams &p, cudaStream_t st) {
    if (p.npairs < 1 || p.npairs > 65535 || p.H > 65535) return cudaErrorInvalidValue;
    lr_kernel<<<dim3((p.W + 127) / 128, p.H, p.npairs), 128, 0, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_combine(const CombineParams &p, cudaStream_t st) {
    if (p.nquads < 1 || p.nquads > 65535 || p.H > 65535) return cudaErrorInvalidValue;
    const dim3 grid((p.W + 127) / 128, p.H, p.nquads);
    if (p.raw_int != nullptr) combine_kernel<true><<<grid, 128, 0, st>>>(p);
    else combine_kernel<false><<<grid, 128, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace sgm
