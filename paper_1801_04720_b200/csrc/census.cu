// census.cu -- census transform (G2-G4) with TMA-staged shared-memory tiles.
//
// out[y][x] bit k = [I(clamp(x+dx), clamp(y+dy)) < I(x, y)] for the k-th neighbour of the
// census_w x census_h window scanned row-major (dy outer, dx inner), centre skipped.
//
// Each CTA owns a 64 x 16 output tile.  One elected thread issues a 3D
// cp.async.bulk.tensor (TMA) for the tile plus its halo -- box {96, 16 + 2*ry, 1} of the
// image stack [nimg][H][pitch] -- into shared memory, completing on an mbarrier with
// expect_tx.  TMA fills out-of-image texels with zeros, not with the clamped border the
// method needs, so every neighbour read goes through clamped image coordinates; the box
// always contains the clamped texel (it spans [x0-16, x0+80) x [y0-ry, y0+16+ry)).  The box
// x origin is x0-16, not x0-rx: TMA requires the innermost start coordinate times the
// element size to be a multiple of 16 bytes.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "sgm_internal.cuh"

#ifndef SGM_CENSUS_SIMD
#define SGM_CENSUS_SIMD 1
#endif

namespace sgm {
namespace {

constexpr int kTileW = 64;
constexpr int kTileH = 16;
constexpr int kHaloX = 16;         // TMA box x origin must be 16-byte aligned: start at x0-16
constexpr int kBoxW = kTileW + 2 * kHaloX;   // 96 bytes, covers rx <= 16
constexpr int kThreads = 256;

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int CW, int CH>
__device__ __forceinline__ uint64_t census_px(const uint8_t *s, int bh, int gx, int gy, int ox,
                                              int oy, int W, int H, int cw_rt, int ch_rt) {
    const int cw = CW > 0 ? CW : cw_rt;
    const int ch = CH > 0 ? CH : ch_rt;
    const int rx = cw / 2, ry = ch / 2;
    (void)bh;
    const int c = s[(gy - oy) * kBoxW + (gx - ox)];
    uint64_t bits = 0;
    int k = 0;
#pragma unroll
    for (int dy = -ry; dy <= ry; ++dy) {
        int yy = gy + dy;
        yy = yy < 0 ? 0 : (yy > H - 1 ? H - 1 : yy);
        const uint8_t *row = s + (yy - oy) * kBoxW;
#pragma unroll
        for (int dx = -rx; dx <= rx; ++dx) {
            if (dx == 0 && dy == 0) continue;
            int xx = gx + dx;
            xx = xx < 0 ? 0 : (xx > W - 1 ? W - 1 : xx);
            const int n = row[xx - ox];
            bits |= uint64_t(n < c) << k;
            ++k;
        }
    }
    return bits;
}

// interior tiles: every window sample inside the image, no clamping (the common case)
template <int CW, int CH>
__device__ __forceinline__ uint64_t census_px_in(const uint8_t *s, int lx, int ly) {
    constexpr int rx = CW / 2, ry = CH / 2;
    const uint8_t *ctr = s + (ly + ry) * kBoxW + (lx + kHaloX);
    const int c = ctr[0];
    uint32_t lo = 0, hi = 0;
    int k = 0;
#pragma unroll
    for (int dy = -ry; dy <= ry; ++dy) {
#pragma unroll
        for (int dx = -rx; dx <= rx; ++dx) {
            if (dx == 0 && dy == 0) continue;
            const uint32_t bit = uint32_t(int(ctr[dy * kBoxW + dx]) < c);
            if (k < 32) lo |= bit << k;
            else hi |= bit << (k - 32);
            ++k;
        }
    }
    return uint64_t(lo) | (uint64_t(hi) << 32);
}

// Four horizontally adjacent interior pixels (x = 4a .. 4a+3 of the tile row ly) at once,
// byte-SIMD: the four centres are the bytes of one word C; for each window offset the four
// neighbours are the bytes of one word N (a PRMT funnel of two aligned row words), and the
// four comparisons N < C are one unsigned per-byte less-than in three ALU ops:
//   lt(bit 7 of each byte) = (~n & c) | (~(n ^ c) & ~d),   d = (n | 0x80..) - (c & 0x7f..)
// (d's byte b has bit 7 set iff n_b mod 128 >= c_b mod 128; no borrow crosses bytes).
// Window bit k of pixel j goes to bit k % 8 of byte j of acc[k / 8]; a final byte transpose
// turns acc[0..7] into the four 64-bit census words (byte g = acc[g] byte j).
template <int CW, int CH>
__device__ __forceinline__ void census_px4_in(const uint8_t *s, int lx, int ly, uint64_t (&out)[4]) {
    constexpr int rx = CW / 2, ry = CH / 2;
    static_assert(rx <= 4, "window wider than 9 needs more row words");
    constexpr int NB = (CW * CH - 1 + 7) / 8;          // census bytes in use
    const uint32_t *ctr = reinterpret_cast<const uint32_t *>(s + (ly + ry) * kBoxW + (lx + kHaloX));
    const uint32_t c = ctr[0];
    const uint32_t c7f = c & 0x7f7f7f7fu;
    uint32_t acc[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) acc[g] = 0;
    int k = 0;
#pragma unroll
    for (int dy = -ry; dy <= ry; ++dy) {
        const uint32_t *row = ctr + dy * (kBoxW / 4);
        const uint32_t w0 = row[-1], w1 = row[0], w2 = row[1];
#pragma unroll
        for (int dx = -rx; dx <= rx; ++dx) {
            if (dx == 0 && dy == 0) continue;
            // bytes x+dx .. x+dx+3
            const uint32_t n = dx < 0 ? __byte_perm(w0, w1, 0x3210 + 0x1111 * (4 + dx))
                                      : (dx == 0 ? w1 : __byte_perm(w1, w2, 0x3210 + 0x1111 * dx));
            const uint32_t d = (n | 0x80808080u) - c7f;
            const uint32_t lt = (~n & c) | (~(n ^ c) & ~d);      // bit 7 of each byte
            const int g = k >> 3, b = k & 7;
            acc[g] |= (lt >> (7 - b)) & (0x01010101u << b);
            ++k;
        }
    }
    // byte transpose: out[j] byte g = acc[g] byte j
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t sel = uint32_t(j) | (uint32_t(j + 4) << 4);   // bytes j of (a, b)
        const uint32_t lo01 = __byte_perm(acc[0], acc[1], sel);
        const uint32_t lo23 = __byte_perm(acc[2], acc[3], sel);
        const uint32_t hi45 = NB > 4 ? __byte_perm(acc[4], acc[5], sel) : 0u;
        const uint32_t hi67 = NB > 6 ? __byte_perm(acc[6], acc[7], sel) : 0u;
        const uint32_t lo = __byte_perm(lo01, lo23, 0x5410);
        const uint32_t hi = __byte_perm(hi45, hi67, 0x5410);
        out[j] = uint64_t(lo) | (uint64_t(hi) << 32);
    }
}

template <int CW, int CH>
__global__ void __launch_bounds__(kThreads) census_kernel(const __grid_constant__ CUtensorMap tmap,
                                                          CensusParams prm, uint64_t *out,
                                                          long long out_stride) {
    const int cw = CW > 0 ? CW : prm.cw;
    const int ch = CH > 0 ? CH : prm.ch;
    (void)cw;
    const int ry = ch / 2;
    const int bh = kTileH + 2 * ry;
    __shared__ __align__(128) uint8_t tile[kBoxW * (kTileH + 2 * 8)];
    __shared__ __align__(8) unsigned long long mbar;

    const int x0 = blockIdx.x * kTileW, y0 = blockIdx.y * kTileH, img = blockIdx.z;
    const int ox = x0 - kHaloX, oy = y0 - ry;       // image coords of tile[0][0]
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        const unsigned bytes = unsigned(kBoxW * bh);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(&mbar)),
                     "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(tile)),
            "l"(&tmap), "r"(ox), "r"(oy), "r"(img), "r"(smem_u32(&mbar))
            : "memory");
    }
    __syncthreads();
    {
        unsigned done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], 0;\n"
                " selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(smem_u32(&mbar))
                : "memory");
        }
    }
    uint64_t *o = out + (long long)img * out_stride;
    if (CW > 0 && x0 - CW / 2 >= 0 && x0 + kTileW + CW / 2 <= prm.W && y0 - CH / 2 >= 0 &&
        y0 + kTileH + CH / 2 <= prm.H) {
        if (SGM_CENSUS_SIMD && CW > 0 && CW <= 9) {
            static_assert(kTileW * kTileH == 4 * kThreads, "one 4-pixel group per thread");
            const int lx = 4 * (threadIdx.x % (kTileW / 4)), ly = threadIdx.x / (kTileW / 4);
            uint64_t v[4];
            census_px4_in<(CW > 0 && CW <= 9 ? CW : 1), (CH > 0 ? CH : 1)>(tile, lx, ly, v);
            ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(o + (long long)(y0 + ly) * prm.W + x0 + lx);
            if (((reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
                dst[0] = make_ulonglong2(v[0], v[1]);
                dst[1] = make_ulonglong2(v[2], v[3]);
            } else {
                uint64_t *d1 = o + (long long)(y0 + ly) * prm.W + x0 + lx;
                d1[0] = v[0]; d1[1] = v[1]; d1[2] = v[2]; d1[3] = v[3];
            }
        } else {
            for (int k = threadIdx.x; k < kTileW * kTileH; k += kThreads) {
                const int lx = k % kTileW, ly = k / kTileW;
                o[(long long)(y0 + ly) * prm.W + x0 + lx] =
                    census_px_in<(CW > 0 ? CW : 1), (CH > 0 ? CH : 1)>(tile, lx, ly);
            }
        }
        return;
    }
    for (int k = threadIdx.x; k < kTileW * kTileH; k += kThreads) {
        const int lx = k % kTileW, ly = k / kTileW;
        const int gx = x0 + lx, gy = y0 + ly;
        if (gx < prm.W && gy < prm.H)
            o[(long long)gy * prm.W + gx] =
                census_px<CW, CH>(tile, bh, gx, gy, ox, oy, prm.W, prm.H, cw, ch);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

}  // namespace

// imgs: nimg images with a constant stride (img_stride bytes) starting at base.
cudaError_t launch_census_stack(const uint8_t *base, long long img_stride, int nimg, long long pitch,
                                int W, int H, int cw, int ch, uint64_t *out, long long out_stride,
                                cudaStream_t st) {
    auto enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (pitch & 15) || (img_stride & 15) || ch / 2 > 8 ||
        cw / 2 > kHaloX)
        return cudaErrorInvalidValue;
    CUtensorMap tmap;
    const int ry = ch / 2;
    cuuint64_t dims[3] = {cuuint64_t(W), cuuint64_t(H), cuuint64_t(nimg)};
    cuuint64_t strides[2] = {cuuint64_t(pitch), cuuint64_t(img_stride)};
    cuuint32_t box[3] = {cuuint32_t(kBoxW), cuuint32_t(kTileH + 2 * ry), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t *>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    CensusParams prm{W, H, cw, ch, nimg};
    dim3 grid((W + kTileW - 1) / kTileW, (H + kTileH - 1) / kTileH, nimg);
    if (cw == 9 && ch == 7)
        census_kernel<9, 7><<<grid, kThreads, 0, st>>>(tmap, prm, out, out_stride);
    else if (cw == 5 && ch == 5)
        census_kernel<5, 5><<<grid, kThreads, 0, st>>>(tmap, prm, out, out_stride);
    else
        census_kernel<0, 0><<<grid, kThreads, 0, st>>>(tmap, prm, out, out_stride);
    return cudaGetLastError();
}

cudaError_t launch_census(const uint8_t *const *imgs, int nimg, long long pitch, int W, int H,
                          int cw, int ch, uint64_t *out, long long out_stride, cudaStream_t st) {
    // independent pointers: one launch per image
    for (int i = 0; i < nimg; ++i) {
        cudaError_t e = launch_census_stack(imgs[i], (long long)H * pitch, 1, pitch, W, H, cw, ch,
                                            out + (long long)i * out_stride, out_stride, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace sgm
