// densify.cu -- edge-aware densification of a sparse field (SPEC
// densify S:253-262, F-6; the gap filling of P:87 and the "Ours (All)" densification of
// P:147 / P:170).  Readings DN1-DN4: a gap pixel p takes the weighted mean of
// its K nearest valid seeds (squared Euclidean distance, ties to the smaller linear index),
// weight 1 / (|p - s| + lambda * sum of the guide's L1 central-difference gradient over the
// interior points of the segment p -> s).
//
// One thread per pixel.  The K nearest seeds come from a ring search: rings of Chebyshev
// radius r = 1, 2, ... are enumerated (sides without any valid pixel skipped in O(1) with
// per-row / per-column prefix counts, so wide holes cost O(radius)) and offered to a
// (distance^2 << 32 | index)-keyed top-K list; the search stops once K seeds are held and
// r^2 exceeds the K-th distance^2 (every later pixel is at least r away), which is exactly
// the exhaustive result.
#include "sgm_internal.cuh"

namespace sgm {
namespace {

constexpr int kDensifyKMax = 64;

__device__ __forceinline__ int grad_l1(const uint8_t *__restrict__ G, int W, int H, int x, int y) {
    const int gx = int(__ldg(G + (long long)y * W + min(x + 1, W - 1))) - int(__ldg(G + (long long)y * W + max(x - 1, 0)));
    const int gy = int(__ldg(G + (long long)min(y + 1, H - 1) * W + x)) - int(__ldg(G + (long long)max(y - 1, 0) * W + x));
    return abs(gx) + abs(gy);
}

struct SeedList {
    unsigned long long key[kDensifyKMax];   // (d^2 << 32) | linear index
};

__device__ __noinline__ unsigned long long seed_insert(SeedList *L, int &cnt, int K, unsigned long long k) {
    int pos = cnt < K ? cnt++ : K - 1;
    while (pos > 0 && L->key[pos - 1] > k) {
        L->key[pos] = L->key[pos - 1];
        --pos;
    }
    L->key[pos] = k;
    return cnt == K ? L->key[K - 1] : ~0ull;
}

// Per-image prefix counts of valid pixels along rows (rowc[img][y][x] = #valid in row y,
// columns < x; W+1 entries per row) and along columns (colc[img][x][y], H+1 per column):
// the ring search skips empty ring sides in O(1).
__global__ void densify_rowcount_kernel(const DensifyParams p, int *__restrict__ rowc) {
    const int rows = p.H * p.n;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        const uint8_t *v = p.valid + (long long)r * p.W;
        int *o = rowc + (long long)r * (p.W + 1);
        int c = 0;
        o[0] = 0;
        for (int x = 0; x < p.W; ++x) { c += v[x] != 0; o[x + 1] = c; }
    }
}
// the guide's L1 gradient g(q) per pixel (DN3), so a segment walk reads one value per step
__global__ void densify_grad_kernel(const DensifyParams p, uint16_t *__restrict__ grad) {
    const long long per = (long long)p.W * p.H, total = per * p.n;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int img = int(t / per);
        const long long q = t - img * per;
        const int y = int(q / p.W), x = int(q - (long long)y * p.W);
        grad[t] = uint16_t(grad_l1(p.guide + img * per, p.W, p.H, x, y));
    }
}

__global__ void densify_colcount_kernel(const DensifyParams p, int *__restrict__ colc) {
    const int cols = p.W * p.n;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cols; t += gridDim.x * blockDim.x) {
        const int img = t / p.W, x = t - img * p.W;
        const uint8_t *v = p.valid + (long long)img * p.W * p.H + x;
        int *o = colc + ((long long)img * p.W + x) * (p.H + 1);
        int c = 0;
        o[0] = 0;
        for (int y = 0; y < p.H; ++y) { c += v[(long long)y * p.W] != 0; o[y + 1] = c; }
    }
}

// floor((2 k a + n) / (2 n)) for k = 1, 2, ... (round-half-up of k a / n), stepped
// incrementally: quotient q and remainder m of (2 k a + n) by 2 n, |2 a| <= 2 n
struct RoundStep {
    int q, m, a2, n2;
    __device__ __forceinline__ RoundStep(int a, int n) : q(0), m(n), a2(2 * a), n2(2 * n) {}
    __device__ __forceinline__ int next() {
        m += a2;
        if (m >= n2) { m -= n2; ++q; }
        else if (m < 0) { m += n2; --q; }
        return q;
    }
};

__global__ void densify_kernel(const DensifyParams p, const int *__restrict__ rowc, const int *__restrict__ colc,
                               const uint16_t *__restrict__ grad) {
    const long long per = (long long)p.W * p.H, total = per * p.n;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int img = int(t / per);
        const long long q = t - img * per;
        const int y = int(q / p.W), x = int(q - (long long)y * p.W);
        const uint8_t *valid = p.valid + img * per;
        const float *field = p.field + img * per * p.C;
        float *out = p.out + t * p.C;
        if (valid[q]) {
            for (int c = 0; c < p.C; ++c) out[c] = field[q * p.C + c];
            continue;
        }
        SeedList L;
        int cnt = 0;
        unsigned long long kth = ~0ull;             // admission bound (K-th key once full)
        const int rmax = max(p.W, p.H);
        for (int r = 1; r <= rmax; ++r) {
            if (cnt == p.K && (unsigned long long)r * r > (kth >> 32)) break;
            // ring of Chebyshev radius r: rows y - r, y + r (full), columns x - r, x + r;
            // each side is clipped to the image and skipped when its prefix count is zero
            for (int side = 0; side < 4; ++side) {
                int fixed, lo, hi;                  // the side's fixed coordinate and range
                if (side < 2) {
                    fixed = side == 0 ? y - r : y + r;
                    if (fixed < 0 || fixed >= p.H) continue;
                    lo = max(x - r, 0); hi = min(x + r, p.W - 1);
                    const int *rc = rowc + ((long long)img * p.H + fixed) * (p.W + 1);
                    if (lo > hi || rc[hi + 1] == rc[lo]) continue;
                } else {
                    fixed = side == 2 ? x - r : x + r;
                    if (fixed < 0 || fixed >= p.W) continue;
                    lo = max(y - r + 1, 0); hi = min(y + r - 1, p.H - 1);
                    const int *cc = colc + ((long long)img * p.W + fixed) * (p.H + 1);
                    if (lo > hi || cc[hi + 1] == cc[lo]) continue;
                }
                for (int k = lo; k <= hi; ++k) {
                    const int sx = side < 2 ? k : fixed, sy = side < 2 ? fixed : k;
                    const long long sq = (long long)sy * p.W + sx;
                    if (!valid[sq]) continue;
                    const int dx = sx - x, dy = sy - y;
                    const unsigned long long key = ((unsigned long long)(dx * dx + dy * dy) << 32) | unsigned(sq);
                    if (key < kth) kth = seed_insert(&L, cnt, p.K, key);
                }
            }
        }
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        float wsum = 0.f;
        for (int k = 0; k < cnt; ++k) {
            const int sq = int(L.key[k] & 0xffffffffu);
            const int sy = sq / p.W, sx = sq - sy * p.W;
            const int dx = sx - x, dy = sy - y;
            const int n = max(abs(dx), abs(dy));
            int g = 0;
            RoundStep rx(dx, n), ry(dy, n);
            const uint16_t *gi = grad + img * per;
            for (int j = 1; j < n; ++j) {
                const int qx = x + rx.next(), qy = y + ry.next();
                g += __ldg(gi + (long long)qy * p.W + qx);
            }
            const float w = 1.0f / (sqrtf(float(dx * dx + dy * dy)) + p.lambda * float(g));
            wsum += w;
            for (int c = 0; c < p.C; ++c) acc[c] = fmaf(w, field[(long long)sq * p.C + c], acc[c]);
        }
        if (cnt == 0) {
            for (int c = 0; c < p.C; ++c) out[c] = 0.f;
            if (p.unfilled) atomicAdd(p.unfilled, 1);
        } else {
            for (int c = 0; c < p.C; ++c) out[c] = acc[c] / wsum;
        }
    }
}

}  // namespace

size_t densify_scratch_bytes(int n, int W, int H) {
    const size_t rown = size_t(n) * H * (W + 1), coln = size_t(n) * W * (H + 1);
    const size_t npx = size_t(n) * W * H;
    return sizeof(int) * (rown + coln) + 2 * npx + 16;
}

cudaError_t launch_densify(const DensifyParams &p, void *scratch_in, cudaStream_t st) {
    if (p.K < 1 || p.K > kDensifyKMax) return cudaErrorInvalidValue;
    cudaError_t e = cudaSuccess;
    if (p.unfilled) e = cudaMemsetAsync(p.unfilled, 0, sizeof(int), st);
    // prefix counts + gradient image: caller scratch, else stream-ordered allocation
    const size_t rown = size_t(p.n) * p.H * (p.W + 1), coln = size_t(p.n) * p.W * (p.H + 1);
    int *scratch = reinterpret_cast<int *>(scratch_in);
    if (!scratch && e == cudaSuccess)
        e = cudaMallocAsync(reinterpret_cast<void **>(&scratch), densify_scratch_bytes(p.n, p.W, p.H), st);
    if (e != cudaSuccess) return e;
    int *rowc = scratch, *colc = scratch + rown;
    uint16_t *grad = reinterpret_cast<uint16_t *>(colc + coln);
    densify_rowcount_kernel<<<(p.H * p.n + 127) / 128, 128, 0, st>>>(p, rowc);
    e = cudaGetLastError();
    if (e == cudaSuccess) densify_colcount_kernel<<<(p.W * p.n + 127) / 128, 128, 0, st>>>(p, colc);
    if (e == cudaSuccess) e = cudaGetLastError();
    const long long total = (long long)p.W * p.H * p.n;
    long long g = (total + 127) / 128;
    if (g > 148LL * 32) g = 148LL * 32;
    if (e == cudaSuccess) densify_grad_kernel<<<unsigned(g < 1 ? 1 : g), 128, 0, st>>>(p, grad);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) densify_kernel<<<unsigned(g < 1 ? 1 : g), 128, 0, st>>>(p, rowc, colc, grad);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (!scratch_in) {
        const cudaError_t e2 = cudaFreeAsync(scratch, st);
        if (e == cudaSuccess) e = e2;
    }
    return e;
}

}  // namespace sgm
