/* flow_oracle.c -- CPU ORACLE (test infrastructure only) for the optical-flow core of
 * arXiv 1801.04720 Sec. 3.2 ("Optical Flow from Flow Fields+"), i.e. SURVEY.md
 * 8(f) rank 2, following SPEC module flow-fields step by step.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py may use this file.  It shares no
 * code with the CUDA path.  Plain loops, no blocking, in the order of the SPEC:
 *   pyramid (2x2 box)            -- "initialized on a lower resolution"
 *   WHT descriptors + kNN init   -- "matching Walsh-Hadamard features using k-dimensional
 *                                   search trees".  The k nearest
 *                                   neighbours are found by exhaustive search, which
 *                                   returns exactly what a kd-tree query returns.
 *   patch data term              -- "fitness of a match is determined by a patch-based
 *                                   data term" (SAD per F-2/F-3)
 *   propagation + random search  -- "propagated into their local neighborhood. After each
 *                                   iteration, a random search" (F-4)
 *   lift                         -- "lifted to the next higher resolution"
 *   consistency filter           -- "two additional inverse flow fields. If any match is
 *                                   inconsistent with any of the inverse fields, it gets
 *                                   filtered" (F-5)
 * Readings FF1-FF10: flow vectors are integers in 1/Q px (Q = 8);
 * the data term is computed exactly in integers (bilinear weights in 1/Q^2 steps), so
 * every accept/reject decision is exact and order-independent within one candidate.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define FQ 8                       /* sub-pixel steps per pixel (FF1) */
#define FQ2 (FQ * FQ)

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* FF2: level l+1 has ((W+1)/2, (H+1)/2) pixels; I'(x,y) = round-half-up mean of the 2x2
 * block at (2x, 2y) with coordinates clamped to the image. */
int orc_ff_downsample(const uint8_t *src, int W, int H, uint8_t *dst)
{
    if (W < 1 || H < 1) return 1;
    const int W2 = (W + 1) / 2, H2 = (H + 1) / 2;
    for (int y = 0; y < H2; ++y)
        for (int x = 0; x < W2; ++x) {
            int s = 0;
            for (int j = 0; j < 2; ++j)
                for (int i = 0; i < 2; ++i)
                    s += src[clampi(2 * y + j, 0, H - 1) * W + clampi(2 * x + i, 0, W - 1)];
            dst[y * W2 + x] = (uint8_t)((s + 2) >> 2);
        }
    return 0;
}

/* Sequency-ordered Walsh functions of length N (N = 4, 8, 16): row k of the natural
 * (Sylvester) Hadamard matrix H[i][j] = (-1)^popcount(i & j) that has exactly k sign
 * changes. */
static void walsh_sequency(int N, int *h /* [N][N] */)
{
    for (int r = 0; r < N; ++r) {
        int row[16], changes = 0;
        for (int j = 0; j < N; ++j) row[j] = (__builtin_popcount(r & j) & 1) ? -1 : 1;
        for (int j = 1; j < N; ++j) changes += row[j] != row[j - 1];
        for (int j = 0; j < N; ++j) h[changes * N + j] = row[j];
    }
}

/* FF3: descriptor of pixel (x, y) = the 16 lowest-sequency 2-D Walsh-Hadamard
 * coefficients c(u, v) = sum_j sum_i P(i, j) w_u(i) w_v(j), u, v in 0..3, of the win x
 * win patch P with top-left corner (x - win/2 + 1, y - win/2 + 1), edge-clamped
 * ("centered ... edge-clamped"), stored exactly (int32) at index v * 4 + u. */
int orc_ff_wht(const uint8_t *img, int W, int H, int win, int32_t *desc /* [H][W][16] */)
{
    if (win != 4 && win != 8 && win != 16) return 1;
    int h[16 * 16];
    walsh_sequency(win, h);
    const int o = win / 2 - 1;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int v = 0; v < 4; ++v)
                for (int u = 0; u < 4; ++u) {
                    int c = 0;
                    for (int j = 0; j < win; ++j)
                        for (int i = 0; i < win; ++i) {
                            const int p = img[clampi(y - o + j, 0, H - 1) * W + clampi(x - o + i, 0, W - 1)];
                            c += p * h[u * win + i] * h[v * win + j];
                        }
                    desc[((int64_t)y * W + x) * 16 + v * 4 + u] = c;
                }
    return 0;
}

/* FF4: patch data term (F-2, F-3).  For every offset (dx, dy) in [-r, r]^2:
 * a = A at (x+dx, y+dy) (edge-clamped); the target position in B, in 1/Q px, is
 * ((x+dx) Q + fu, (y+dy) Q + fv); inside [0, (W-1) Q] x [0, (H-1) Q] its bilinear value
 * is b = sum_k w_k B(tap_k) with integer weights (Q - fx)(Q - fy), fx (Q - fy),
 * (Q - fx) fy, fx fy (fx, fy = position mod Q), taps clamped to the image (a clamped tap
 * has weight 0); the term adds |Q^2 a - b|.  Outside, it adds penalty * Q^2.  The sum is
 * the patch SAD in units of 1/Q^2 gray levels. */
int32_t orc_ff_patch_cost(const uint8_t *A, const uint8_t *B, int W, int H, int x, int y,
                          int fu, int fv, int r, int penalty)
{
    int32_t s = 0;
    for (int dy = -r; dy <= r; ++dy)
        for (int dx = -r; dx <= r; ++dx) {
            const int a = A[clampi(y + dy, 0, H - 1) * W + clampi(x + dx, 0, W - 1)];
            const int px = (x + dx) * FQ + fu, py = (y + dy) * FQ + fv;
            if (px < 0 || py < 0 || px > (W - 1) * FQ || py > (H - 1) * FQ) {
                s += penalty * FQ2;
                continue;
            }
            const int ix = px / FQ, fx = px % FQ, iy = py / FQ, fy = py % FQ;
            const int ix1 = ix + 1 < W ? ix + 1 : W - 1, iy1 = iy + 1 < H ? iy + 1 : H - 1;
            const int b = (FQ - fx) * (FQ - fy) * B[iy * W + ix] + fx * (FQ - fy) * B[iy * W + ix1] +
                          (FQ - fx) * fy * B[iy1 * W + ix] + fx * fy * B[iy1 * W + ix1];
            const int d = FQ2 * a - b;
            s += d < 0 ? -d : d;
        }
    return s;
}

/* FF5: k nearest neighbours of every A descriptor among all B descriptors by squared
 * Euclidean distance, ties to the smaller B index; candidate flow = (xb - xa, yb - ya)
 * px; the field keeps, in kNN order, the first candidate of minimal data term. */
int orc_ff_knn_init(const uint8_t *A, const uint8_t *B, int W, int H, int win, int knn,
                    int r, int penalty, int32_t *flow /* [H][W][2] */, int32_t *cost,
                    int32_t *nn /* [H][W][knn] B indices, may be NULL */)
{
    if (knn < 1 || knn > 16) return 1;
    const int64_t n = (int64_t)W * H;
    int32_t *da = malloc(sizeof(int32_t) * 16 * n), *db = malloc(sizeof(int32_t) * 16 * n);
    if (!da || !db) { free(da); free(db); return 2; }
    int rc = orc_ff_wht(A, W, H, win, da) | orc_ff_wht(B, W, H, win, db);
    for (int64_t p = 0; p < n && rc == 0; ++p) {
        int64_t bd[16];
        int32_t bi[16];
        int cnt = 0;
        for (int64_t q = 0; q < n; ++q) {
            int64_t d = 0;
            for (int k = 0; k < 16; ++k) {
                const int64_t e = (int64_t)da[p * 16 + k] - db[q * 16 + k];
                d += e * e;
            }
            /* insert (d, q) into the sorted list of the knn best (strictly better only:
             * an equal distance keeps the earlier, smaller index) */
            if (cnt < knn || d < bd[cnt - 1]) {
                int pos = cnt < knn ? cnt++ : knn - 1;
                while (pos > 0 && bd[pos - 1] > d) {
                    bd[pos] = bd[pos - 1];
                    bi[pos] = bi[pos - 1];
                    --pos;
                }
                bd[pos] = d;
                bi[pos] = (int32_t)q;
            }
        }
        const int xa = (int)(p % W), ya = (int)(p / W);
        int32_t best = INT32_MAX, bu = 0, bv = 0;
        for (int k = 0; k < cnt; ++k) {
            const int xb = bi[k] % W, yb = bi[k] / W;
            const int fu = (xb - xa) * FQ, fv = (yb - ya) * FQ;
            const int32_t c = orc_ff_patch_cost(A, B, W, H, xa, ya, fu, fv, r, penalty);
            if (c < best) { best = c; bu = fu; bv = fv; }
            if (nn) nn[p * knn + k] = bi[k];
        }
        flow[2 * p] = bu;
        flow[2 * p + 1] = bv;
        cost[p] = best;
    }
    free(da);
    free(db);
    return rc;
}

/* FF6: counter-based random stream (F-4): splitmix64 of a key built from the seed, the
 * level, the sweep and the pixel. */
uint64_t orc_ff_rng(uint64_t seed, int level, int sweep, int x, int y)
{
    uint64_t z = seed ^ ((uint64_t)(level & 0xff) << 56) ^ ((uint64_t)(sweep & 0xff) << 48) ^
                 ((uint64_t)(y & 0xffffff) << 24) ^ (uint64_t)(x & 0xffffff);
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* FF7: one propagation sweep: sweep s even scans rows top->bottom, each row
 * left->right, offering the left then the upper neighbour's current vector; s odd scans
 * bottom->top, right->left, offering the right then the lower neighbour's.  A candidate
 * replaces the incumbent iff its data term is strictly lower.  Then the random search
 * (S:231): every pixel tests its vector plus an offset (ou, ov), each uniform in
 * [-R Q, R Q] (R = max(R0 >> s, 1) px): z = rng(seed, level, s, x, y),
 * ou = (z mod 2^32) mod (2RQ+1) - RQ, ov = (z >> 32) mod (2RQ+1) - RQ; accepted iff
 * strictly better.  The random search reads only the pixel's own vector. */
int orc_ff_sweep(const uint8_t *A, const uint8_t *B, int W, int H, int r, int penalty,
                 int sweep, int level, int R0, uint64_t seed, int32_t *flow, int32_t *cost)
{
    const int fwd = (sweep % 2) == 0;
    for (int jj = 0; jj < H; ++jj) {
        const int y = fwd ? jj : H - 1 - jj;
        for (int ii = 0; ii < W; ++ii) {
            const int x = fwd ? ii : W - 1 - ii;
            const int64_t p = (int64_t)y * W + x;
            const int nx[2] = {fwd ? x - 1 : x + 1, x};
            const int ny[2] = {y, fwd ? y - 1 : y + 1};
            for (int k = 0; k < 2; ++k) {
                if (nx[k] < 0 || nx[k] >= W || ny[k] < 0 || ny[k] >= H) continue;
                const int64_t q = (int64_t)ny[k] * W + nx[k];
                const int fu = flow[2 * q], fv = flow[2 * q + 1];
                const int32_t c = orc_ff_patch_cost(A, B, W, H, x, y, fu, fv, r, penalty);
                if (c < cost[p]) {
                    cost[p] = c;
                    flow[2 * p] = fu;
                    flow[2 * p + 1] = fv;
                }
            }
        }
    }
    int R = R0 >> sweep;
    if (R < 1) R = 1;
    const uint32_t span = (uint32_t)(2 * R * FQ + 1);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const int64_t p = (int64_t)y * W + x;
            const uint64_t z = orc_ff_rng(seed, level, sweep, x, y);
            const int ou = (int)((uint32_t)z % span) - R * FQ;
            const int ov = (int)((uint32_t)(z >> 32) % span) - R * FQ;
            const int fu = flow[2 * p] + ou, fv = flow[2 * p + 1] + ov;
            const int32_t c = orc_ff_patch_cost(A, B, W, H, x, y, fu, fv, r, penalty);
            if (c < cost[p]) {
                cost[p] = c;
                flow[2 * p] = fu;
                flow[2 * p + 1] = fv;
            }
        }
    return 0;
}

/* FF8: lift: fine pixel (x, y) takes 2 x the vector of coarse pixel
 * (min(x/2, Wc-1), min(y/2, Hc-1)); its data term is recomputed at the fine level. */
int orc_ff_lift(const uint8_t *A, const uint8_t *B, int W, int H, int Wc, int Hc,
                const int32_t *coarse, int r, int penalty, int32_t *flow, int32_t *cost)
{
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const int64_t p = (int64_t)y * W + x;
            const int64_t c = (int64_t)clampi(y / 2, 0, Hc - 1) * Wc + clampi(x / 2, 0, Wc - 1);
            flow[2 * p] = 2 * coarse[2 * c];
            flow[2 * p + 1] = 2 * coarse[2 * c + 1];
            cost[p] = orc_ff_patch_cost(A, B, W, H, x, y, flow[2 * p], flow[2 * p + 1], r, penalty);
        }
    return 0;
}

/* One match field A -> B: pyramid of `levels`, kNN init at the coarsest
 * level, `sweeps` propagation + random-search sweeps per level, lift between levels. */
int orc_ff_field(const uint8_t *A, const uint8_t *B, int W, int H, int levels, int r,
                 int sweeps, int R0, int win, int knn, int penalty, uint64_t seed,
                 int32_t *flow, int32_t *cost)
{
    if (levels < 1 || levels > 8 || W < 1 || H < 1) return 1;
    const uint8_t *pa[8], *pb[8];
    int pw[8], ph[8];
    uint8_t *own[16] = {0};
    pa[0] = A; pb[0] = B; pw[0] = W; ph[0] = H;
    for (int l = 1; l < levels; ++l) {
        pw[l] = (pw[l - 1] + 1) / 2;
        ph[l] = (ph[l - 1] + 1) / 2;
        own[2 * l] = malloc((size_t)pw[l] * ph[l]);
        own[2 * l + 1] = malloc((size_t)pw[l] * ph[l]);
        orc_ff_downsample(pa[l - 1], pw[l - 1], ph[l - 1], own[2 * l]);
        orc_ff_downsample(pb[l - 1], pw[l - 1], ph[l - 1], own[2 * l + 1]);
        pa[l] = own[2 * l];
        pb[l] = own[2 * l + 1];
    }
    int32_t *f = NULL, *c = NULL, *fc = NULL;
    int rc = 0;
    for (int l = levels - 1; l >= 0 && rc == 0; --l) {
        const int64_t n = (int64_t)pw[l] * ph[l];
        int32_t *nf = malloc(sizeof(int32_t) * 2 * n), *nc = malloc(sizeof(int32_t) * n);
        if (l == levels - 1)
            rc = orc_ff_knn_init(pa[l], pb[l], pw[l], ph[l], win, knn, r, penalty, nf, nc, NULL);
        else
            rc = orc_ff_lift(pa[l], pb[l], pw[l], ph[l], pw[l + 1], ph[l + 1], fc, r, penalty, nf, nc);
        for (int s = 0; s < sweeps && rc == 0; ++s)
            rc = orc_ff_sweep(pa[l], pb[l], pw[l], ph[l], r, penalty, s, l, R0, seed, nf, nc);
        free(fc);
        free(c);
        fc = nf;
        c = nc;
        f = nf;
    }
    if (rc == 0) {
        memcpy(flow, f, sizeof(int32_t) * 2 * (size_t)W * H);
        memcpy(cost, c, sizeof(int32_t) * (size_t)W * H);
    }
    free(fc);
    free(c);
    for (int k = 0; k < 16; ++k) free(own[k]);
    return rc;
}

/* FF9: consistency: x survives iff its target t = x Q + F(x) lies in
 * [0, (W-1) Q] x [0, (H-1) Q] and, for BOTH inverse fields G, |F(x) + G(t)| <= thr_q / Q
 * px, with G(t) bilinear (integer weights in 1/Q^2) -- compared exactly in units of
 * 1/Q^3 px: (Q^2 F + sum w G)^2 summed over (u, v) <= (Q^2 thr_q)^2. */
int orc_ff_consistency(const int32_t *F, const int32_t *G1, const int32_t *G2, int W, int H,
                       int thr_q, uint8_t *valid)
{
    const int64_t lim = (int64_t)thr_q * FQ2;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const int64_t p = (int64_t)y * W + x;
            const int tx = x * FQ + F[2 * p], ty = y * FQ + F[2 * p + 1];
            int ok = tx >= 0 && ty >= 0 && tx <= (W - 1) * FQ && ty <= (H - 1) * FQ;
            for (int g = 0; g < 2 && ok; ++g) {
                const int32_t *G = g == 0 ? G1 : G2;
                const int ix = tx / FQ, fx = tx % FQ, iy = ty / FQ, fy = ty % FQ;
                const int ix1 = ix + 1 < W ? ix + 1 : W - 1, iy1 = iy + 1 < H ? iy + 1 : H - 1;
                const int64_t w00 = (FQ - fx) * (FQ - fy), w10 = fx * (FQ - fy);
                const int64_t w01 = (FQ - fx) * fy, w11 = fx * fy;
                const int64_t t00 = (int64_t)iy * W + ix, t10 = (int64_t)iy * W + ix1;
                const int64_t t01 = (int64_t)iy1 * W + ix, t11 = (int64_t)iy1 * W + ix1;
                int64_t e[2];
                for (int k = 0; k < 2; ++k)
                    e[k] = (int64_t)FQ2 * F[2 * p + k] + w00 * G[2 * t00 + k] + w10 * G[2 * t10 + k] +
                           w01 * G[2 * t01 + k] + w11 * G[2 * t11 + k];
                ok = e[0] * e[0] + e[1] * e[1] <= lim * lim;
            }
            valid[p] = (uint8_t)ok;
        }
    return 0;
}

/* The optical-flow step (F-5): forward field A -> B (seed, r), two inverse
 * fields B -> A (seed + 1, r) and (seed + 2, r + 2), consistency filter.  flow_out in
 * 1/Q px; valid_out the filter mask. */
int orc_ff_flow(const uint8_t *A, const uint8_t *B, int W, int H, int levels, int r, int sweeps,
                int R0, int win, int knn, int penalty, uint64_t seed, int thr_q,
                int32_t *flow_out, uint8_t *valid_out)
{
    const size_t n = (size_t)W * H;
    int32_t *g1 = malloc(sizeof(int32_t) * 2 * n), *g2 = malloc(sizeof(int32_t) * 2 * n);
    int32_t *c = malloc(sizeof(int32_t) * n);
    int rc = (!g1 || !g2 || !c) ? 2 : 0;
    if (!rc) rc = orc_ff_field(A, B, W, H, levels, r, sweeps, R0, win, knn, penalty, seed, flow_out, c);
    if (!rc) rc = orc_ff_field(B, A, W, H, levels, r, sweeps, R0, win, knn, penalty, seed + 1, g1, c);
    if (!rc) rc = orc_ff_field(B, A, W, H, levels, r + 2, sweeps, R0, win, knn, penalty, seed + 2, g2, c);
    if (!rc) rc = orc_ff_consistency(flow_out, g1, g2, W, H, thr_q, valid_out);
    free(g1);
    free(g2);
    free(c);
    return rc;
}

/* ------------------------------------------------------------------ */
/* Densification (SPEC densify S:253-262, F-6:   */
/* "K-nearest seeds under edge-aware line-integral distance with        */
/* inverse-distance weights"; the gap filling the paper   */
/* delegates to EpicFlow, and the "Ours (All)" densification,     */
/* P:147).  Readings DN1-DN4:                         */
/*   d_e(p, s) = |p - s| + lambda * sum_k g(q_k)                         */
/* with q_k = the interior points of the segment p -> s (n = max(|dx|,  */
/* |dy|) steps, q_k = p + round-half-up(k (s - p) / n), k = 1..n-1) and */
/* g(q) = |G(x+1,y) - G(x-1,y)| + |G(x,y+1) - G(x,y-1)| (clamped), G the */
/* guide image.  A pixel with valid != 0 keeps its C values exactly; a  */
/* gap pixel p takes the 1/d_e-weighted mean of the K valid seeds of    */
/* smallest d_e (DN1: ties to the smaller linear index), d_e evaluated  */
/* as sqrt((double)|p-s|^2) + (double)lambda * (double)sum (one rounding */
/* each, so the ranking is reproducible bit for bit).  window <= 0:     */
/* every seed of the image is a candidate (the SPEC's definition);      */
/* window > 0: only seeds within Chebyshev distance                     */
/* max(window, rho_K(p)) are, rho_K(p) = the smallest Chebyshev radius  */
/* holding >= K seeds (the whole image if it has fewer).  An image with */
/* no valid pixel yields zeros (returns 3).                             */
/* ------------------------------------------------------------------ */
static int grad_l1(const uint8_t *G, int W, int H, int x, int y)
{
    const int gx = (int)G[y * W + clampi(x + 1, 0, W - 1)] - (int)G[y * W + clampi(x - 1, 0, W - 1)];
    const int gy = (int)G[clampi(y + 1, 0, H - 1) * W + x] - (int)G[clampi(y - 1, 0, H - 1) * W + x];
    return (gx < 0 ? -gx : gx) + (gy < 0 ? -gy : gy);
}

/* floor((2 a + b) / (2 b)) for b > 0: round-half-up of a / b */
static int div_round(int a, int b)
{
    const int num = 2 * a + b, den = 2 * b;
    return num >= 0 ? num / den : -((-num + den - 1) / den);
}

double orc_edge_distance(const uint8_t *G, int W, int H, int px, int py, int sx, int sy, double lambda)
{
    const int dx = sx - px, dy = sy - py;
    const int n = (dx < 0 ? -dx : dx) > (dy < 0 ? -dy : dy) ? (dx < 0 ? -dx : dx) : (dy < 0 ? -dy : dy);
    long long acc = 0;
    for (int k = 1; k < n; ++k)
        acc += grad_l1(G, W, H, px + div_round(k * dx, n), py + div_round(k * dy, n));
    return sqrt((double)dx * dx + (double)dy * dy) + lambda * (double)acc;
}

static int cheb(int ax, int ay, int bx, int by)
{
    const int dx = ax > bx ? ax - bx : bx - ax, dy = ay > by ? ay - by : by - ay;
    return dx > dy ? dx : dy;
}

/* Densified value of one gap pixel p = (px, py) (the body of orc_densify). */
static void densify_pixel(const float *field, const uint8_t *valid, const uint8_t *guide, int W, int H, int C,
                          int K, float lambda, int window, int px, int py, double *o)
{
    const int64_t n = (int64_t)W * H;
    /* candidate radius: the whole image, or max(window, rho_K(p)) */
    int R = W > H ? W : H;
    if (window > 0) {
        int *hist = calloc((size_t)R + 1, sizeof(int));
        for (int64_t q = 0; q < n; ++q)
            if (valid[q]) hist[cheb((int)(q % W), (int)(q / W), px, py)]++;
        int rho = R, seen = 0;
        for (int r = 0; r <= R; ++r) {
            seen += hist[r];
            if (seen >= K) { rho = r; break; }
        }
        free(hist);
        R = window > rho ? window : rho;
    }
    double bd[64];
    int64_t bi[64];
    int cnt = 0;
    for (int64_t q = 0; q < n; ++q) {              /* every candidate, ranked by (d_e, index) */
        if (!valid[q]) continue;
        const int sx = (int)(q % W), sy = (int)(q / W);
        if (cheb(sx, sy, px, py) > R) continue;
        const double d = orc_edge_distance(guide, W, H, px, py, sx, sy, (double)lambda);
        if (cnt < K || d < bd[cnt - 1]) {          /* q ascends: equal d keeps the smaller index */
            int pos = cnt < K ? cnt++ : K - 1;
            while (pos > 0 && bd[pos - 1] > d) {
                bd[pos] = bd[pos - 1];
                bi[pos] = bi[pos - 1];
                --pos;
            }
            bd[pos] = d;
            bi[pos] = q;
        }
    }
    double wsum = 0.0, acc[4] = {0, 0, 0, 0};
    for (int k = 0; k < cnt; ++k) {
        const double w = 1.0 / bd[k];
        wsum += w;
        for (int c = 0; c < C; ++c) acc[c] += w * field[bi[k] * C + c];
    }
    for (int c = 0; c < C; ++c) o[c] = cnt ? acc[c] / wsum : 0.0;
}

int orc_densify(const float *field, const uint8_t *valid, const uint8_t *guide, int W, int H, int C,
                int K, float lambda, int window, double *out)
{
    if (K < 1 || K > 64 || C < 1 || C > 4) return 1;
    const int64_t n = (int64_t)W * H;
    int64_t nseed = 0;
    for (int64_t p = 0; p < n; ++p) nseed += valid[p] != 0;
    for (int64_t p = 0; p < n; ++p) {
        if (valid[p]) {
            for (int c = 0; c < C; ++c) out[p * C + c] = field[p * C + c];
            continue;
        }
        densify_pixel(field, valid, guide, W, H, C, K, lambda, window, (int)(p % W), (int)(p / W), out + p * C);
    }
    return nseed == 0 ? 3 : 0;
}

/* The same at a list of pixels xy[npts][2] (for parity samples of full-size images). */
int orc_densify_points(const float *field, const uint8_t *valid, const uint8_t *guide, int W, int H, int C,
                       int K, float lambda, int window, int npts, const int *xy, double *out)
{
    if (K < 1 || K > 64 || C < 1 || C > 4) return 1;
    for (int i = 0; i < npts; ++i) {
        const int x = xy[2 * i], y = xy[2 * i + 1];
        const int64_t p = (int64_t)y * W + x;
        if (valid[p]) {
            for (int c = 0; c < C; ++c) out[i * C + c] = field[p * C + c];
        } else {
            densify_pixel(field, valid, guide, W, H, C, K, lambda, window, x, y, out + i * C);
        }
    }
    return 0;
}
