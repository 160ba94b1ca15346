/*
 * sgm_oracle.c -- plain, slow, obviously-correct CPU ORACLE for the hot path
 * of Schuster et al., "Combining Stereo Disparity and Optical Flow for Basic
 * Scene Flow" (arXiv 1801.04720).
 *
 * THIS IS TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and
 * bench.py (its cpu_baseline leg and `--impl reference`) may load or call it.
 * It shares no code, header, table or constant with the CUDA product path
 * (paper_1801_04720_b200/), and the product path never imports it.
 *
 * Citations: P:n = reference PAPER.md line n, S:n = reference SPEC.md line n,
 * G# = the reading numbered # in DESIGN.md section "Readings" (taken from
 * SURVEY.md 8(c)).  Every function follows the algorithm in the paper's (or
 * the spec's) order, one pixel / one disparity at a time, no blocking, no
 * fusion, no reordering.  Floating point is double (fp64) except where a
 * float decides an integer (G16/G18: the x' = x + u membership test), where
 * the kernel's float32 is used on both sides.
 *
 * Compile: gcc -O2 -ffp-contract=off -fPIC -shared (no SIMD intrinsics).
 *
 * Parity status per function (details in DESIGN.md "Oracle pins"):
 *   orc_census, orc_cost, orc_path, orc_aggregate, orc_wta, orc_lr_check,
 *   orc_disparity, orc_combine, orc_reproject : pinned (tests/test_oracle_*.py)
 *   end-to-end against the paper's KITTI numbers : parity unpinned (no data).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------ */
/* helpers                                                              */
/* ------------------------------------------------------------------ */

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Hamming weight: the compiler's popcount primitive (a library step; pinned
 * against an independent bit count in tests/test_oracle_pins.py). */
static int bitcount64(uint64_t v) { return __builtin_popcountll(v); }

/* ------------------------------------------------------------------ */
/* O1: census transform                                                 */
/* S:110-118 (bit = 1 iff neighbour < centre, window^2-1 bits, edge-    */
/* clamped borders); G2 (window is cw wide x ch tall), G3 (strict <,    */
/* centre skipped, clamp), G4 (row-major scan dy outer / dx inner,      */
/* k-th neighbour -> bit k, LSB first).                                 */
/* ------------------------------------------------------------------ */
int orc_census(const uint8_t *img, int W, int H, int64_t pitch, int cw, int ch,
               uint64_t *out)
{
    if (W < 1 || H < 1 || cw < 1 || ch < 1 || (cw % 2) == 0 || (ch % 2) == 0)
        return 1;                                   /* S:115 "even window" error */
    if (cw * ch - 1 > 64) return 1;
    const int rx = cw / 2, ry = ch / 2;
    for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
            const int centre = img[(int64_t)y * pitch + x];
            uint64_t bits = 0;
            int k = 0;
            for (int dy = -ry; dy <= ry; ++dy) {
                for (int dx = -rx; dx <= rx; ++dx) {
                    if (dx == 0 && dy == 0) continue;
                    const int yy = clampi(y + dy, 0, H - 1);
                    const int xx = clampi(x + dx, 0, W - 1);
                    const int n = img[(int64_t)yy * pitch + xx];
                    if (n < centre) bits |= ((uint64_t)1) << k;
                    ++k;
                }
            }
            out[(int64_t)y * W + x] = bits;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* O2: matching cost volume                                             */
/* cost(x,y,d) = Hamming(census_ref(x,y), census_match(x-d,y))*/
/* out of image -> descriptor length (G5: C_max = w*h-1).        */
/* s = -1: left image is the reference (match at x-d);                  */
/* s = +1: right image is the reference (match at x+d) -- G12.          */
/* Layout: out[(y*W + x)*D + d], uint8.                                 */
/* ------------------------------------------------------------------ */
int orc_cost(const uint64_t *cen_ref, const uint64_t *cen_match, int W, int H,
             int D, int s, int cmax, uint8_t *out)
{
    if (W < 1 || H < 1 || D < 1 || (s != -1 && s != 1) || cmax < 0 || cmax > 255) return 1;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int d = 0; d < D; ++d) {
                const int xm = x + s * d;
                int c;
                if (xm >= 0 && xm < W)
                    c = bitcount64(cen_ref[(int64_t)y * W + x] ^ cen_match[(int64_t)y * W + xm]);
                else
                    c = cmax;
                out[((int64_t)y * W + x) * D + d] = (uint8_t)c;
            }
    return 0;
}

/* ------------------------------------------------------------------ */
/* O3: one aggregation path r = (rx, ry)                                */
/* P:73 ("eight different paths radiating from each target pixel");    */
/* recursion S:129:                                                     */
/*  L_r(p,d) = C(p,d) + min( L_r(p-r,d), L_r(p-r,d-1)+P1, L_r(p-r,d+1)+P1,*/
/*                           min_k L_r(p-r,k)+P2 ) - min_k L_r(p-r,k)   */
/* path start (p-r outside the image): L_r(p,d) = C(p,d).       */
/* d-1 / d+1 terms outside [0, D-1] are omitted (G7).                   */
/* Pixels are visited so that p-r is always visited before p.          */
/* Layout: cost uint8 [y][x][d], L int32 [y][x][d].                     */
/* ------------------------------------------------------------------ */
int orc_path(const uint8_t *cost, int W, int H, int D, int P1, int P2,
             int rx, int ry, int32_t *L)
{
    if (W < 1 || H < 1 || D < 1) return 1;
    if (rx < -1 || rx > 1 || ry < -1 || ry > 1 || (rx == 0 && ry == 0)) return 1;
    const int y_first = (ry >= 0) ? 0 : H - 1, y_step = (ry >= 0) ? 1 : -1;
    const int x_first = (rx >= 0) ? 0 : W - 1, x_step = (rx >= 0) ? 1 : -1;
    for (int iy = 0, y = y_first; iy < H; ++iy, y += y_step) {
        for (int ix = 0, x = x_first; ix < W; ++ix, x += x_step) {
            const int64_t p = (int64_t)y * W + x;
            const int px = x - rx, py = y - ry;               /* p - r */
            if (px < 0 || px >= W || py < 0 || py >= H) {
                for (int d = 0; d < D; ++d) L[p * D + d] = cost[p * D + d];
                continue;
            }
            const int64_t q = (int64_t)py * W + px;
            int m = L[q * D + 0];
            for (int k = 1; k < D; ++k)
                if (L[q * D + k] < m) m = L[q * D + k];
            for (int d = 0; d < D; ++d) {
                int best = L[q * D + d];
                if (d >= 1 && L[q * D + d - 1] + P1 < best) best = L[q * D + d - 1] + P1;
                if (d <= D - 2 && L[q * D + d + 1] + P1 < best) best = L[q * D + d + 1] + P1;
                if (m + P2 < best) best = m + P2;
                L[p * D + d] = cost[p * D + d] + best - m;
            }
        }
    }
    return 0;
}

/* The 8 directions of P:73 / S:130 (horizontal +-, vertical +-, 4 diagonals). */
static const int DIRS[8][2] = {
    { 1, 0}, {-1, 0}, { 0, 1}, { 0, -1}, { 1, 1}, {-1, -1}, {-1, 1}, { 1, -1}
};

/* S = sum over the 8 paths of L_r.  S as uint32 [y][x][d]. */
int orc_aggregate(const uint8_t *cost, int W, int H, int D, int P1, int P2, uint32_t *S)
{
    if (W < 1 || H < 1 || D < 1) return 1;
    const int64_t n = (int64_t)W * H * D;
    int32_t *L = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!L) return 2;
    for (int64_t i = 0; i < n; ++i) S[i] = 0;
    for (int r = 0; r < 8; ++r) {
        if (orc_path(cost, W, H, D, P1, P2, DIRS[r][0], DIRS[r][1], L) != 0) { free(L); return 1; }
        for (int64_t i = 0; i < n; ++i) S[i] += (uint32_t)L[i];
    }
    free(L);
    return 0;
}

/* ------------------------------------------------------------------ */
/* O4: winner-take-all + parabola sub-pixel                             */
/* d* = argmin_d S, smallest index on ties (G10);     */
/* if 0 < d* < D-1: offset = (S(d*-1) - S(d*+1)) /                      */
/*                           (2 (S(d*-1) + S(d*+1) - 2 S(d*)))          */
/* clamped to [-0.5, 0.5]; denominator 0 -> offset 0 (G11);      */
/* boundary d* gets no offset.  fp64.                                   */
/* ------------------------------------------------------------------ */
int orc_wta(const uint32_t *S, int W, int H, int D, int16_t *d_int, double *d_sub)
{
    if (W < 1 || H < 1 || D < 1) return 1;
    for (int64_t p = 0; p < (int64_t)W * H; ++p) {
        const uint32_t *s = S + p * D;
        int best = 0;
        for (int d = 1; d < D; ++d)
            if (s[d] < s[best]) best = d;                 /* strict: smallest index wins */
        double sub = (double)best;
        if (best > 0 && best < D - 1) {
            const double a = (double)s[best - 1], b = (double)s[best], c = (double)s[best + 1];
            const double den = 2.0 * (a + c - 2.0 * b);
            double off = 0.0;
            if (den != 0.0) off = (a - c) / den;
            if (off < -0.5) off = -0.5;
            if (off > 0.5) off = 0.5;
            sub = (double)best + off;
        }
        d_int[p] = (int16_t)best;
        d_sub[p] = sub;
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* O5: left-right consistency check                                     */
/* P:74 ("left-right consistency check ... remove wrongly estimated     */
/* values ... non-dense"); integer reading G13:              */
/*   valid(x,y) iff x - d*_L >= 0 and |d*_L(x,y) - d*_R(x - d*_L, y)| <= T */
/* invalid -> invalid_disp (G14: -1).                                   */
/* ------------------------------------------------------------------ */
int orc_lr_check(const int16_t *dl_int, const double *dl_sub, const int16_t *dr_int,
                 int W, int H, int T, int invalid_disp,
                 int16_t *out_int, double *out_sub, uint8_t *valid)
{
    if (W < 1 || H < 1 || T < 0) return 1;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const int64_t p = (int64_t)y * W + x;
            const int dl = dl_int[p];
            const int xr = x - dl;
            int ok = 0;
            if (xr >= 0 && xr < W) {
                const int dr = dr_int[(int64_t)y * W + xr];
                const int diff = dl > dr ? dl - dr : dr - dl;
                ok = diff <= T;
            }
            valid[p] = (uint8_t)ok;
            out_int[p] = ok ? (int16_t)dl : (int16_t)invalid_disp;
            out_sub[p] = ok ? dl_sub[p] : (double)invalid_disp;
        }
    return 0;
}

/* ------------------------------------------------------------------ */
/* One SGM view: census of both images is given; cost -> aggregate ->   */
/* WTA.  s = -1 left-reference, s = +1 right-reference (G12).           */
/* Optional intermediates (may be NULL): cost_out [y][x][D] uint8,      */
/* S_out [y][x][D] uint32.                                              */
/* ------------------------------------------------------------------ */
int orc_sgm_view(const uint64_t *cen_ref, const uint64_t *cen_match, int W, int H,
                 int D, int s, int cmax, int P1, int P2,
                 int16_t *d_int, double *d_sub, uint8_t *cost_out, uint32_t *S_out)
{
    const int64_t n = (int64_t)W * H * D;
    uint8_t *C = cost_out ? cost_out : (uint8_t *)malloc((size_t)n);
    uint32_t *S = S_out ? S_out : (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    int rc = 2;
    if (C && S) {
        rc = orc_cost(cen_ref, cen_match, W, H, D, s, cmax, C);
        if (rc == 0) rc = orc_aggregate(C, W, H, D, P1, P2, S);
        if (rc == 0) rc = orc_wta(S, W, H, D, d_int, d_sub);
    }
    if (!cost_out) free(C);
    if (!S_out) free(S);
    return rc;
}

/* ------------------------------------------------------------------ */
/* Whole SGM for one rectified pair:         */
/* census(L), census(R), left view, right view, LR check.               */
/* Outputs: LR-checked left-view int / sub-pixel / mask; the raw        */
/* per-view WTA results may be requested (NULL to skip).               */
/* ------------------------------------------------------------------ */
int orc_disparity(const uint8_t *left, const uint8_t *right, int W, int H, int64_t pitch,
                  int D, int cw, int ch, int P1, int P2, int T, int invalid_disp,
                  int16_t *out_int, double *out_sub, uint8_t *valid,
                  int16_t *dl_int_raw, double *dl_sub_raw, int16_t *dr_int_raw, double *dr_sub_raw)
{
    const int64_t npx = (int64_t)W * H;
    const int cmax = cw * ch - 1;
    uint64_t *cl = (uint64_t *)malloc((size_t)npx * 8), *cr = (uint64_t *)malloc((size_t)npx * 8);
    int16_t *dli = (int16_t *)malloc((size_t)npx * 2), *dri = (int16_t *)malloc((size_t)npx * 2);
    double *dls = (double *)malloc((size_t)npx * 8), *drs = (double *)malloc((size_t)npx * 8);
    int rc = 2;
    if (cl && cr && dli && dri && dls && drs) {
        rc = orc_census(left, W, H, pitch, cw, ch, cl);
        if (rc == 0) rc = orc_census(right, W, H, pitch, cw, ch, cr);
        if (rc == 0) rc = orc_sgm_view(cl, cr, W, H, D, -1, cmax, P1, P2, dli, dls, NULL, NULL);
        if (rc == 0) rc = orc_sgm_view(cr, cl, W, H, D, +1, cmax, P1, P2, dri, drs, NULL, NULL);
        if (rc == 0) rc = orc_lr_check(dli, dls, dri, W, H, T, invalid_disp, out_int, out_sub, valid);
        if (rc == 0) {
            if (dl_int_raw) memcpy(dl_int_raw, dli, (size_t)npx * 2);
            if (dl_sub_raw) memcpy(dl_sub_raw, dls, (size_t)npx * 8);
            if (dr_int_raw) memcpy(dr_int_raw, dri, (size_t)npx * 2);
            if (dr_sub_raw) memcpy(dr_sub_raw, drs, (size_t)npx * 8);
        }
    }
    free(cl); free(cr); free(dli); free(dri); free(dls); free(drs);
    return rc;
}

/* ------------------------------------------------------------------ */
/* O6: combination, Eq. (4) with the bilinear warp of        */
/* Eq. (5).                                                 */
/*  x' = x + F(x); in Omega iff 0 <= x' <= W-1 and             */
/*  0 <= y' <= H-1 (G16; closed domain S:45), computed in float32 as    */
/*  the kernel does (a float decides an integer: task rule), NaN ->     */
/*  outside.  floor / fractional part {x} = x - floor(x).       */
/*  The "+1" tap index is clamped to the border (G17, SPEC D-1).        */
/*  Validity of D1(x+F(x)) under interpolation: rule 0 = every tap with  */
/*  nonzero weight valid (G18, default); rule 1 = all four taps valid   */
/*  (SPEC D-2).  Valid output: F valid (G23), D0(x) valid, x' in Omega, */
/*  D1 valid -> S = (u, v, D0(x), D1(x')); else S = 0, mask 0 (G14).    */
/*  Eq. (5) is evaluated in the paper's term order, in fp64.            */
/* Layout: d0/d1 double [y][x], flow float [y][x][2] (u, v), sf double  */
/* [y][x][4] = (u, v, d0, d1).  flow_valid may be NULL (all valid).     */
/* ------------------------------------------------------------------ */
int orc_combine(const double *d0, const uint8_t *v0, const double *d1, const uint8_t *v1,
                const float *flow, const uint8_t *flow_valid, int W, int H, int rule,
                double *sf, uint8_t *valid)
{
    if (W < 1 || H < 1 || (rule != 0 && rule != 1)) return 1;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const int64_t p = (int64_t)y * W + x;
            const float u = flow[2 * p + 0], v = flow[2 * p + 1];
            double *o = sf + 4 * p;
            o[0] = o[1] = o[2] = o[3] = 0.0;
            valid[p] = 0;
            if (flow_valid && !flow_valid[p]) continue;
            if (!v0[p]) continue;
            const float xp = (float)x + u;             /* float32, as decided on both sides */
            const float yp = (float)y + v;
            if (!(xp >= 0.0f && xp <= (float)(W - 1) && yp >= 0.0f && yp <= (float)(H - 1)))
                continue;                               /* Eq. (4): x + F(x) not in Omega */
            const int x0 = (int)floorf(xp), y0 = (int)floorf(yp);
            const float fx = xp - (float)x0, fy = yp - (float)y0;   /* {x'}, {y'} exact */
            const int x1 = x0 + 1 <= W - 1 ? x0 + 1 : W - 1;
            const int y1 = y0 + 1 <= H - 1 ? y0 + 1 : H - 1;
            const int64_t q00 = (int64_t)y0 * W + x0, q10 = (int64_t)y0 * W + x1;
            const int64_t q01 = (int64_t)y1 * W + x0, q11 = (int64_t)y1 * W + x1;
            int ok;
            if (rule == 1) {
                ok = v1[q00] && v1[q10] && v1[q01] && v1[q11];
            } else {
                ok = v1[q00];
                if (fx != 0.0f) ok = ok && v1[q10];
                if (fy != 0.0f) ok = ok && v1[q01];
                if (fx != 0.0f && fy != 0.0f) ok = ok && v1[q11];
            }
            if (!ok) continue;                          /* Eq. (4): D1(x+F(x)) not valid */
            const double ax = (double)fx, ay = (double)fy;
            const double warped = d1[q00] * (1.0 - ax) * (1.0 - ay)
                                + d1[q10] * ax * (1.0 - ay)
                                + d1[q01] * (1.0 - ax) * ay
                                + d1[q11] * ax * ay;
            o[0] = (double)u;
            o[1] = (double)v;
            o[2] = d0[p];
            o[3] = warped;
            valid[p] = 1;
        }
    return 0;
}

/* ------------------------------------------------------------------ */
/* O7: 3D interpretation ("fully describe the 3D motion and 3D     */
/* geometry given the camera intrinsics and extrinsics"; "the     */
/* difference of the disparity values yields the missing motion         */
/* component in direction of viewing").                     */
/*  Z = f B / d, X = (x - cx) Z / f, Y = (y - cy) Z / f (G20).          */
/*  P0 from (x, y, d0); P1 from (x + u, y + v, d1); dP = P1 - P0.        */
/*  Valid iff S valid and d0 > 0 and d1 > 0 (G21, S:362/S:371          */
/*  skip-and-mark); invalid -> zeros.  fp64.                            */
/* Layout: sf double [y][x][4]; p0, p1, dp double [y][x][3].            */
/* ------------------------------------------------------------------ */
int orc_reproject(const double *sf, const uint8_t *valid_sf, int W, int H,
                  double f, double B, double cx, double cy,
                  double *p0, double *p1, double *dp, uint8_t *valid3d)
{
    if (W < 1 || H < 1 || !(f > 0.0) || !(B > 0.0)) return 1;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const int64_t p = (int64_t)y * W + x;
            const double *s = sf + 4 * p;
            double *a = p0 + 3 * p, *b = p1 + 3 * p, *c = dp + 3 * p;
            a[0] = a[1] = a[2] = b[0] = b[1] = b[2] = c[0] = c[1] = c[2] = 0.0;
            valid3d[p] = 0;
            if (!valid_sf[p] || !(s[2] > 0.0) || !(s[3] > 0.0)) continue;
            const double Z0 = f * B / s[2];
            const double X0 = ((double)x - cx) * Z0 / f;
            const double Y0 = ((double)y - cy) * Z0 / f;
            const double xe = (double)x + s[0], ye = (double)y + s[1];
            const double Z1 = f * B / s[3];
            const double X1 = (xe - cx) * Z1 / f;
            const double Y1 = (ye - cy) * Z1 / f;
            a[0] = X0; a[1] = Y0; a[2] = Z0;
            b[0] = X1; b[1] = Y1; b[2] = Z1;
            c[0] = X1 - X0; c[1] = Y1 - Y0; c[2] = Z1 - Z0;
            valid3d[p] = 1;
        }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Evaluation (SPEC eval S:449-499; Table 1      */
/* semantics P:130-155, density P:159 / S:314-322).  KITTI outlier rule */
/* (SPEC E-1, an external convention the paper invokes at P:131):       */
/* outlier iff err > tau_abs (3 px) and err > tau_rel (5%) x the        */
/* ground-truth magnitude.                                      */
/* The decision is taken in float32 -- the kernel's precision, because  */
/* a float decides an integer count -- with each operation rounded     */
/* separately (no contraction).  Split 0 = all ground-truth pixels      */
/* ("Occ"), split 1 = non-occluded ones ("Noc").  Over ground-truth     */
/* pixels that the estimate covers ("Est"):                      */
/*   D1 err = |d0 - gt_d0|,  D2 err = |d1 - gt_d1| (gt_d1 = disparity   */
/*   at t+1 of the point seen at x), Fl err = |(u,v) - gt_flow|,         */
/*   SF = D1 or D2 or Fl outlier.                                       */
/* counts[s][0..5] = {n_gt, n_eval, n_d1, n_d2, n_fl, n_sf};            */
/* density = n_eval / n_gt.  gt_valid may be NULL (every pixel).        */
/* ------------------------------------------------------------------ */
static int kitti_outlier(float err, float mag, float tau_abs, float tau_rel)
{
    const float rel = tau_rel * mag;
    return err > tau_abs && err > rel;
}

int orc_evaluate(const float *sf, const uint8_t *valid_sf, const float *gt_d0,
                 const float *gt_d1, const float *gt_flow, const uint8_t *gt_valid,
                 const uint8_t *gt_noc, int W, int H, float tau_abs, float tau_rel,
                 long long *counts /* [2][6] */)
{
    if (W < 1 || H < 1) return 1;
    for (int k = 0; k < 12; ++k) counts[k] = 0;
    for (int64_t p = 0; p < (int64_t)W * H; ++p) {
        if (gt_valid && !gt_valid[p]) continue;
        for (int split = 0; split < 2; ++split) {
            if (split == 1 && !gt_noc[p]) continue;
            long long *c = counts + 6 * split;
            c[0] += 1;
            if (!valid_sf[p]) continue;
            c[1] += 1;
            const float u = sf[4 * p + 0], v = sf[4 * p + 1];
            const float d0 = sf[4 * p + 2], d1 = sf[4 * p + 3];
            const float e1 = fabsf(d0 - gt_d0[p]);
            const float e2 = fabsf(d1 - gt_d1[p]);
            const float du = u - gt_flow[2 * p + 0], dv = v - gt_flow[2 * p + 1];
            const float du2 = du * du, dv2 = dv * dv;
            const float ef = sqrtf(du2 + dv2);
            const float gu2 = gt_flow[2 * p + 0] * gt_flow[2 * p + 0];
            const float gv2 = gt_flow[2 * p + 1] * gt_flow[2 * p + 1];
            const float mf = sqrtf(gu2 + gv2);
            const int o1 = kitti_outlier(e1, fabsf(gt_d0[p]), tau_abs, tau_rel);
            const int o2 = kitti_outlier(e2, fabsf(gt_d1[p]), tau_abs, tau_rel);
            const int of = kitti_outlier(ef, mf, tau_abs, tau_rel);
            c[2] += o1;
            c[3] += o2;
            c[4] += of;
            c[5] += (o1 || o2 || of);
        }
    }
    return 0;
}
