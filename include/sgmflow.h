/* sgmflow.h -- C ABI of the optical-flow core of arXiv 1801.04720 (Sec. 3.2 "Optical Flow
 * from Flow Fields+"): SURVEY.md 8(f) rank 2, the step that produces the flow F
 * the scene-flow combination consumes (sgm_scene_flow's `flow` / `flow_valid`).
 *
 * What it computes (SPEC flow-fields S:189-292, readings FF1-FF10 in DESIGN.md):
 *   - an image pyramid of `levels` 2x2-box levels ("initialized on a lower resolution");
 *   - at the coarsest level, 16 lowest-sequency Walsh-Hadamard coefficients per pixel and the
 *     k nearest descriptors of the other frame (exhaustive search, exactly the result of the
 *     paper's k-d tree query), keeping the candidate of least data term;
 *   - per level, `sweeps` propagation sweeps (alternating scan direction, left/up resp.
 *     right/down neighbours, strict improvement) each followed by a random search with a
 *     counter-based RNG and radius search_radius >> sweep (>= 1 px);
 *   - lift x2 to the next level;
 *   - the forward field and two inverse fields (seed+1 / radius r and seed+2 / radius r+2,
 *     F-5), and the consistency filter: a match survives iff it is consistent with BOTH
 *     inverse fields within consistency_q / 8 px ("If any match is inconsistent with any
 *     of the inverse fields, it gets filtered").
 * Flow vectors are integers in 1/8 px; the data term is the integer patch SAD of the
 * (2r+1)^2 window with bilinear target sampling in 1/64 weight steps and `penalty` per
 * sample outside the target image (F-2, F-3).  All decisions are exact: results are
 * bit-identical to the CPU oracle (oracle/flow_oracle.c) and deterministic.
 *
 * Images are uint8 grayscale, dense (row pitch = width).  All pointers are device memory
 * unless stated otherwise.  Calls are asynchronous on `stream` (a cudaStream_t, NULL =
 * legacy default stream) and use per-handle scratch: do not run two calls of one handle
 * concurrently.  Errors: SGM_ERR_INVALID_ARGUMENT for bad arguments (checked before any
 * work is enqueued), SGM_ERR_CUDA / SGM_ERR_OUT_OF_MEMORY from the runtime
 * (sgm_flow_last_error_string() has the detail).
 */
#ifndef SGMFLOW_H
#define SGMFLOW_H

#include "sgmsf.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sgm_flow_params {
    int32_t width, height;    /* level-0 image size, 1..16384 */
    int32_t levels;           /* pyramid levels 1..8 (SPEC default 3) */
    int32_t patch_radius;     /* r: (2r+1)^2 patch; r + 2 <= 7 (the second inverse field) (4) */
    int32_t sweeps;           /* propagation + random-search sweeps per level, 0..64 (8) */
    int32_t search_radius;    /* random-search radius of sweep 0 in px, >= 1 (8) */
    int32_t desc_window;      /* WHT window: 4, 8 or 16 (8) */
    int32_t knn;              /* nearest descriptors tried at initialisation, 1..8 (4) */
    int32_t consistency_q;    /* consistency threshold in 1/8 px, >= 0 (8 = 1.0 px) */
    int32_t penalty;          /* per-sample data term outside the target image, 0..255 (20) */
    int32_t max_batch;        /* most frame pairs per call, >= 1 */
    uint64_t seed;            /* RNG seed of the forward field (inverse fields: +1, +2) */
} sgm_flow_params;

typedef struct sgm_flow_handle sgm_flow_handle;

/* Create a handle on `device`, allocating scratch for max_batch pairs (synchronous).
 * `*out` is set only on SGM_OK. */
SGM_API sgm_status sgm_flow_create(const sgm_flow_params *p, int32_t device, sgm_flow_handle **out);
SGM_API void sgm_flow_destroy(sgm_flow_handle *h);
SGM_API const char *sgm_flow_last_error_string(void);
/* Kernels launched by this handle so far. */
SGM_API int64_t sgm_flow_launch_count(sgm_flow_handle *h);

/* The optical-flow step for n frame pairs: frames0 / frames1 [n][H][W] (frame t
 * and t+1 of the left camera).  Outputs (any may be NULL, not all): flow [n][H][W][2]
 * float32 (u, v) px = the forward field / 8 (exact), valid [n][H][W] the consistency mask
 * (pass both to sgm_scene_flow as flow / flow_valid); fields_q [n][3][H][W][2] int32 the
 * forward and the two inverse fields in 1/8 px.  1 <= n <= max_batch. */
SGM_API sgm_status sgm_flow(sgm_flow_handle *h, int32_t n, const uint8_t *frames0,
                    const uint8_t *frames1, float *flow, uint8_t *valid, int32_t *fields_q,
                    void *stream);

/* ---- densification ------------------------------- */
/* Edge-aware gap filling of a sparse field (SPEC densify S:253-262, decision F-6 "K-nearest
 * seeds under edge-aware line-integral distance with inverse-distance weights"; the gap
 * filling the paper delegates to EpicFlow, and the "Ours (All)" densification, P:147,
 * P:170): a pixel with valid != 0 keeps its values exactly; a gap pixel p takes the
 * 1/d_e-weighted mean of the K valid seeds s of smallest edge-aware distance
 *   d_e(p, s) = |p - s| + lambda * sum_k g(q_k)
 * (ties to the smaller linear index), q_k the interior points of the segment p -> s (n =
 * max(|dx|,|dy|) steps, rounded half up) and g the guide's L1 central-difference gradient
 * (readings DN1-DN4).  d_e is evaluated in fp64 as sqrt(|p-s|^2) + lambda * G, one rounding
 * each: the seed choice is reproducible bit for bit.  Candidates: window <= 0 = every seed of
 * the image (the SPEC's definition); window > 0 = the seeds within Chebyshev distance
 * max(window, rho_K(p)), rho_K(p) the smallest Chebyshev radius holding K seeds (a bounded-
 * cost approximation; pixels whose search provably found the window-0 answer -- the K-th d_e
 * fell below the ring radius -- are counted in *certified).  No handle: plain device
 * pointers, run on the device that owns `field`.
 *   field, out [n][H][W][C] float32 (C = 1..4: flow (u, v), scene flow (u, v, d0, d1), ...);
 *   valid, guide [n][H][W] uint8; 1 <= K <= 64; lambda >= 0 (gray levels -> px, 1.0);
 *   unfilled (device int32, nullable): number of pixels of images without any valid pixel
 *   (their output is 0, the SPEC's "zero valid pixels" error);
 *   certified (device int32, nullable): gap pixels with a provably window-0 result;
 *   scratch: device, 16-byte aligned, scratch_bytes >= sgm_densify_scratch_bytes(n, W, H)
 *   (row / column prefix counts, the gap list and the guide gradient); NULL = a stream-
 *   ordered allocation inside the call (slower, and not capturable in every CUDA-graph
 *   setting).  n * W * H < 2^31.
 * Ranking and weights in fp64, output float32. */
SGM_API sgm_status sgm_densify(int32_t n, int32_t width, int32_t height, int32_t channels,
                       const float *field, const uint8_t *valid, const uint8_t *guide,
                       int32_t K, float lambda, int32_t window, float *out, int32_t *unfilled,
                       int32_t *certified, void *scratch, int64_t scratch_bytes, void *stream);

/* Scratch bytes sgm_densify needs for n images of width x height (-1 if invalid). */
SGM_API int64_t sgm_densify_scratch_bytes(int32_t n, int32_t width, int32_t height);

/* ---- instrumentation ------------------------------------------------------ */
enum { SGM_FLOW_NUM_STAGES = 3 };   /* propagation (incl. the fused random search), -, kNN */

/* Enable (1) / disable (0) CUDA-event timing of the propagation kernels (the random search
 * runs inside them; stage 1 stays 0) and the kNN kernels of every following sgm_flow /
 * sgm_flow_field call (events on the call's stream). */
SGM_API sgm_status sgm_flow_set_timing(sgm_flow_handle *h, int32_t enable);

/* Summed kernel time (ms) per stage of the last timed call into ms[SGM_FLOW_NUM_STAGES]
 * (waits for its events); returns the number of stages written, 0 if nothing was timed. */
SGM_API int32_t sgm_flow_read_timing(sgm_flow_handle *h, float *ms);

/* ---- stage-wise entry points (parity tests, debugging) ------------------- */

/* One match field per pair, A_k -> B_k, through the whole pyramid with (seed, radius):
 * A, B [n][H][W]; flow_q [n][H][W][2] int32 (1/8 px); cost [n][H][W] (nullable). */
SGM_API sgm_status sgm_flow_field(sgm_flow_handle *h, int32_t n, const uint8_t *A, const uint8_t *B,
                          uint64_t seed, int32_t radius, int32_t *flow_q, int32_t *cost,
                          void *stream);

/* WHT descriptors of one w x hgt image: desc [hgt][w][16] int32 (16-byte aligned). */
SGM_API sgm_status sgm_flow_descriptors(sgm_flow_handle *h, const uint8_t *img, int32_t w,
                                int32_t hgt, int32_t *desc, void *stream);

/* Data term of nq queries {x, y, fu, fv} (fu, fv in 1/8 px) between w x hgt images A, B
 * with patch radius 0..7: out[nq]. */
SGM_API sgm_status sgm_flow_patch_cost(sgm_flow_handle *h, const uint8_t *A, const uint8_t *B,
                               int32_t w, int32_t hgt, int32_t radius, int32_t nq,
                               const int32_t *queries, int32_t *out, void *stream);

/* kNN initialisation of one field A -> B at a single level (w * hgt <= width * height):
 * flow_q [hgt][w][2], cost [hgt][w]; nn [hgt][w][knn] B indices (nullable). */
SGM_API sgm_status sgm_flow_knn_init(sgm_flow_handle *h, const uint8_t *A, const uint8_t *B,
                             int32_t w, int32_t hgt, int32_t radius, int32_t *flow_q,
                             int32_t *cost, int32_t *nn, void *stream);

/* One propagation sweep + random search of one field at a single level, in place on
 * flow_q [hgt][w][2] / cost [hgt][w] (cost must be the data term of flow_q); `level` and
 * `sweep` select the RNG stream and the scan direction (even: top-left first). */
SGM_API sgm_status sgm_flow_sweep(sgm_flow_handle *h, const uint8_t *A, const uint8_t *B, int32_t w,
                          int32_t hgt, int32_t radius, int32_t sweep, int32_t level,
                          uint64_t seed, int32_t *flow_q, int32_t *cost, void *stream);

/* Consistency mask of one forward field F against two inverse fields G1, G2 (all
 * [hgt][w][2] int32 in 1/8 px): valid [hgt][w]. */
SGM_API sgm_status sgm_flow_consistency(sgm_flow_handle *h, const int32_t *F, const int32_t *G1,
                                const int32_t *G2, int32_t w, int32_t hgt, uint8_t *valid,
                                void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SGMFLOW_H */
