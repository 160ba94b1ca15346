/*
 * sgmsf.h -- C ABI of the B200 (sm_100a) SGM stereo + basic scene flow library
 * (libsgmsf.so), implementing the hot path of Schuster et al., "Combining
 * Stereo Disparity and Optical Flow for Basic Scene Flow" (arXiv 1801.04720).
 *
 * Citations: P:n = PAPER.md line n (section / equation given), S:n = SPEC.md
 * line n, G# = reading
 *
 * General conventions
 *  - Every pointer argument is DEVICE memory of the handle's device unless the
 *    function name ends in _host.  The caller owns every input and output
 *    buffer; the handle owns only its scratch (allocated once in sgm_create).
 *    Nothing is allocated per call.
 *  - Layouts are row-major [H][W] (x fastest), with a trailing channel /
 *    disparity dimension where stated.  Images may carry a row pitch; every
 *    other buffer is dense.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call only enqueues work on `stream` and returns without a host
 *    synchronisation (except sgm_create / sgm_destroy).  Asynchronous device
 *    faults surface at the caller's next synchronisation.
 *  - Argument errors are detected synchronously, before anything is enqueued,
 *    and return SGM_ERR_INVALID_ARGUMENT.  Every CUDA failure seen after
 *    validation (launch or copy errors, whatever their CUDA code) returns
 *    SGM_ERR_CUDA.  No C++ exception crosses this ABI.
 *  - Device faults: the sweeps' cross-CTA waits are bounded; a wait that times
 *    out (a scheduling / logic error) writes a fault code into a host-mapped
 *    word of the handle, the affected rows store no disparities, and every
 *    later compute entry point of the handle returns SGM_ERR_CUDA until
 *    sgm_get_device_error(h, &code, 1) clears the fault.
 *  - A handle is bound to one device: every entry point makes that device
 *    current for the duration of the call and restores the caller's current
 *    device (of this library's runtime) on return.  A handle is not
 *    re-entrant: use one handle per concurrent stream.  Identical inputs give
 *    bit-identical outputs.
 */
#ifndef SGMSF_H
#define SGMSF_H

#include <stdint.h>

#if defined(__GNUC__)
#define SGM_API __attribute__((visibility("default")))
#else
#define SGM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sgm_status {
    SGM_OK = 0,
    SGM_ERR_INVALID_ARGUMENT = 1,
    SGM_ERR_UNSUPPORTED = 2,
    SGM_ERR_CUDA = 3,
    SGM_ERR_OUT_OF_MEMORY = 4
} sgm_status;

/* Method parameters (BASELINE.json configs). */
typedef struct sgm_params {
    int32_t width;          /* W >= 1: the shared image domain Omega */
    int32_t height;         /* H >= 1 */
    int32_t num_disp;       /* D disparity levels, d in [0, D-1] (G6); 1 <= D <= 256 */
    int32_t census_w;       /* census window width, odd (G2) */
    int32_t census_h;       /* census window height, odd; census_w*census_h-1 <= 63 (the
                               backward sweep reads the cost from 6 spare bits of S_fwd) */
    int32_t p1;             /* small-jump penalty P1, 0 <= P1 <= P2 (G8) */
    int32_t p2;             /* large-jump penalty P2; C_max + P2 <= 255 where
                               C_max = census_w*census_h-1 (G5, G9) */
    int32_t lr_threshold;   /* T >= 0, integer pixels (G13) */
    int32_t invalid_disp;   /* value written for invalid disparities (G14: -1) */
    int32_t bilinear_rule;  /* 0: taps with nonzero weight must be valid (G18);
                               1: all four taps valid (SPEC D-2) */
    int32_t max_batch;      /* >= 1: most frame quads one sgm_scene_flow call takes
                               (sizes the scratch) */
} sgm_params;

/* Pinhole camera of the rectified rig ("camera intrinsics and extrinsics";
 * G19/G20).  X right, Y down, Z forward, metres. */
typedef struct sgm_camera {
    float f_px;             /* focal length in pixels, > 0 */
    float baseline_m;       /* stereo baseline in metres, > 0 */
    float cx, cy;           /* principal point in pixels */
} sgm_camera;

typedef struct sgm_handle sgm_handle;

/* Result buffers of sgm_scene_flow (Eq. (3)/(4), P:96/P:118 3D).
 * Any pointer except sf and valid_sf may be NULL to skip that output. */
typedef struct sgm_sceneflow_out {
    float   *sf;            /* [n][H][W][4] = (u, v, d0, d1) (Eq. (3)); 0 where invalid */
    uint8_t *valid_sf;      /* [n][H][W] 1 = S(x) defined (Eq. (4)) */
    float   *p0;            /* [n][H][W][4] = (X, Y, Z, 0) of x at t (NULL: not stored) */
    float   *dp;            /* [n][H][W][4] = (dX, dY, dZ, 0) motion (NULL: skip 3D) */
    uint8_t *valid_3d;      /* [n][H][W] 1 = S valid and d0 > 0 and d1 > 0 (G21); required
                               with dp */
    int16_t *disp_int;      /* [n][2][H][W] LR-checked integer D0 (t), D1 (t+1) */
    float   *disp_sub;      /* [n][2][H][W] LR-checked sub-pixel D0, D1 (-1 invalid) */
    uint8_t *disp_valid;    /* [n][2][H][W] LR masks of D0, D1 */
} sgm_sceneflow_out;

/* Create a handle on `device`: validates `p` (SGM_ERR_INVALID_ARGUMENT on: W
 * or H < 1, D outside 1..256, even census side, a 1x1 census window (no bits),
 * census_w*census_h-1 > 63, P1 < 0, P2 < P1, C_max+P2 > 255, T < 0,
 * bilinear_rule not 0/1, max_batch < 1; SGM_ERR_UNSUPPORTED on H > 65535,
 * W*H >= 2^31, 2*max_batch > 65535 or a census side > 17 -- launch-geometry
 * limits of the kernels, checked here so that no later call fails half-way
 * through its launches) and allocates all scratch for max_batch quads
 * (SGM_ERR_OUT_OF_MEMORY if that fails).  Synchronous; the caller's current
 * device is restored.  `*out` is set only on SGM_OK. */
SGM_API sgm_status sgm_create(const sgm_params *p, int32_t device, sgm_handle **out);

/* Free the handle and its scratch after synchronising the device.  NULL-safe. */
SGM_API void sgm_destroy(sgm_handle *h);

/* Static description of a status code (never NULL). */
SGM_API const char *sgm_status_string(sgm_status s);

/* Human-readable description of the most recent CUDA failure seen by this
 * thread inside the library (e.g. "cudaErrorInvalidValue: invalid argument"). */
SGM_API const char *sgm_last_error_string(void);

/* Census transform of one uint8 image (G2-G4): out[y][x] bit k =
 * [neighbour k < centre] over the census_w x census_h window scanned row-major
 * (dy outer, dx inner), centre skipped, coordinates clamped to the image.
 * img: [H] rows of `pitch_bytes` (pitch >= W, pitch % 16 == 0, img 16-byte
 * aligned: the tile is staged by TMA).  census: [H][W] uint64, LSB = bit 0. */
SGM_API sgm_status sgm_census(sgm_handle *h, const uint8_t *img, int64_t pitch_bytes,
                      uint64_t *census, void *stream);

/* Matching cost volume of one view (G5, G12), debug / parity path:
 * view 0 (left reference): C(x,y,d) = popcount(cen_left(x,y) ^ cen_right(x-d,y));
 * view 1 (right reference): C(x,y,d) = popcount(cen_right(x,y) ^ cen_left(x+d,y));
 * a match outside the image costs C_max = census_w*census_h-1.
 * cost: [H][W][D] uint8. */
SGM_API sgm_status sgm_cost(sgm_handle *h, const uint64_t *cen_left, const uint64_t *cen_right,
                    int32_t view, uint8_t *cost, void *stream);

/* Aggregated cost S = sum over the 8 paths (recursion S:129,
 * G7) of one view, computed by the fused cost+aggregation sweeps and
 * materialised for parity: agg [H][W][D] uint16 (S <= 8*(C_max+P2), G9).
 * view as in sgm_cost.  Uses the handle's view-0 scratch. */
SGM_API sgm_status sgm_aggregate(sgm_handle *h, const uint64_t *cen_left, const uint64_t *cen_right,
                         int32_t view, uint16_t *agg, void *stream);

/* Winner-take-all + parabola sub-pixel (G10/G11) on a materialised
 * agg [H][W][D] uint16: d_int = smallest argmin, d_sub = d_int + (a-c)/(2(a+c-2b))
 * for 0 < d_int < D-1 (float32, IEEE division), else d_int.  Every pixel gets a
 * value.  d_int [H][W] int16, d_sub [H][W] float32. */
SGM_API sgm_status sgm_wta(sgm_handle *h, const uint16_t *agg, int16_t *d_int, float *d_sub,
                   void *stream);

/* Left-right consistency check (integer reading G13):
 * valid(x,y) iff x - dl(x,y) >= 0 and |dl(x,y) - dr(x - dl(x,y), y)| <= T.
 * out_int / out_sub = dl_int / dl_sub where valid, else invalid_disp; valid
 * [H][W] uint8.  dl_int, dr_int [H][W] int16 raw WTA maps of the left- and
 * right-reference views; dl_sub [H][W] float32. */
SGM_API sgm_status sgm_lr_check(sgm_handle *h, const int16_t *dl_int, const float *dl_sub,
                        const int16_t *dr_int, int16_t *out_int, float *out_sub,
                        uint8_t *valid, void *stream);

/* Whole SGM on one rectified pair: census of both
 * images, fused cost+8-path aggregation of the left- and right-reference views,
 * WTA + sub-pixel, LR check.  Equals the stage-wise composition
 * sgm_census -> sgm_aggregate -> sgm_wta -> sgm_lr_check bit for bit.
 * left/right as in sgm_census (same pitch); outputs as in sgm_lr_check. */
SGM_API sgm_status sgm_disparity(sgm_handle *h, const uint8_t *left, const uint8_t *right,
                         int64_t pitch_bytes, int16_t *out_int, float *out_sub,
                         uint8_t *valid, void *stream);

/* Combination Eq. (4) with the bilinear warp of Eq. (5) and the 3D
 * interpretation (G15-G23):
 *   x' = x + F(x) in float32; defined iff F valid, d0 valid, 0 <= x' <= W-1,
 *   0 <= y' <= H-1 and D1 valid on the bilinear footprint (bilinear_rule);
 *   sf = (u, v, d0(x), D1(x')) else 0;  Z = f B / d, X = (x-cx) Z / f,
 *   Y = (y-cy) Z / f; p0 from (x, d0), end point from (x', d1), dp = P1 - P0;
 *   valid_3d = valid_sf and d0 > 0 and d1 > 0.
 * d0, d1 [H][W] float32 (LR-checked sub-pixel maps at t, t+1); v0, v1 [H][W]
 * uint8; flow [H][W][2] float32 (u, v); flow_valid nullable (all valid, G23);
 * sf [H][W][4]; dp [H][W][4] nullable (skip 3D; then valid_3d may be NULL); p0
 * [H][W][4] nullable (P0 is still computed for dp but not stored).
 */
SGM_API sgm_status sgm_combine_sceneflow(sgm_handle *h, const float *d0, const uint8_t *v0,
                                 const float *d1, const uint8_t *v1, const float *flow,
                                 const uint8_t *flow_valid, const sgm_camera *cam,
                                 float *sf, float *p0, float *dp, uint8_t *valid_sf,
                                 uint8_t *valid_3d, void *stream);

/* The whole hot path for n independent frame quadruples (Fig. 2):
 * SGM at t and t+1 (4 census images, 4 views, 2 LR checks) and the
 * combination + 3D, as 5 kernel launches for the whole batch.
 * images: [n][4][H] rows of pitch_bytes, order I_l^t, I_r^t, I_l^{t+1},
 * I_r^{t+1} (pitch % 16 == 0, 16-byte aligned); flow: [n][H][W][2];
 * flow_valid: [n][H][W] or NULL; 1 <= n <= max_batch. */
SGM_API sgm_status sgm_scene_flow(sgm_handle *h, int32_t n, const uint8_t *images, int64_t pitch_bytes,
                          const float *flow, const uint8_t *flow_valid,
                          const sgm_camera *cam, const sgm_sceneflow_out *out, void *stream);

/* Same as sgm_scene_flow but every buffer (inputs and the non-NULL outputs of
 * *out) is HOST memory, densely packed ([n][4][H][W] images).  The call enqueues,
 * on internal streams of the handle, a 1D host->device copy into one of two
 * staging slots, the pipeline, and device->host copies of the requested outputs,
 * then makes `stream` wait for the copies; the results are available after the
 * caller synchronises `stream`.  Consecutive host-entry calls on a handle are
 * ordered among themselves through the slots' events, not through `stream`, so
 * calls issued back to back pipeline: the upload of call k+1 and the download of
 * call k-1 overlap the kernels of call k.  Use page-locked host memory, keep the
 * host buffers of a call untouched until its results are available, and do not
 * interleave other entry points of the same handle without synchronising. */
SGM_API sgm_status sgm_scene_flow_host(sgm_handle *h, int32_t n, const uint8_t *images,
                               const float *flow, const uint8_t *flow_valid,
                               const sgm_camera *cam, const sgm_sceneflow_out *out,
                               void *stream);

/* ---- streaming (video) mode ---------------------- */
/* n consecutive scene-flow quads of ONE stereo video share their frames: quad k =
 * (frame k, frame k+1), so each frame's LR-checked disparity map is computed once and
 * serves as D1 of quad k-1 and D0 of quad k -- n+1 SGM pairs instead of 2n (the reuse
 * the paper names as future work).  Every quad's results are bit-identical to
 * sgm_scene_flow on (frame k, frame k+1).
 *   images: [n+1][2][H] rows of pitch_bytes, frame k = (I_l^k, I_r^k) (pitch % 16 == 0,
 *   16-byte aligned); flow: [n][H][W][2] from frame k to k+1; flow_valid [n][H][W] or
 *   NULL; out->sf, valid_sf, p0, dp, valid_3d: per quad, [n][...] as in sgm_scene_flow;
 *   out->disp_int / disp_sub / disp_valid (optional): per FRAME, [n+1][H][W].
 * 1 <= n <= max_batch.  5 kernel launches for the whole video segment. */
SGM_API sgm_status sgm_scene_flow_stream(sgm_handle *h, int32_t n, const uint8_t *images,
                                 int64_t pitch_bytes, const float *flow,
                                 const uint8_t *flow_valid, const sgm_camera *cam,
                                 const sgm_sceneflow_out *out, void *stream);

/* Host-buffer twin of sgm_scene_flow_stream, pipelined exactly like
 * sgm_scene_flow_host: images dense [n+1][2][H][W] pinned host memory, the other
 * buffers host memory with the shapes above. */
SGM_API sgm_status sgm_scene_flow_stream_host(sgm_handle *h, int32_t n, const uint8_t *images,
                                      const float *flow, const uint8_t *flow_valid,
                                      const sgm_camera *cam, const sgm_sceneflow_out *out,
                                      void *stream);

/* ---- evaluation ---------------------------------- */
/* KITTI scene-flow outlier counts for n quadruples (Table 1 semantics P:130-155,
 * "Est" = sparse evaluation; density P:159; outlier rule SPEC E-1 / S:467, an
 * external convention the paper invokes as "the KITTI metric").  Over the
 * ground-truth pixels (gt_valid != 0; NULL = every pixel) that the estimate covers
 * (valid_sf != 0), a pixel is a D1 / D2 / Fl outlier iff its error exceeds tau_abs
 * AND tau_rel x the ground-truth magnitude:  D1 |d0 - gt_d0|, D2 |d1 - gt_d1|,
 * Fl ||(u,v) - gt_flow|| against ||gt_flow||, each decided in float32 with
 * separately rounded operations; SF = outlier in any of the three.  Split 0 = all
 * ground-truth pixels ("Occ"), split 1 = those with gt_noc != 0 ("Noc").
 *   sf [n][H][W][4], valid_sf [n][H][W]  (sgm_scene_flow's outputs);
 *   gt_d0, gt_d1 [n][H][W] float32 (gt_d1 = disparity at t+1 of the point seen
 *   at x, i.e. already warped to frame t); gt_flow [n][H][W][2] float32;
 *   gt_valid (nullable), gt_noc [n][H][W] uint8.  All device memory, sf 16-byte and
 *   gt_flow 8-byte aligned.
 *   counts: device [n][2][6] uint64 = {n_gt, n_eval, n_d1, n_d2, n_fl, n_sf} per
 *   split; overwritten (integer sums in a fixed order: deterministic).  Uses
 *   per-handle scratch: do not run two sgm_evaluate calls of one handle concurrently.
 *   Rates = n_x / n_eval, density = n_eval / n_gt.
 * SGM_ERR_INVALID_ARGUMENT on NULL required pointers, misalignment, n outside
 * 1..max_batch, tau_abs < 0 or tau_rel < 0 (or NaN), counts not 8-byte aligned.
 * One kernel launch. */
SGM_API sgm_status sgm_evaluate(sgm_handle *h, int32_t n, const float *sf, const uint8_t *valid_sf,
                        const float *gt_d0, const float *gt_d1, const float *gt_flow,
                        const uint8_t *gt_valid, const uint8_t *gt_noc, float tau_abs,
                        float tau_rel, uint64_t *counts, void *stream);

/* KITTI rates from one [2][6] count block of sgm_evaluate (E3): for each
 * split (0 = Occ, 1 = Noc) rates[split][0..3] = 100 * {n_d1, n_d2, n_fl, n_sf} / n_eval
 * (percent of the evaluated pixels) and rates[split][4] = 100 * n_eval / n_gt (density,
 * percent); a zero denominator gives NaN.  Host memory in and out (copy the device counts
 * back first), no handle, no device work, thread-safe.  SGM_ERR_INVALID_ARGUMENT on NULL. */
SGM_API sgm_status sgm_eval_rates(const uint64_t *counts, double *rates);

/* ---- instrumentation ----------------------------------------------------- */
enum { SGM_NUM_STAGES = 5 };   /* census, sweep_fwd, sweep_bwd_wta, lr_check, combine */

/* Enable (1) / disable (0) CUDA-event timing of every kernel that
 * sgm_scene_flow / sgm_scene_flow_host enqueue (events are recorded on the
 * launch stream, also inside CUDA-graph capture). */
SGM_API sgm_status sgm_set_timing(sgm_handle *h, int32_t enable);

/* After the caller synchronised the stream: per-stage durations (ms) of the
 * last timed sgm_scene_flow call into ms[SGM_NUM_STAGES].  Returns the number
 * of stages written (0 if timing was off or nothing ran). */
SGM_API int32_t sgm_read_timing(sgm_handle *h, float *ms);

/* Static stage name for index 0..SGM_NUM_STAGES-1 ("?" otherwise). */
SGM_API const char *sgm_stage_name(int32_t stage);

/* Number of kernels this handle has launched so far (all entry points). */
SGM_API int64_t sgm_launch_count(sgm_handle *h);

/* Internal geometry, for tests and roofline accounting: padded disparity
 * count Dp (multiple of 64), cells per lane, compute warps per CTA of the
 * sweeps (the maximum band height, 17), and the band height chosen for a full
 * batch (each call picks bands of 10..17 rows so that its CTA count fills
 * whole waves of the device's SMs). Any pointer may be NULL. */
SGM_API sgm_status sgm_get_geometry(sgm_handle *h, int32_t *dp, int32_t *cells_per_lane,
                            int32_t *sweep_warps, int32_t *band_rows);

/* Debugging aid: when `trace` (device memory, >= 4 * (sweep_warps + 1) * 4 * max_batch *
 * ceil(H / 10) uint64) is non-NULL, every sweep CTA warp writes {start ns, end ns,
 * SM id, 0} of its row loop at index (ticket * (sweep_warps + 1) + warp) * 4 (the last
 * launch wins).  NULL disables it (default). */
SGM_API sgm_status sgm_debug_set_trace(sgm_handle *h, uint64_t *trace);

/* Device fault word of the handle (see "Device faults" above): *code = 0 (no fault),
 * 1 (a backward-sweep row timed out waiting for its view's forward sweep) or 2 (a band
 * timed out waiting for the band above it).  Reads host memory: call it after
 * synchronising the stream of the call in question.  clear != 0 resets the word, after
 * which the entry points work again.  code may be NULL. */
SGM_API sgm_status sgm_get_device_error(sgm_handle *h, int32_t *code, int32_t clear);

/* Debugging / fault-injection flags of the sweeps (default: env SGM_DEBUG_FLAGS or 0):
 * 1 = no inter-warp / inter-band waits, 2 = no band handoff (both give WRONG results;
 * timing experiments only), 4 = force every bounded cross-CTA wait to time out (tests
 * the fault reporting), 16 = keep the consumed band-handoff lines in L2 (no discard;
 * traffic experiments).  SGM_ERR_INVALID_ARGUMENT outside 0..31. */
SGM_API sgm_status sgm_debug_set_flags(sgm_handle *h, int32_t flags);

#ifdef __cplusplus
}
#endif
#endif /* SGMSF_H */
