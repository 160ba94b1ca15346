// sgm_internal.cuh -- device-side building blocks shared by the sm_100a kernels
// of libsgmsf.so.  Nothing here is shared with oracle/ (the CPU oracle).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sgm {

// ----------------------------------------------------------------- constants
// (the SGM_* macros select A/B variants of the sweep geometry; the defaults are the product)
#ifndef SGM_NW
#define SGM_NW 17
#endif
#ifndef SGM_RING_WIDE
#define SGM_RING_WIDE 16
#endif
#ifndef SGM_G_WIDE
#define SGM_G_WIDE 0
#endif
#ifndef SGM_MINB
#define SGM_MINB 1
#endif
constexpr int kRing = 8;        // row->row handoff ring (positions) for CPL > 4
constexpr int kRingWide = SGM_RING_WIDE;   // ... for CPL <= 4 (fits 16 warps x 16 x 3 x 256 B)
constexpr int kGroupWide = SGM_G_WIDE;     // ring sync group for CPL <= 4 (0: CPL positions)
constexpr int kSweepCtasPerSm = SGM_MINB;  // resident sweep CTAs per SM
#ifndef SGM_FINE_GROUP
#define SGM_FINE_GROUP 1
#endif
constexpr int kFineGroup = SGM_FINE_GROUP; // ring sync group of the latency mode (CPL <= 4)
constexpr int kRing0 = 16;      // band-input ring of warp 0 (positions)
constexpr int kPublish = 8;     // forward sweep's band-output publication granularity (positions)
constexpr int kPubDepth = 4;    // producer -> publisher-warp handoff depth (groups)
// SGM sweep bands: a CTA carries one band of up to kBandRowsMax rows (one compute warp per
// row); the host picks the band height per call in [kBandRowsMin, kBandRowsMax] so that
// the CTA count fills whole waves of the SMs (band_geometry in api.cu)
constexpr int kBandRowsMax = SGM_NW;
constexpr int kBandRowsMin = SGM_NW < 10 ? SGM_NW : 10;

// ----------------------------------------------------------------- kernel params
struct SweepParams {
    int W, H, D, Dp;
    int P1, P2, cmax;
    int nviews, nbands;
    int band_q, band_r;       // band b has band_q + (b < band_r) rows, from row b*band_q + min(b, band_r)
    int vgroup;               // ticket order: groups of vgroup views, band-major inside a group
    int fine_sync;            // latency mode (< 2 waves of CTAs): finer row-to-row sync groups
    // u16x2 constants of the path update, precomputed on the host (kernel-parameter operands
    // instead of per-lane registers): P1, -P1, P2 - P1, 2 P1 in both halves, -4 P1 (S bias)
    uint32_t k_p1x2, k_negp1x2, k_p2mp1x2, k_twop1x2, k_negb4;
    // census images [img][H][W]; batch views: view v -> pair v/2, side v%2
    //   side 0: ref = img 2*(v/2), match = img 2*(v/2)+1, mirror 0 (left reference)
    //   side 1: ref = img 2*(v/2)+1, match = img 2*(v/2), mirror 1 (right reference)
    const uint64_t *cen;
    long long cen_img_stride;
    // explicit single-view mode (sgm_aggregate / sgm_disparity with user census)
    int explicit_mode;
    const uint64_t *ref0, *match0;
    int mirror0;
    // forward-sweep sum S_fwd [view][H][W][Dp] in view coordinates (mirrored for right views)
    uint16_t *sfwd;
    long long sfwd_view_stride;
    // backward-sweep outputs
    int16_t *dint;            // [view][H][W] raw WTA (original x)
    float *dsub;              // [view][H][W]
    long long disp_view_stride;
    uint16_t *sout;           // debug: S [H][W][D] of view 0 (original x), or null
    // inter-band handoff
    uint16_t *gbuf;           // [view][band][W][3][Dp]
    int *progress;            // [view][band]
    int *ticket;              // CTA ticket counter (zeroed before launch)
    int *fwd_done;            // [view] forward-sweep rows finished (the backward sweep's band 0
                              // starts a view once it reaches H: the two launches overlap)
    unsigned long long *trace; // debug: per (ticket, warp) {start ns, end ns, smid, 0} or null
    int debug_flags;           // debug (env SGM_DEBUG_FLAGS / sgm_debug_set_flags): 1 = no
                               // inter-warp/band waits, 2 = no band handoff, 4 = force the
                               // bounded cross-CTA waits to time out (fault-reporting test)
    int one;                   // always 1 (opaque to the compiler: keeps adds on the FMA pipe)
    int *err;                  // device fault word (mapped host memory) or null: a timed-out
                               // cross-CTA wait stores its SGM_FAULT_* code here
};

// device fault codes written into SweepParams::err (reported by sgm_get_device_error)
constexpr int kFaultFwdDone = 1;     // backward sweep: the view's forward sweep never completed
constexpr int kFaultBandInput = 2;   // a band's predecessor never published its last row

// Sets the calling thread's current device for the lifetime of the object and restores
// the previous one (the library links a static cudart, whose current device is separate
// from the caller's runtime; every entry point of a handle runs on the handle's device).
struct DeviceGuard {
    int prev = -1;
    cudaError_t status = cudaSuccess;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) { cudaGetLastError(); prev = -1; }
        if (prev != dev) status = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard &) = delete;
    DeviceGuard &operator=(const DeviceGuard &) = delete;
};

struct CensusParams {
    int W, H, cw, ch, nimg;
};

struct LrParams {
    int W, H, T, invalid, npairs;
    const int16_t *dl; const float *dls; const int16_t *dr;
    long long in_stride_l, in_stride_r;   // elements between consecutive pairs
    int16_t *out_int; float *out_sub; uint8_t *valid;
    long long out_stride;
};

struct CombineParams {
    int W, H, rule, nquads;
    const float *d0, *d1; const uint8_t *v0, *v1;
    long long disp_stride;                 // elements between quads for d0/d1/v0/v1
    const float *flow; const uint8_t *flow_valid;
    float f, B, cx, cy, fB;
    float *sf, *p0, *dp; uint8_t *valid_sf, *valid_3d;
    // fused LR check (raw_int != nullptr): the LR-checked maps are not materialised; the
    // kernel applies the check (G13) to the raw WTA maps of the views [2 * pair + side] at the
    // pixels it reads.  Quad q uses pairs q * pair_step (t) and q * pair_step + 1 (t+1).
    const int16_t *raw_int; const float *raw_sub;
    long long view_stride;                 // elements between consecutive views
    int pair_step, T;
    float invalid;
};

struct EvalParams {
    int W, H, nquads;
    const float *sf; const uint8_t *valid_sf;
    const float *gt_d0, *gt_d1, *gt_flow; const uint8_t *gt_valid, *gt_noc;
    float tau_abs, tau_rel;
    unsigned long long *counts;            // [nquads][2][6]
    unsigned *part;                        // [grid blocks][12] block partials (scratch)
    unsigned *ticket;                      // zero between launches (the last block resets it)
};

// Optical-flow fields of a batch (flow.cu): pair k's level images A_k = A + k img_stride,
// B_k = B + k img_stride; field f = k fpp + kind (kind 0: A->B; 1, 2: B->A, F-5).
struct FFFields {
    int W, H, fpp, nfields;
    const uint8_t *A, *B;
    long long img_stride;          // elements between pairs (also for QA / QB)
    const uint32_t *QA, *QB;       // quad images of A, B (flow.cu ff_quad_kernel)
    int radius[3];
    uint64_t seed[3];
    int penalty;
    int32_t *flow;                 // [nfields][H][W][2] (1/8 px)
    int32_t *cost;                 // [nfields][H][W]
};

// Densification (densify.cu): n images of W x H, C channels
struct DensifyParams {
    int n, W, H, C, K;
    float lambda;
    int window;                    // <= 0: every seed competes; > 0: Chebyshev max(window, rho_K)
    const float *field;            // [n][H][W][C]
    const uint8_t *valid, *guide;  // [n][H][W]
    float *out;                    // [n][H][W][C]
    int *unfilled;                 // nullable: pixels left without a seed
    int *certified;                // nullable: gap pixels whose result provably equals window 0
};

// ----------------------------------------------------------------- launchers (host)
cudaError_t launch_census(const uint8_t *const *imgs, int nimg, long long pitch, int W, int H,
                          int cw, int ch, uint64_t *out, long long out_stride, cudaStream_t st);
cudaError_t launch_cost(const uint64_t *ref, const uint64_t *match, int W, int H, int D, int s,
                        int cmax, uint8_t *cost, cudaStream_t st);
size_t sweep_sync_ints(int nviews, int nbands);   // ints of a call's sweep sync buffer
cudaError_t launch_sweeps(const SweepParams &p, int cpl, bool c64, int nw, bool debug_s,
                          cudaStream_t st, cudaEvent_t mid_ev_a, cudaEvent_t mid_ev_b,
                          int *launches);
cudaError_t launch_wta(const uint16_t *agg, int W, int H, int D, int16_t *dint, float *dsub,
                       cudaStream_t st);
cudaError_t launch_lr(const LrParams &p, cudaStream_t st);
cudaError_t launch_repitch(const uint8_t *src, uint8_t *dst, int W, long long pitch, long long rows,
                           cudaStream_t st);
cudaError_t launch_combine(const CombineParams &p, cudaStream_t st);
cudaError_t launch_evaluate(const EvalParams &p, cudaStream_t st);
cudaError_t launch_densify(const DensifyParams &p, void *scratch, cudaStream_t st);
size_t densify_scratch_bytes(int n, int W, int H);
int evaluate_max_blocks();   // scratch rows launch_evaluate may use besides one per quad
cudaError_t ff_launch_downsample(const uint8_t *src, long long src_stride, int W, int H, uint8_t *dst,
                                 long long dst_stride, int nimg, cudaStream_t st);
cudaError_t ff_launch_wht(const uint8_t *img, long long img_stride, int W, int H, int win, int nimg,
                          int32_t *desc, cudaStream_t st);
cudaError_t ff_launch_knn(const int32_t *desc, int n, int nprob, int knn, int win, int32_t *nn, void *scratch,
                          cudaStream_t st);
size_t ff_knn_scratch_bytes(long long entries);
size_t ff_knn_tc_scratch_bytes(long long entries);
cudaError_t ff_launch_knn_tc(const int32_t *desc, int n, int nprob, int knn, int32_t *nn, void *scratch,
                             cudaStream_t st);
cudaError_t ff_launch_init(const FFFields &F, const int32_t *nn, int knn, cudaStream_t st);
cudaError_t ff_launch_lift(const FFFields &F, const int32_t *coarse, int Wc, int Hc, cudaStream_t st);
// stage timer of the flow handle (flow_api.cu): begin(category) / end() around a launch
struct FFTimer {
    virtual void begin(int cat) = 0;
    virtual void end() = 0;
};
cudaError_t ff_launch_sweep(const FFFields &F, int sweep, int level, int R0, int *sync, cudaStream_t st,
                            int *launches, FFTimer *timer = nullptr);
long long ff_sync_ints(int nfields, int W, int H);
size_t ff_prop_smem(int W);
cudaError_t ff_launch_consistency(const int32_t *F, const int32_t *G1, const int32_t *G2, long long fstride,
                                  long long gstride, int W, int H, int n, int thr_q, uint8_t *valid,
                                  float *fout, cudaStream_t st);
cudaError_t ff_launch_cost_query(const uint8_t *A, const uint32_t *QB, int W, int H, int r, int penalty, int nq,
                                 const int32_t *q, int32_t *out, cudaStream_t st);
cudaError_t ff_launch_quad(const uint8_t *src, long long src_stride, int W, int H, int nimg, uint32_t *dst,
                           long long dst_stride, cudaStream_t st);

}  // namespace sgm
