// api.cu -- the C ABI of libsgmsf.so (include/sgmsf.h): handle, validation, scratch,
// launch orchestration on the caller's stream, status codes, instrumentation.
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <cstring>
#include <new>

#include "../../include/sgmsf.h"
#include "sgm_internal.cuh"

namespace sgm {
cudaError_t launch_census_stack(const uint8_t *base, long long img_stride, int nimg, long long pitch,
                                int W, int H, int cw, int ch, uint64_t *out, long long out_stride,
                                cudaStream_t st);
int sweep_warps_for(int cpl);
}  // namespace sgm

struct sgm_handle {
    sgm_params prm;
    int device = 0;
    int cpl = 0, dp = 0, nw = 0;
    int nbands = 0;                 // allocated bands per view: ceil(H / kBandRowsMin)
    int nsm = 148;                  // SMs of the device (band_geometry)
    bool c64 = false;
    int cmax = 0;
    long long npx = 0;
    int max_views = 0;
    // scratch (device)
    uint64_t *census = nullptr;     // [4*max_batch][H][W]
    uint16_t *sfwd = nullptr;       // [4*max_batch][H][W][Dp], after a front guard
    uint16_t *sfwd_alloc = nullptr; // the allocation: kSfwdGuard positions of Dp, then sfwd
    int16_t *dint = nullptr;        // [4*max_batch][H][W]
    float *dsub = nullptr;          // [4*max_batch][H][W]
    int16_t *lr_int = nullptr;      // [2*max_batch][H][W]
    float *lr_sub = nullptr;
    uint8_t *lr_valid = nullptr;
    uint16_t *gbuf = nullptr;       // 2 x [4*max_batch][bands of the call][W][3][Dp] (<= nbands)
    int *sync = nullptr;            // sweep sync buffer (sgm::sweep_sync_ints ints)
    unsigned *eval_part = nullptr;  // [evaluate_max_blocks() + max_batch][12] + ticket
    // staging for the _host entry point (device): two slots so that back-to-back calls
    // pipeline (upload of call k+1 and download of call k-1 overlap the kernels of call k)
    long long stage_pitch = 0;
    struct Stage {
        uint8_t *img_dense = nullptr;   // [max_batch][4][H][W] (1D host copy target)
        uint8_t *img = nullptr;         // [max_batch][4][H][pitch]
        float *flow = nullptr;          // [max_batch][H][W][2]
        uint8_t *fvalid = nullptr;      // [max_batch][H][W]
        float *sf = nullptr, *p0 = nullptr, *dp = nullptr;   // [max_batch][H][W][4]
        uint8_t *vsf = nullptr, *v3 = nullptr;               // [max_batch][H][W]
        int16_t *di = nullptr; float *ds = nullptr; uint8_t *dv = nullptr;   // [max_batch][2][H][W]
        cudaEvent_t ev_in = nullptr, ev_comp = nullptr, ev_out = nullptr;
        bool used = false;
    } stage[2];
    int slot = 0;
    cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
    int *sync_host = nullptr;       // sweep sync buffer of the host entry's compute stream
    // instrumentation
    bool timing = false;
    bool timed = false;
    cudaEvent_t ev[SGM_NUM_STAGES + 1] = {};
    long long launches = 0;
    unsigned long long *trace = nullptr;   // debug timeline buffer (caller-owned, device)
    int debug_flags = 0;                   // SweepParams::debug_flags (env SGM_DEBUG_FLAGS)
    // device fault word: mapped pinned host memory the sweeps write a fault code into when a
    // bounded cross-CTA wait times out; every compute entry point checks it (no sync needed)
    int *err_host = nullptr;
    int *err_dev = nullptr;
};

namespace {

thread_local char g_last_error[256] = "no error";

sgm_status from_cuda(cudaError_t e) {
    if (e == cudaSuccess) return SGM_OK;
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    // argument errors are caught by the entry points' validation before anything is
    // enqueued; a CUDA error seen afterwards (any code) is a CUDA failure
    if (e == cudaErrorMemoryAllocation) return SGM_ERR_OUT_OF_MEMORY;
    return SGM_ERR_CUDA;
}

// A fault word set by an earlier kernel (sticky until sgm_get_device_error clears it)
// makes every compute entry point fail; the word is host memory, so no sync is needed.
bool device_faulted(const sgm_handle *h) {
    const int code = h->err_host ? *reinterpret_cast<volatile const int *>(h->err_host) : 0;
    if (code == 0) return false;
    snprintf(g_last_error, sizeof(g_last_error),
             "device fault %d: a sweep's cross-CTA wait timed out (%s); results of that call are "
             "invalid -- sgm_get_device_error clears the fault", code,
             code == sgm::kFaultFwdDone ? "forward sweep never completed" : "band input never published");
    return true;
}

// Entry-point prologue: the handle's device becomes current for the call (restored on
// return) and a pending device fault is reported.
#define SGM_ENTRY(h)                                                  \
    sgm::DeviceGuard guard_((h)->device);                             \
    if (guard_.status != cudaSuccess) return from_cuda(guard_.status); \
    if (device_faulted(h)) return SGM_ERR_CUDA;

template <class T>
cudaError_t dalloc(T **p, size_t count) {
    return cudaMalloc(reinterpret_cast<void **>(p), count * sizeof(T) + 256);
}

void free_all(sgm_handle *h) {
    void *ptrs[] = {h->census, h->sfwd_alloc, h->dint, h->dsub, h->lr_int, h->lr_sub, h->lr_valid,
                    h->gbuf, h->sync, h->sync_host, h->eval_part};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (h->err_host) cudaFreeHost(h->err_host);
    for (auto &st : h->stage) {
        void *sp[] = {st.img_dense, st.img, st.flow, st.fvalid, st.sf, st.p0, st.dp, st.vsf, st.v3,
                      st.di, st.ds, st.dv};
        for (void *p : sp)
            if (p) cudaFree(p);
        for (cudaEvent_t e : {st.ev_in, st.ev_comp, st.ev_out})
            if (e) cudaEventDestroy(e);
    }
    for (cudaStream_t s : {h->s_in, h->s_comp, h->s_out})
        if (s) cudaStreamDestroy(s);
    for (auto &e : h->ev)
        if (e) cudaEventDestroy(e);
}

// Band height of the sweeps for a call with `nviews` views (one CTA per band, one CTA per
// SM).  Rule fitted to measurements on this B200 (K2):
//  * with >= 2 waves of 16-row bands, 16 rows (4 compute warps per SM sub-partition) are
//    the most efficient; 17 rows (18 warps: 5 compute warps on one sub-partition) only pay
//    when they save a whole wave (32 Driving views, H = 375: 23 bands of 16-17 rows = 736
//    CTAs = 5 waves instead of 24 x 16 = 768 CTAs = 6; 7.30 -> 7.17 ms per step);
//  * below 2 waves the SMs are under-filled and shorter bands spread the work: the height
//    in [kBandRowsMin, 16] minimising ceil(CTAs / SMs) * T(h), T(h) = h/16 (1 + 0.012
//    (16 - h)) (fewer warps hide less latency), is taken (one Driving quad: 35 bands of
//    10-11 rows on 140 SMs instead of 24 x 16 on 96: 3.46 -> 3.31 ms).
// Rows are spread evenly over the bands (heights differ by <= 1).  SGM_BAND_ROWS
// (environment, experiments) forces the height.
void band_geometry(int H, int nviews, int nsm, int *nbands, int *q, int *r) {
    static const int forced = [] {
        const char *e = getenv("SGM_BAND_ROWS");
        return e ? atoi(e) : 0;
    }();
    constexpr int hi = sgm::kBandRowsMax, lo = hi > sgm::kBandRowsMin ? hi - 1 : hi;
    nsm *= sgm::kSweepCtasPerSm;                   // CTA slots
    auto bands = [&](int rows) { return (H + rows - 1) / rows; };
    auto waves = [&](int nb) { return ((long long)nviews * nb + nsm - 1) / nsm; };
    int nb;
    if (forced >= sgm::kBandRowsMin && forced <= sgm::kBandRowsMax) {
        nb = bands(forced);
    } else if ((long long)nviews * bands(lo) >= 2LL * nsm) {
        // hi rows only when that saves more than ~6 % of the waves: lo = 16 rows (4 compute
        // warps per SM sub-partition) runs ~5 % more rows per second than 17 (64 quads: 42
        // waves of 16 rows 43.67 ms vs 40 waves of 17 rows 43.89; 8 quads: 6 waves of 16 rows
        // 6.21 ms vs 5 waves of 17 rows 5.99)
        nb = 100 * waves(bands(hi)) < 94 * waves(bands(lo)) ? bands(hi) : bands(lo);
    } else {
        nb = bands(lo);
        double best = -1.0;
        for (int rows = lo; rows >= sgm::kBandRowsMin; --rows) {
            const int n = bands(rows), bq = H / n, br = H % n;
            auto t = [](int h) { return h / 16.0 * (1.0 + 0.012 * (16 - h)); };
            const double cost = double(waves(n)) * ((n - br) * t(bq) + br * t(bq + 1)) / n;
            if (best < 0 || cost < best - 1e-9) { best = cost; nb = n; }
        }
    }
    *nbands = nb;
    *q = H / nb;
    *r = H % nb;
}

// Views per ticket group of the sweeps (SweepParams::vgroup).  SGM_VIEW_GROUP
// (environment, experiments) forces it.
int view_group(int nviews, int nbands, int nsm) {
    static const int forced = [] {
        const char *e = getenv("SGM_VIEW_GROUP");
        return e ? atoi(e) : 0;
    }();
    (void)nbands; (void)nsm;
    int g = forced > 0 ? forced : nviews;
    return g < nviews ? g : nviews;
}

sgm::SweepParams sweep_params(const sgm_handle *h, int nviews, int *sync = nullptr) {
    sgm::SweepParams p{};
    const long long v0 = 0;
    p.W = h->prm.width; p.H = h->prm.height; p.D = h->prm.num_disp; p.Dp = h->dp;
    p.P1 = h->prm.p1; p.P2 = h->prm.p2; p.cmax = h->cmax;
    p.k_p1x2 = uint32_t(p.P1) * 0x10001u;
    p.k_negp1x2 = (uint32_t(0x10000 - p.P1) & 0xFFFFu) * 0x10001u;
    p.k_p2mp1x2 = uint32_t(p.P2 - p.P1) * 0x10001u;
    p.k_twop1x2 = 2u * p.k_p1x2;
    p.k_negb4 = 0u - 4u * p.k_p1x2;
    p.nviews = nviews;
    band_geometry(p.H, nviews, h->nsm, &p.nbands, &p.band_q, &p.band_r);
    p.vgroup = view_group(nviews, p.nbands, h->nsm);
    p.fine_sync = (long long)nviews * p.nbands < 2LL * h->nsm * sgm::kSweepCtasPerSm ? 1 : 0;
    if (const char *e = getenv("SGM_FINE_SYNC")) p.fine_sync = atoi(e);   // experiments
    p.cen = h->census + v0 * h->npx; p.cen_img_stride = h->npx;
    p.explicit_mode = 0;
    p.sfwd = h->sfwd + v0 * h->npx * h->dp; p.sfwd_view_stride = h->npx * h->dp;
    p.dint = h->dint + v0 * h->npx; p.dsub = h->dsub + v0 * h->npx; p.disp_view_stride = h->npx;
    p.sout = nullptr;
    p.gbuf = h->gbuf + v0 * p.nbands * (long long)h->prm.width * 3 * h->dp;
    if (!sync) sync = h->sync;
    p.progress = sync + 1; p.ticket = sync;
    p.trace = h->trace;
    p.debug_flags = h->debug_flags;
    p.one = 1;
    p.err = h->err_dev;
    return p;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Both sweeps of a call (sweep.cu).
cudaError_t run_sweeps(const sgm::SweepParams &p, int cpl, bool c64, int nw, bool debug_s, cudaStream_t st,
                       cudaEvent_t mid_a, cudaEvent_t mid_b, int *launches) {
    return sgm::launch_sweeps(p, cpl, c64, nw, debug_s, st, mid_a, mid_b, launches);
}

}  // namespace

extern "C" {

const char *sgm_status_string(sgm_status s) {
    switch (s) {
        case SGM_OK: return "ok";
        case SGM_ERR_INVALID_ARGUMENT: return "invalid argument";
        case SGM_ERR_UNSUPPORTED: return "unsupported";
        case SGM_ERR_CUDA: return "CUDA error";
        case SGM_ERR_OUT_OF_MEMORY: return "out of device memory";
    }
    return "unknown status";
}

const char *sgm_last_error_string(void) { return g_last_error; }

const char *sgm_stage_name(int32_t stage) {
    static const char *names[SGM_NUM_STAGES] = {"census", "sweep_fwd", "sweep_bwd_wta", "lr_check",
                                                "combine"};
    return (stage >= 0 && stage < SGM_NUM_STAGES) ? names[stage] : "?";
}

sgm_status sgm_create(const sgm_params *p, int32_t device, sgm_handle **out) {
    if (!p || !out) return SGM_ERR_INVALID_ARGUMENT;
    const int W = p->width, H = p->height, D = p->num_disp;
    const int cw = p->census_w, ch = p->census_h;
    if (W < 1 || H < 1 || D < 1 || D > 256) return SGM_ERR_INVALID_ARGUMENT;
    if (cw < 1 || ch < 1 || (cw % 2) == 0 || (ch % 2) == 0 || cw * ch - 1 > 63 || cw * ch < 2)
        return SGM_ERR_INVALID_ARGUMENT;
    if (cw > 17 || ch > 17) return SGM_ERR_UNSUPPORTED;      // TMA box halo limits
    if (p->p1 < 0 || p->p2 < p->p1 || (cw * ch - 1) + p->p2 > 255) return SGM_ERR_INVALID_ARGUMENT;
    if (p->lr_threshold < 0 || (p->bilinear_rule != 0 && p->bilinear_rule != 1) || p->max_batch < 1)
        return SGM_ERR_INVALID_ARGUMENT;
    if ((long long)W * H * 4LL * p->max_batch > (1LL << 40)) return SGM_ERR_INVALID_ARGUMENT;
    // launch-geometry limits of the per-pixel kernels (grid y = H, grid z = pairs / quads):
    // checked here so that no later call can fail half-way through its launch sequence
    if (H > 65535 || (long long)W * H >= (1LL << 31)) return SGM_ERR_UNSUPPORTED;
    if (2LL * p->max_batch > 65535) return SGM_ERR_UNSUPPORTED;

    sgm_handle *h = new (std::nothrow) sgm_handle();
    if (!h) return SGM_ERR_OUT_OF_MEMORY;
    h->prm = *p;
    h->device = device;
    h->cmax = cw * ch - 1;
    h->c64 = h->cmax > 32;
    h->cpl = 2 * ((D + 63) / 64);
    h->dp = 32 * h->cpl;
    h->nw = sgm::sweep_warps_for(h->cpl);
    h->nbands = (H + sgm::kBandRowsMin - 1) / sgm::kBandRowsMin;
    h->npx = (long long)W * H;
    h->max_views = 4 * p->max_batch;
    if (const char *dbg = getenv("SGM_DEBUG_FLAGS")) h->debug_flags = atoi(dbg);

    sgm::DeviceGuard guard(device);
    cudaError_t e = guard.status;
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, device);
    const size_t nv = size_t(h->max_views), npx = size_t(h->npx);
    h->stage_pitch = ((long long)W + 15) / 16 * 16;
    if (e == cudaSuccess) e = dalloc(&h->census, nv * npx);
    // the backward sweep prefetches S_fwd a few positions ahead without clamping: the
    // first row's prefetch reads into the front guard
    constexpr size_t kSfwdGuard = 64;   // (covers the optional L2 prefetch distance too)
    if (e == cudaSuccess) e = dalloc(&h->sfwd_alloc, (nv * npx + kSfwdGuard) * size_t(h->dp));
    if (e == cudaSuccess) h->sfwd = h->sfwd_alloc + kSfwdGuard * size_t(h->dp);
    if (e == cudaSuccess) e = dalloc(&h->dint, nv * npx);
    if (e == cudaSuccess) e = dalloc(&h->dsub, nv * npx);
    if (e == cudaSuccess) e = dalloc(&h->lr_int, nv / 2 * npx);
    if (e == cudaSuccess) e = dalloc(&h->lr_sub, nv / 2 * npx);
    if (e == cudaSuccess) e = dalloc(&h->lr_valid, nv / 2 * npx);
    // band handoff rows: one half per sweep (the two sweeps of a call overlap)
    if (e == cudaSuccess) e = dalloc(&h->gbuf, 2 * nv * size_t(h->nbands) * size_t(W) * 3 * size_t(h->dp));
    const size_t nsync = sgm::sweep_sync_ints(int(nv), h->nbands);
    if (e == cudaSuccess) e = dalloc(&h->sync, nsync);
    if (e == cudaSuccess) e = dalloc(&h->sync_host, nsync);
    const size_t eval_rows = size_t(sgm::evaluate_max_blocks()) + size_t(p->max_batch);
    if (e == cudaSuccess) e = dalloc(&h->eval_part, eval_rows * 12 + 1);
    if (e == cudaSuccess) e = cudaMemset(h->eval_part + eval_rows * 12, 0, sizeof(unsigned));
    const size_t mb = size_t(p->max_batch);
    for (auto &st : h->stage) {
        if (e == cudaSuccess) e = dalloc(&st.img_dense, nv * size_t(H) * size_t(W));
        if (e == cudaSuccess) e = dalloc(&st.img, nv * size_t(H) * size_t(h->stage_pitch));
        if (e == cudaSuccess) e = dalloc(&st.flow, mb * npx * 2);
        if (e == cudaSuccess) e = dalloc(&st.fvalid, mb * npx);
        if (e == cudaSuccess) e = dalloc(&st.sf, mb * npx * 4);
        if (e == cudaSuccess) e = dalloc(&st.p0, mb * npx * 4);
        if (e == cudaSuccess) e = dalloc(&st.dp, mb * npx * 4);
        if (e == cudaSuccess) e = dalloc(&st.vsf, mb * npx);
        if (e == cudaSuccess) e = dalloc(&st.v3, mb * npx);
        if (e == cudaSuccess) e = dalloc(&st.di, mb * npx * 2);
        if (e == cudaSuccess) e = dalloc(&st.ds, mb * npx * 2);
        if (e == cudaSuccess) e = dalloc(&st.dv, mb * npx * 2);
        for (cudaEvent_t *ev : {&st.ev_in, &st.ev_comp, &st.ev_out})
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    }
    for (cudaStream_t *sp : {&h->s_in, &h->s_comp, &h->s_out})
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(sp, cudaStreamNonBlocking);
    for (int i = 0; i <= SGM_NUM_STAGES && e == cudaSuccess; ++i) e = cudaEventCreate(&h->ev[i]);
    if (e == cudaSuccess) e = cudaMemset(h->sync, 0, sizeof(int) * nsync);
    if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void **>(&h->err_host), 4 * sizeof(int),
                                            cudaHostAllocMapped);
    if (e == cudaSuccess) {
        memset(h->err_host, 0, 4 * sizeof(int));
        e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&h->err_dev), h->err_host, 0);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaGetLastError();
        free_all(h);
        delete h;
        return from_cuda(e);
    }
    *out = h;
    return SGM_OK;
}

void sgm_destroy(sgm_handle *h) {
    if (!h) return;
    sgm::DeviceGuard guard(h->device);
    cudaDeviceSynchronize();
    free_all(h);
    delete h;
}

sgm_status sgm_get_geometry(sgm_handle *h, int32_t *dp, int32_t *cells_per_lane,
                            int32_t *sweep_warps, int32_t *band_rows) {
    if (!h) return SGM_ERR_INVALID_ARGUMENT;
    if (dp) *dp = h->dp;
    if (cells_per_lane) *cells_per_lane = h->cpl;
    if (sweep_warps) *sweep_warps = h->nw;
    if (band_rows) {                // band height chosen for a full batch (4 * max_batch views)
        int nb, q, r;
        band_geometry(h->prm.height, h->max_views, h->nsm, &nb, &q, &r);
        *band_rows = q + (r > 0);
    }
    return SGM_OK;
}

int64_t sgm_launch_count(sgm_handle *h) { return h ? h->launches : 0; }

sgm_status sgm_debug_set_trace(sgm_handle *h, uint64_t *trace) {
    if (!h) return SGM_ERR_INVALID_ARGUMENT;
    h->trace = reinterpret_cast<unsigned long long *>(trace);
    return SGM_OK;
}

sgm_status sgm_debug_set_flags(sgm_handle *h, int32_t flags) {
    if (!h || flags < 0 || flags > 31) return SGM_ERR_INVALID_ARGUMENT;
    h->debug_flags = flags;
    return SGM_OK;
}

sgm_status sgm_get_device_error(sgm_handle *h, int32_t *code, int32_t clear) {
    if (!h) return SGM_ERR_INVALID_ARGUMENT;
    volatile int *w = reinterpret_cast<volatile int *>(h->err_host);
    if (code) *code = w ? *w : 0;
    if (clear && w) *w = 0;
    return SGM_OK;
}

sgm_status sgm_set_timing(sgm_handle *h, int32_t enable) {
    if (!h) return SGM_ERR_INVALID_ARGUMENT;
    h->timing = enable != 0;
    h->timed = false;
    return SGM_OK;
}

int32_t sgm_read_timing(sgm_handle *h, float *ms) {
    if (!h || !ms || !h->timed) return 0;
    sgm::DeviceGuard guard(h->device);
    for (int i = 0; i < SGM_NUM_STAGES; ++i) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, h->ev[i], h->ev[i + 1]) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        ms[i] = t;
    }
    return SGM_NUM_STAGES;
}

sgm_status sgm_census(sgm_handle *h, const uint8_t *img, int64_t pitch_bytes, uint64_t *census,
                      void *stream) {
    if (!h || !img || !census || pitch_bytes < h->prm.width || (pitch_bytes % 16) != 0 ||
        !aligned16(img))
        return SGM_ERR_INVALID_ARGUMENT;
    SGM_ENTRY(h);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = sgm::launch_census_stack(img, (long long)h->prm.height * pitch_bytes, 1,
                                             pitch_bytes, h->prm.width, h->prm.height,
                                             h->prm.census_w, h->prm.census_h, census, h->npx, st);
    if (e == cudaSuccess) ++h->launches;
    return from_cuda(e);
}

sgm_status sgm_cost(sgm_handle *h, const uint64_t *cen_left, const uint64_t *cen_right,
                    int32_t view, uint8_t *cost, void *stream) {
    if (!h || !cen_left || !cen_right || !cost || (view != 0 && view != 1))
        return SGM_ERR_INVALID_ARGUMENT;
    SGM_ENTRY(h);
    const uint64_t *ref = view == 0 ? cen_left : cen_right;
    const uint64_t *match = view == 0 ? cen_right : cen_left;
    cudaError_t e = sgm::launch_cost(ref, match, h->prm.width, h->prm.height, h->prm.num_disp,
                                     view == 0 ? -1 : 1, h->cmax, cost,
                                     static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) ++h->launches;
    return from_cuda(e);
}

sgm_status sgm_aggregate(sgm_handle *h, const uint64_t *cen_left, const uint64_t *cen_right,
                         int32_t view, uint16_t *agg, void *stream) {
    if (!h || !cen_left || !cen_right || !agg || (view != 0 && view != 1))
        return SGM_ERR_INVALID_ARGUMENT;
    SGM_ENTRY(h);
    sgm::SweepParams p = sweep_params(h, 1);
    p.explicit_mode = 1;
    p.ref0 = view == 0 ? cen_left : cen_right;
    p.match0 = view == 0 ? cen_right : cen_left;
    p.mirror0 = view;
    p.dint = nullptr;
    p.dsub = nullptr;
    p.sout = agg;
    int n = 0;
    cudaError_t e = run_sweeps(p, h->cpl, h->c64, h->nw, true,
                                       static_cast<cudaStream_t>(stream), nullptr, nullptr, &n);
    h->launches += n;
    return from_cuda(e);
}

sgm_status sgm_wta(sgm_handle *h, const uint16_t *agg, int16_t *d_int, float *d_sub, void *stream) {
    if (!h || !agg || !d_int || !d_sub) return SGM_ERR_INVALID_ARGUMENT;
    SGM_ENTRY(h);
    cudaError_t e = sgm::launch_wta(agg, h->prm.width, h->prm.height, h->prm.num_disp, d_int, d_sub,
                                    static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) ++h->launches;
    return from_cuda(e);
}

sgm_status sgm_lr_check(sgm_handle *h, const int16_t *dl_int, const float *dl_sub,
                        const int16_t *dr_int, int16_t *out_int, float *out_sub, uint8_t *valid,
                        void *stream) {
    if (!h || !dl_int || !dl_sub || !dr_int || !out_int || !out_sub || !valid)
        return SGM_ERR_INVALID_ARGUMENT;
    SGM_ENTRY(h);
    sgm::LrParams p{};
    p.W = h->prm.width; p.H = h->prm.height; p.T = h->prm.lr_threshold;
    p.invalid = h->prm.invalid_disp; p.npairs = 1;
    p.dl = dl_int; p.dls = dl_sub; p.dr = dr_int;
    p.in_stride_l = p.in_stride_r = 0;
    p.out_int = out_int; p.out_sub = out_sub; p.valid = valid; p.out_stride = 0;
    cudaError_t e = sgm::launch_lr(p, static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) ++h->launches;
    return from_cuda(e);
}

sgm_status sgm_disparity(sgm_handle *h, const uint8_t *left, const uint8_t *right,
                         int64_t pitch_bytes, int16_t *out_int, float *out_sub, uint8_t *valid,
                         void *stream) {
    if (!h || !left || !right || !out_int || !out_sub || !valid) return SGM_ERR_INVALID_ARGUMENT;
    if (pitch_bytes < h->prm.width || (pitch_bytes % 16) != 0 || !aligned16(left) ||
        !aligned16(right))
        return SGM_ERR_INVALID_ARGUMENT;
    SGM_ENTRY(h);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int W = h->prm.width, H = h->prm.height;
    cudaError_t e = sgm::launch_census_stack(left, (long long)H * pitch_bytes, 1, pitch_bytes, W, H,
                                             h->prm.census_w, h->prm.census_h, h->census, h->npx, st);
    if (e == cudaSuccess) {
        ++h->launches;
        e = sgm::launch_census_stack(right, (long long)H * pitch_bytes, 1, pitch_bytes, W, H,
                                     h->prm.census_w, h->prm.census_h, h->census + h->npx, h->npx, st);
    }
    if (e == cudaSuccess) {
        ++h->launches;
        sgm::SweepParams p = sweep_params(h, 2);
        int n = 0;
        e = run_sweeps(p, h->cpl, h->c64, h->nw, false, st, nullptr, nullptr, &n);
        h->launches += n;
    }
    if (e == cudaSuccess) {
        sgm::LrParams p{};
        p.W = W; p.H = H; p.T = h->prm.lr_threshold; p.invalid = h->prm.invalid_disp; p.npairs = 1;
        p.dl = h->dint; p.dls = h->dsub; p.dr = h->dint + h->npx;
        p.out_int = out_int; p.out_sub = out_sub; p.valid = valid;
        e = sgm::launch_lr(p, st);
        if (e == cudaSuccess) ++h->launches;
    }
    return from_cuda(e);
}

sgm_status sgm_combine_sceneflow(sgm_handle *h, const float *d0, const uint8_t *v0, const float *d1,
                                 const uint8_t *v1, const float *flow, const uint8_t *flow_valid,
                                 const sgm_camera *cam, float *sf, float *p0, float *dp,
                                 uint8_t *valid_sf, uint8_t *valid_3d, void *stream) {
    if (!h || !d0 || !v0 || !d1 || !v1 || !flow || !sf || !valid_sf) return SGM_ERR_INVALID_ARGUMENT;
    const bool want3d = p0 || dp || valid_3d;
    if (want3d && (!dp || !valid_3d || !cam)) return SGM_ERR_INVALID_ARGUMENT;
    if (want3d && !(cam->f_px > 0.f && cam->baseline_m > 0.f)) return SGM_ERR_INVALID_ARGUMENT;
    if (!aligned16(sf) || (p0 && !aligned16(p0)) || (dp && !aligned16(dp)) ||
        (reinterpret_cast<uintptr_t>(flow) & 7))
        return SGM_ERR_INVALID_ARGUMENT;
    SGM_ENTRY(h);
    sgm::CombineParams p{};
    p.W = h->prm.width; p.H = h->prm.height; p.rule = h->prm.bilinear_rule; p.nquads = 1;
    p.d0 = d0; p.d1 = d1; p.v0 = v0; p.v1 = v1; p.disp_stride = 0;
    p.flow = flow; p.flow_valid = flow_valid;
    if (cam) {
        p.f = cam->f_px; p.B = cam->baseline_m; p.cx = cam->cx; p.cy = cam->cy;
        p.fB = cam->f_px * cam->baseline_m;
    }
    p.sf = sf; p.p0 = p0; p.dp = want3d ? dp : nullptr; p.valid_sf = valid_sf; p.valid_3d = valid_3d;
    cudaError_t e = sgm::launch_combine(p, static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) ++h->launches;
    return from_cuda(e);
}

sgm_status sgm_evaluate(sgm_handle *h, int32_t n, const float *sf, const uint8_t *valid_sf,
                        const float *gt_d0, const float *gt_d1, const float *gt_flow,
                        const uint8_t *gt_valid, const uint8_t *gt_noc, float tau_abs,
                        float tau_rel, uint64_t *counts, void *stream) {
    if (!h || !sf || !valid_sf || !gt_d0 || !gt_d1 || !gt_flow || !gt_noc || !counts)
        return SGM_ERR_INVALID_ARGUMENT;
    if (n < 1 || n > h->prm.max_batch) return SGM_ERR_INVALID_ARGUMENT;
    if (!(tau_abs >= 0.f) || !(tau_rel >= 0.f)) return SGM_ERR_INVALID_ARGUMENT;
    if (!aligned16(sf) || (reinterpret_cast<uintptr_t>(gt_flow) & 7) ||
        (reinterpret_cast<uintptr_t>(gt_d0) & 3) || (reinterpret_cast<uintptr_t>(gt_d1) & 3) ||
        (reinterpret_cast<uintptr_t>(counts) & 7))
        return SGM_ERR_INVALID_ARGUMENT;
    SGM_ENTRY(h);
    sgm::EvalParams p{};
    p.W = h->prm.width; p.H = h->prm.height; p.nquads = n;
    p.sf = sf; p.valid_sf = valid_sf; p.gt_d0 = gt_d0; p.gt_d1 = gt_d1; p.gt_flow = gt_flow;
    p.gt_valid = gt_valid; p.gt_noc = gt_noc; p.tau_abs = tau_abs; p.tau_rel = tau_rel;
    p.counts = reinterpret_cast<unsigned long long *>(counts);
    p.part = h->eval_part;
    p.ticket = h->eval_part + (size_t(sgm::evaluate_max_blocks()) + size_t(h->prm.max_batch)) * 12;
    cudaError_t e = sgm::launch_evaluate(p, static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) ++h->launches;
    return from_cuda(e);
}

sgm_status sgm_eval_rates(const uint64_t *counts, double *rates) {
    if (!counts || !rates) return SGM_ERR_INVALID_ARGUMENT;
    const double nan = std::numeric_limits<double>::quiet_NaN();
    for (int split = 0; split < 2; ++split) {
        const uint64_t *c = counts + 6 * split;
        double *r = rates + 5 * split;
        const uint64_t n_gt = c[0], n_ev = c[1];
        for (int k = 0; k < 4; ++k) r[k] = n_ev ? 100.0 * double(c[2 + k]) / double(n_ev) : nan;
        r[4] = n_gt ? 100.0 * double(n_ev) / double(n_gt) : nan;
    }
    return SGM_OK;
}

// 3D outputs need dp, valid_3d and a camera with f > 0, B > 0 (validated before any enqueue)
static bool camera_ok(const sgm_sceneflow_out *out, const sgm_camera *cam) {
    const bool want3d = out->p0 || out->dp || out->valid_3d;
    if (!want3d) return true;
    return out->dp && out->valid_3d && cam && cam->f_px > 0.f && cam->baseline_m > 0.f;
}

// The batched hot path.  Quad mode: images [n][4][H][pitch] = n independent quads, 2n
// stereo pairs, quad k combines pairs 2k and 2k+1.  Stream mode: images [n+1][2][H][pitch]
// = n+1 frames of one stereo video, n+1 pairs, quad k combines pairs k and k+1 (each
// frame's map computed once).  The disparity outputs are per pair.
static sgm_status scene_flow_impl(sgm_handle *h, int32_t n, bool stream, const uint8_t *images,
                                  int64_t pitch, const float *flow, const uint8_t *flow_valid,
                                  const sgm_camera *cam, const sgm_sceneflow_out *out,
                                  cudaStream_t st, int *sync = nullptr) {
    const int W = h->prm.width, H = h->prm.height;
    const long long npx = h->npx;
    const int npairs = stream ? n + 1 : 2 * n;
    const bool want3d = out->p0 || out->dp || out->valid_3d;
    if (want3d && (!out->dp || !out->valid_3d || !cam)) return SGM_ERR_INVALID_ARGUMENT;
    if (want3d && !(cam->f_px > 0.f && cam->baseline_m > 0.f)) return SGM_ERR_INVALID_ARGUMENT;
    const bool timing = h->timing;
    auto mark = [&](int i) {
        if (timing) cudaEventRecord(h->ev[i], st);
    };
    mark(0);
    cudaError_t e = sgm::launch_census_stack(images, (long long)H * pitch, 2 * npairs, pitch, W, H,
                                             h->prm.census_w, h->prm.census_h, h->census, npx, st);
    if (e != cudaSuccess) return from_cuda(e);
    ++h->launches;
    mark(1);
    {
        sgm::SweepParams p = sweep_params(h, 2 * npairs, sync);
        int nl = 0;
        e = run_sweeps(p, h->cpl, h->c64, h->nw, false, st, timing ? h->ev[2] : nullptr,
                               nullptr, &nl);
        h->launches += nl;
        if (e != cudaSuccess) return from_cuda(e);
    }
    mark(3);
    int16_t *di = out->disp_int ? out->disp_int : h->lr_int;
    float *ds = out->disp_sub ? out->disp_sub : h->lr_sub;
    uint8_t *dv = out->disp_valid ? out->disp_valid : h->lr_valid;
    // No disparity map asked for: the LR check is fused into the combination kernel (the
    // LR-checked maps are never materialised, one launch less).  SGM_DEBUG_FLAGS & 64 keeps
    // the separate LR kernel (A/B, parity of the two forms).
    const bool fuse_lr = !out->disp_int && !out->disp_sub && !out->disp_valid && !(h->debug_flags & 64);
    if (!fuse_lr) {
        sgm::LrParams p{};
        p.W = W; p.H = H; p.T = h->prm.lr_threshold; p.invalid = h->prm.invalid_disp;
        p.npairs = npairs;
        p.dl = h->dint; p.dls = h->dsub; p.dr = h->dint + npx;
        p.in_stride_l = p.in_stride_r = 2 * npx;
        p.out_int = di; p.out_sub = ds; p.valid = dv; p.out_stride = npx;
        e = sgm::launch_lr(p, st);
        if (e != cudaSuccess) return from_cuda(e);
        ++h->launches;
    }
    mark(4);
    {
        sgm::CombineParams p{};
        p.W = W; p.H = H; p.rule = h->prm.bilinear_rule; p.nquads = n;
        p.d0 = ds; p.d1 = ds + npx; p.v0 = dv; p.v1 = dv + npx;
        p.disp_stride = stream ? npx : 2 * npx;
        p.flow = flow; p.flow_valid = flow_valid;
        if (cam) {
            p.f = cam->f_px; p.B = cam->baseline_m; p.cx = cam->cx; p.cy = cam->cy;
            p.fB = cam->f_px * cam->baseline_m;
        }
        p.sf = out->sf; p.valid_sf = out->valid_sf;
        p.p0 = out->p0; p.dp = want3d ? out->dp : nullptr; p.valid_3d = out->valid_3d;
        if (fuse_lr) {
            p.raw_int = h->dint; p.raw_sub = h->dsub; p.view_stride = npx;
            p.pair_step = stream ? 1 : 2; p.T = h->prm.lr_threshold;
            p.invalid = float(h->prm.invalid_disp);
        }
        e = sgm::launch_combine(p, st);
        if (e != cudaSuccess) return from_cuda(e);
        ++h->launches;
    }
    mark(5);
    if (timing) h->timed = true;
    return SGM_OK;
}

// Both modes take 1..max_batch quads (stream mode: n+1 <= 2 max_batch pairs fit the
// 4 max_batch views of scratch).
static bool batch_ok(const sgm_handle *h, int32_t n, bool) { return n >= 1 && n <= h->prm.max_batch; }

static sgm_status scene_flow_dev(sgm_handle *h, int32_t n, bool stream, const uint8_t *images,
                                 int64_t pitch_bytes, const float *flow, const uint8_t *flow_valid,
                                 const sgm_camera *cam, const sgm_sceneflow_out *out, void *stream_) {
    if (!h || !images || !flow || !out || !out->sf || !out->valid_sf) return SGM_ERR_INVALID_ARGUMENT;
    if (!batch_ok(h, n, stream)) return SGM_ERR_INVALID_ARGUMENT;
    if (pitch_bytes < h->prm.width || (pitch_bytes % 16) != 0 || !aligned16(images) ||
        !aligned16(out->sf) || (out->p0 && !aligned16(out->p0)) || (out->dp && !aligned16(out->dp)) ||
        (reinterpret_cast<uintptr_t>(flow) & 7))
        return SGM_ERR_INVALID_ARGUMENT;
    if (!camera_ok(out, cam)) return SGM_ERR_INVALID_ARGUMENT;
    SGM_ENTRY(h);
    return scene_flow_impl(h, n, stream, images, pitch_bytes, flow, flow_valid, cam, out,
                           static_cast<cudaStream_t>(stream_));
}

sgm_status sgm_scene_flow(sgm_handle *h, int32_t n, const uint8_t *images, int64_t pitch_bytes,
                          const float *flow, const uint8_t *flow_valid, const sgm_camera *cam,
                          const sgm_sceneflow_out *out, void *stream) {
    return scene_flow_dev(h, n, false, images, pitch_bytes, flow, flow_valid, cam, out, stream);
}

sgm_status sgm_scene_flow_stream(sgm_handle *h, int32_t n, const uint8_t *images, int64_t pitch_bytes,
                                 const float *flow, const uint8_t *flow_valid, const sgm_camera *cam,
                                 const sgm_sceneflow_out *out, void *stream) {
    return scene_flow_dev(h, n, true, images, pitch_bytes, flow, flow_valid, cam, out, stream);
}

static sgm_status scene_flow_host_impl(sgm_handle *h, int32_t n, bool stream_mode,
                                       const uint8_t *images, const float *flow,
                                       const uint8_t *flow_valid, const sgm_camera *cam,
                                       const sgm_sceneflow_out *out, void *stream) {
    if (!h || !images || !flow || !out || !out->sf || !out->valid_sf) return SGM_ERR_INVALID_ARGUMENT;
    if (!batch_ok(h, n, stream_mode)) return SGM_ERR_INVALID_ARGUMENT;
    const long long nimg = stream_mode ? 2LL * (n + 1) : 4LL * n;   // images in the batch
    const long long nmaps = nimg / 2;                                // LR-checked maps
    const bool want3d = out->p0 || out->dp || out->valid_3d;
    if (!camera_ok(out, cam)) return SGM_ERR_INVALID_ARGUMENT;
    SGM_ENTRY(h);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int W = h->prm.width, H = h->prm.height;
    const long long npx = h->npx;
    // Three internal streams and two staging slots.  Call k uses slot k % 2:
    //   copy-in  : wait until call k-2's kernels stopped reading the slot; 1D copies in
    //   compute  : wait for the copy-in and for call k-2's copy-out of the slot; re-pitch,
    //              census, sweeps, LR, combination (one launch set for the whole batch)
    //   copy-out : wait for the compute; copy the requested results to the host
    // and `stream` waits for the copy-out.  Calls issued back to back therefore overlap
    // the upload of k+1 and the download of k-1 with the kernels of k.
    sgm_handle::Stage &sg = h->stage[h->slot];
    h->slot ^= 1;
    const bool timing = h->timing;
    h->timing = false;
    cudaError_t e = cudaSuccess;
    if (sg.used) e = cudaStreamWaitEvent(h->s_in, sg.ev_comp, 0);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(sg.img_dense, images, size_t(nimg * H * W), cudaMemcpyHostToDevice, h->s_in);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(sg.flow, flow, sizeof(float) * 2 * npx * n, cudaMemcpyHostToDevice, h->s_in);
    if (e == cudaSuccess && flow_valid)
        e = cudaMemcpyAsync(sg.fvalid, flow_valid, size_t(npx) * n, cudaMemcpyHostToDevice, h->s_in);
    if (e == cudaSuccess) e = cudaEventRecord(sg.ev_in, h->s_in);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->s_comp, sg.ev_in, 0);
    if (e == cudaSuccess && sg.used) e = cudaStreamWaitEvent(h->s_comp, sg.ev_out, 0);
    if (e == cudaSuccess) e = sgm::launch_repitch(sg.img_dense, sg.img, W, h->stage_pitch, nimg * H, h->s_comp);
    if (e != cudaSuccess) { h->timing = timing; return from_cuda(e); }
    ++h->launches;
    sgm_sceneflow_out dev{};
    dev.sf = sg.sf;
    dev.valid_sf = sg.vsf;
    if (want3d) { dev.p0 = out->p0 ? sg.p0 : nullptr; dev.dp = sg.dp; dev.valid_3d = sg.v3; }
    // (no disparity map requested: none is staged, and the LR check runs fused in the
    // combination kernel)
    if (out->disp_int || out->disp_sub || out->disp_valid) {
        dev.disp_int = sg.di; dev.disp_sub = sg.ds; dev.disp_valid = sg.dv;
    }
    sgm_status s = scene_flow_impl(h, n, stream_mode, sg.img, h->stage_pitch, sg.flow,
                                   flow_valid ? sg.fvalid : nullptr, cam, &dev, h->s_comp,
                                   h->sync_host);
    h->timing = timing;
    if (s != SGM_OK) return s;
    sg.used = true;
    e = cudaEventRecord(sg.ev_comp, h->s_comp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->s_out, sg.ev_comp, 0);
    auto d2h = [&](void *dst, const void *src, size_t bytes) {
        if (dst && e == cudaSuccess) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->s_out);
    };
    d2h(out->sf, sg.sf, sizeof(float) * 4 * npx * n);
    d2h(out->valid_sf, sg.vsf, size_t(npx) * n);
    if (want3d) {
        d2h(out->p0, sg.p0, sizeof(float) * 4 * npx * n);
        d2h(out->dp, sg.dp, sizeof(float) * 4 * npx * n);
        d2h(out->valid_3d, sg.v3, size_t(npx) * n);
    }
    d2h(out->disp_int, sg.di, sizeof(int16_t) * npx * nmaps);
    d2h(out->disp_sub, sg.ds, sizeof(float) * npx * nmaps);
    d2h(out->disp_valid, sg.dv, size_t(npx) * nmaps);
    if (e == cudaSuccess) e = cudaEventRecord(sg.ev_out, h->s_out);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, sg.ev_out, 0);
    return from_cuda(e);
}

sgm_status sgm_scene_flow_host(sgm_handle *h, int32_t n, const uint8_t *images, const float *flow,
                               const uint8_t *flow_valid, const sgm_camera *cam,
                               const sgm_sceneflow_out *out, void *stream) {
    return scene_flow_host_impl(h, n, false, images, flow, flow_valid, cam, out, stream);
}

sgm_status sgm_scene_flow_stream_host(sgm_handle *h, int32_t n, const uint8_t *images,
                                      const float *flow, const uint8_t *flow_valid,
                                      const sgm_camera *cam, const sgm_sceneflow_out *out,
                                      void *stream) {
    return scene_flow_host_impl(h, n, true, images, flow, flow_valid, cam, out, stream);
}

}  // extern "C"
