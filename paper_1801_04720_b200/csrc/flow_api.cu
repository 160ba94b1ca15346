// flow_api.cu -- C ABI of the optical-flow core (include/sgmflow.h): handle, scratch,
// the batched field / flow pipelines and the stage-wise entry points used for parity.
#include <cstdio>
#include <cstring>

#include "../../include/sgmflow.h"
#include "sgm_internal.cuh"

struct sgm_flow_handle {
    sgm_flow_params prm{};
    int device = 0;
    int lw[8] = {}, lh[8] = {};      // level sizes
    long long lper[8] = {};          // pixels per level image
    long long pyr_off[8] = {};       // offset of level l in a pyramid buffer (per image)
    long long pyr_img = 0;           // bytes of one image's pyramid
    uint8_t *pyr = nullptr;          // [max_batch][2][pyr_img]: level images of A_k, B_k
    uint32_t *quad = nullptr;        // [max_batch][2][pyr_img]: their quad images (same offsets)
    int32_t *desc = nullptr;         // [2 max_batch][Wc Hc][16]
    int32_t *nn = nullptr;           // [2 max_batch][Wc Hc][knn]
    void *knn_scratch = nullptr;     // packed descriptors for the tensor-core kNN
    int32_t *flow[2] = {nullptr, nullptr};   // ping-pong [3 max_batch][W H][2]
    int32_t *cost[2] = {nullptr, nullptr};   // [3 max_batch][W H]
    int *sync = nullptr;             // ticket + band progress of the propagation kernel
    long long launches = 0;
    // instrumentation: event pairs around every launch of a category (prop, search, knn,
    // other) of the last timed sgm_flow / sgm_flow_field call
    bool timing = false;
    static constexpr int kMaxEv = 256;
    cudaEvent_t ev[kMaxEv] = {};
    int ev_cat[kMaxEv / 2] = {};
    int nev = 0;
};

namespace {

thread_local char g_ff_error[256] = "no error";

sgm_status ff_status(cudaError_t e) {
    if (e == cudaSuccess) return SGM_OK;
    snprintf(g_ff_error, sizeof(g_ff_error), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    if (e == cudaErrorMemoryAllocation) return SGM_ERR_OUT_OF_MEMORY;
    return SGM_ERR_CUDA;
}

// Entry-point prologue: the handle's device is current for the call (restored on return).
#define FF_ENTRY(dev)                        \
    sgm::DeviceGuard guard_(dev);            \
    if (guard_.status != cudaSuccess) return ff_status(guard_.status);

template <class T>
cudaError_t ff_alloc(T **p, size_t count) {
    return cudaMalloc(reinterpret_cast<void **>(p), count * sizeof(T) + 256);
}

void ff_free(sgm_flow_handle *h) {
    void *ptrs[] = {h->knn_scratch, h->pyr, h->quad, h->desc, h->nn, h->flow[0], h->flow[1], h->cost[0], h->cost[1], h->sync};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    for (auto &e : h->ev)
        if (e) cudaEventDestroy(e);
}

// timing helpers: mark(cat) before a launch, done() after it
struct Timer : sgm::FFTimer {
    sgm_flow_handle *h;
    cudaStream_t st;
    Timer(sgm_flow_handle *h_, cudaStream_t st_) : h(h_), st(st_) {}
    void begin(int cat) override {
        if (!h->timing || h->nev + 2 > sgm_flow_handle::kMaxEv) return;
        h->ev_cat[h->nev / 2] = cat;
        cudaEventRecord(h->ev[h->nev], st);
    }
    void end() override {
        if (!h->timing || h->nev + 2 > sgm_flow_handle::kMaxEv) return;
        cudaEventRecord(h->ev[h->nev + 1], st);
        h->nev += 2;
    }
};

bool params_ok(const sgm_flow_params *p) {
    if (!p) return false;
    // the row handoff packs vectors into 20-bit fields (+-65536 px in 1/8 px)
    if (p->width < 1 || p->height < 1 || p->width > 16384 || p->height > 16384) return false;
    if (p->levels < 1 || p->levels > 8) return false;
    if (p->patch_radius < 0 || p->patch_radius + 2 > 7) return false;    // r+2 <= 7 (256 samples)
    if (p->sweeps < 0 || p->sweeps > 64 || p->search_radius < 1) return false;
    if (p->desc_window != 4 && p->desc_window != 8 && p->desc_window != 16) return false;
    if (p->knn < 1 || p->knn > 8 || p->consistency_q < 0 || p->penalty < 0 || p->penalty > 255) return false;
    if (p->max_batch < 1) return false;
    return true;
}

// One batch of fields through the whole pyramid.  fpp = 1: fields A_k -> B_k with
// (seed, radius); fpp = 3: forward + two inverse fields (F-5).  The level-0 images of the
// batch must already be in the pyramid buffer.  Result: level-0 fields in h->flow[res],
// h->cost[res].
cudaError_t run_fields(sgm_flow_handle *h, int n, int fpp, uint64_t seed, int radius, cudaStream_t st,
                       int *res) {
    const sgm_flow_params &P = h->prm;
    const int L = P.levels;
    cudaError_t e = cudaSuccess;
    Timer T(h, st);
    if (h->timing) h->nev = 0;
    // pyramid of the 2n images (A_k, B_k interleaved, one pyramid per image)
    for (int l = 1; l < L && e == cudaSuccess; ++l) {
        e = sgm::ff_launch_downsample(h->pyr + h->pyr_off[l - 1], h->pyr_img, h->lw[l - 1], h->lh[l - 1],
                                      h->pyr + h->pyr_off[l], h->pyr_img, 2 * n, st);
        if (e == cudaSuccess) ++h->launches;
    }
    // quad images of every level (the data term reads them)
    for (int l = 0; l < L && e == cudaSuccess; ++l) {
        e = sgm::ff_launch_quad(h->pyr + h->pyr_off[l], h->pyr_img, h->lw[l], h->lh[l], 2 * n,
                                h->quad + h->pyr_off[l], h->pyr_img, st);
        if (e == cudaSuccess) ++h->launches;
    }
    if (e != cudaSuccess) return e;
    const int c = L - 1;
    // descriptors + kNN at the coarsest level
    e = sgm::ff_launch_wht(h->pyr + h->pyr_off[c], h->pyr_img, h->lw[c], h->lh[c], P.desc_window, 2 * n,
                           h->desc, st);
    if (e != cudaSuccess) return e;
    ++h->launches;
    T.begin(2);
    e = sgm::ff_launch_knn(h->desc, int(h->lper[c]), 2 * n, P.knn, P.desc_window, h->nn, h->knn_scratch, st);
    T.end();
    if (e != cudaSuccess) return e;
    ++h->launches;
    sgm::FFFields F{};
    F.fpp = fpp;
    F.nfields = fpp * n;
    F.img_stride = 2 * h->pyr_img;
    F.radius[0] = radius; F.radius[1] = radius; F.radius[2] = radius + 2;
    F.seed[0] = seed; F.seed[1] = seed + 1; F.seed[2] = seed + 2;
    F.penalty = P.penalty;
    int cur = 0;
    for (int l = c; l >= 0 && e == cudaSuccess; --l) {
        F.W = h->lw[l]; F.H = h->lh[l];
        F.A = h->pyr + h->pyr_off[l];
        F.B = F.A + h->pyr_img;
        F.QA = h->quad + h->pyr_off[l];
        F.QB = F.QA + h->pyr_img;
        F.flow = h->flow[cur]; F.cost = h->cost[cur];
        if (l == c) {
            e = sgm::ff_launch_init(F, h->nn, P.knn, st);
        } else {
            e = sgm::ff_launch_lift(F, h->flow[cur ^ 1], h->lw[l + 1], h->lh[l + 1], st);
        }
        if (e == cudaSuccess) ++h->launches;
        for (int s = 0; s < P.sweeps && e == cudaSuccess; ++s) {
            int nl = 0;
            e = sgm::ff_launch_sweep(F, s, l, P.search_radius, h->sync, st, &nl,
                                     h->timing ? &T : nullptr);
            h->launches += nl;
        }
        cur ^= 1;
    }
    *res = cur ^ 1;
    return e;
}

cudaError_t upload_pairs(sgm_flow_handle *h, int n, const uint8_t *A, const uint8_t *B, cudaStream_t st,
                         cudaMemcpyKind kind) {
    const size_t img = size_t(h->lper[0]);
    cudaError_t e = cudaMemcpy2DAsync(h->pyr, size_t(2 * h->pyr_img), A, img, img, size_t(n), kind, st);
    if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(h->pyr + h->pyr_img, size_t(2 * h->pyr_img), B, img, img, size_t(n), kind, st);
    return e;
}

}  // namespace

extern "C" {

const char *sgm_flow_last_error_string(void) { return g_ff_error; }

sgm_status sgm_flow_create(const sgm_flow_params *p, int32_t device, sgm_flow_handle **out) {
    if (!out || !params_ok(p)) return SGM_ERR_INVALID_ARGUMENT;
    sgm_flow_handle *h = new sgm_flow_handle;
    h->prm = *p;
    h->device = device;
    sgm::DeviceGuard guard(device);
    cudaError_t e = guard.status;
    int W = p->width, H = p->height;
    long long off = 0;
    for (int l = 0; l < p->levels; ++l) {
        h->lw[l] = W; h->lh[l] = H;
        h->lper[l] = (long long)W * H;
        h->pyr_off[l] = off;
        off += (h->lper[l] + 15) / 16 * 16;
        W = (W + 1) / 2; H = (H + 1) / 2;
    }
    h->pyr_img = off;
    const size_t mb = size_t(p->max_batch);
    const size_t n0 = size_t(h->lper[0]), nc = size_t(h->lper[p->levels - 1]);
    if (e == cudaSuccess) e = ff_alloc(&h->pyr, mb * 2 * size_t(h->pyr_img));
    if (e == cudaSuccess) e = ff_alloc(&h->quad, mb * 2 * size_t(h->pyr_img));
    // descriptors / neighbour lists: the batch at the coarsest level, or one pair at level 0
    // (the stage-wise sgm_flow_knn_init)
    const size_t nd = 2 * mb * nc > 2 * n0 ? 2 * mb * nc : 2 * n0;
    if (e == cudaSuccess) e = ff_alloc(&h->desc, nd * 16);
    if (e == cudaSuccess) e = ff_alloc(&h->nn, nd * size_t(p->knn));
    if (e == cudaSuccess) e = cudaMalloc(&h->knn_scratch, sgm::ff_knn_scratch_bytes((long long)nd));
    for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
        e = ff_alloc(&h->flow[k], 3 * mb * n0 * 2);
        if (e == cudaSuccess) e = ff_alloc(&h->cost[k], 3 * mb * n0);
    }
    if (e == cudaSuccess) e = ff_alloc(&h->sync, size_t(sgm::ff_sync_ints(3 * p->max_batch, p->width, p->height)));
    for (auto &ev : h->ev)
        if (e == cudaSuccess) e = cudaEventCreate(&ev);
    if (e != cudaSuccess) {
        sgm_status s = ff_status(e);
        ff_free(h);
        delete h;
        cudaGetLastError();
        return s;
    }
    *out = h;
    return SGM_OK;
}

void sgm_flow_destroy(sgm_flow_handle *h) {
    if (!h) return;
    sgm::DeviceGuard guard(h->device);
    cudaDeviceSynchronize();
    ff_free(h);
    delete h;
}

int64_t sgm_flow_launch_count(sgm_flow_handle *h) { return h ? h->launches : 0; }

sgm_status sgm_flow_set_timing(sgm_flow_handle *h, int32_t enable) {
    if (!h) return SGM_ERR_INVALID_ARGUMENT;
    h->timing = enable != 0;
    h->nev = 0;
    return SGM_OK;
}

int32_t sgm_flow_read_timing(sgm_flow_handle *h, float *ms) {
    if (!h || !ms || h->nev == 0) return 0;
    sgm::DeviceGuard guard(h->device);
    for (int k = 0; k < SGM_FLOW_NUM_STAGES; ++k) ms[k] = 0.f;
    for (int i = 0; i < h->nev; i += 2) {
        float t = 0.f;
        if (cudaEventSynchronize(h->ev[i + 1]) != cudaSuccess ||
            cudaEventElapsedTime(&t, h->ev[i], h->ev[i + 1]) != cudaSuccess)
            return 0;
        ms[h->ev_cat[i / 2]] += t;
    }
    return SGM_FLOW_NUM_STAGES;
}

sgm_status sgm_flow_descriptors(sgm_flow_handle *h, const uint8_t *img, int32_t w, int32_t hgt,
                                int32_t *desc, void *stream) {
    if (!h || !img || !desc || w < 1 || hgt < 1) return SGM_ERR_INVALID_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(desc) & 15) != 0) return SGM_ERR_INVALID_ARGUMENT;
    FF_ENTRY(h->device);
    cudaError_t e = sgm::ff_launch_wht(img, 0, w, hgt, h->prm.desc_window, 1, desc,
                                       static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) ++h->launches;
    return ff_status(e);
}

sgm_status sgm_flow_patch_cost(sgm_flow_handle *h, const uint8_t *A, const uint8_t *B, int32_t w,
                               int32_t hgt, int32_t radius, int32_t nq, const int32_t *queries,
                               int32_t *out, void *stream) {
    if (!h || !A || !B || !queries || !out || w < 1 || hgt < 1 || nq < 0 || radius < 0 || radius > 7)
        return SGM_ERR_INVALID_ARGUMENT;
    if (nq == 0) return SGM_OK;
    if ((long long)w * hgt > h->lper[0]) return SGM_ERR_INVALID_ARGUMENT;
    FF_ENTRY(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = sgm::ff_launch_quad(B, 0, w, hgt, 1, h->quad, 0, st);
    if (e == cudaSuccess)
        e = sgm::ff_launch_cost_query(A, h->quad, w, hgt, radius, h->prm.penalty, nq, queries, out, st);
    if (e == cudaSuccess) h->launches += 2;
    return ff_status(e);
}

sgm_status sgm_flow_knn_init(sgm_flow_handle *h, const uint8_t *A, const uint8_t *B, int32_t w,
                             int32_t hgt, int32_t radius, int32_t *flow_q, int32_t *cost,
                             int32_t *nn, void *stream) {
    if (!h || !A || !B || !flow_q || !cost || w < 1 || hgt < 1 || radius < 0 || radius > 7)
        return SGM_ERR_INVALID_ARGUMENT;
    const long long n = (long long)w * hgt;
    if (n > h->lper[0]) return SGM_ERR_INVALID_ARGUMENT;     // scratch sized for level 0
    FF_ENTRY(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // images into the scratch pyramid slot 0 as one "pair" (A, B), level-0 layout
    cudaError_t e = cudaMemcpyAsync(h->pyr, A, size_t(n), cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h->pyr + h->pyr_img, B, size_t(n), cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = sgm::ff_launch_quad(h->pyr, h->pyr_img, w, hgt, 2, h->quad, h->pyr_img, st);
    if (e == cudaSuccess) e = sgm::ff_launch_wht(h->pyr, h->pyr_img, w, hgt, h->prm.desc_window, 2, h->desc, st);
    if (e == cudaSuccess) e = sgm::ff_launch_knn(h->desc, int(n), 1, h->prm.knn, h->prm.desc_window, nn ? nn : h->nn, h->knn_scratch, st);
    sgm::FFFields F{};
    F.W = w; F.H = hgt; F.fpp = 1; F.nfields = 1;
    F.A = h->pyr; F.B = h->pyr + h->pyr_img; F.img_stride = 2 * h->pyr_img;
    F.QA = h->quad; F.QB = h->quad + h->pyr_img;
    F.radius[0] = radius; F.penalty = h->prm.penalty;
    F.flow = flow_q; F.cost = cost;
    if (e == cudaSuccess) e = sgm::ff_launch_init(F, nn ? nn : h->nn, h->prm.knn, st);
    if (e == cudaSuccess) h->launches += 4;
    return ff_status(e);
}

sgm_status sgm_flow_sweep(sgm_flow_handle *h, const uint8_t *A, const uint8_t *B, int32_t w, int32_t hgt,
                          int32_t radius, int32_t sweep, int32_t level, uint64_t seed, int32_t *flow_q,
                          int32_t *cost, void *stream) {
    if (!h || !A || !B || !flow_q || !cost || w < 1 || hgt < 1 || radius < 0 || radius > 7 || sweep < 0 ||
        level < 0)
        return SGM_ERR_INVALID_ARGUMENT;
    if (hgt > h->prm.height || w > h->prm.width) return SGM_ERR_INVALID_ARGUMENT;
    FF_ENTRY(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    sgm::FFFields F{};
    F.W = w; F.H = hgt; F.fpp = 1; F.nfields = 1;
    F.A = A; F.B = B; F.img_stride = 0;
    F.QA = h->quad; F.QB = h->quad + h->pyr_img;       // scratch slots of pair 0
    F.radius[0] = radius; F.seed[0] = seed; F.penalty = h->prm.penalty;
    F.flow = flow_q; F.cost = cost;
    cudaError_t e = sgm::ff_launch_quad(A, 0, w, hgt, 1, h->quad, 0, st);
    if (e == cudaSuccess) e = sgm::ff_launch_quad(B, 0, w, hgt, 1, h->quad + h->pyr_img, 0, st);
    int nl = 2;
    if (e == cudaSuccess) e = sgm::ff_launch_sweep(F, sweep, level, h->prm.search_radius, h->sync, st, &nl);
    h->launches += nl;
    return ff_status(e);
}

sgm_status sgm_flow_consistency(sgm_flow_handle *h, const int32_t *F, const int32_t *G1, const int32_t *G2,
                                int32_t w, int32_t hgt, uint8_t *valid, void *stream) {
    if (!h || !F || !G1 || !G2 || !valid || w < 1 || hgt < 1) return SGM_ERR_INVALID_ARGUMENT;
    FF_ENTRY(h->device);
    cudaError_t e = sgm::ff_launch_consistency(F, G1, G2, 0, 0, w, hgt, 1, h->prm.consistency_q, valid,
                                               nullptr, static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) ++h->launches;
    return ff_status(e);
}

sgm_status sgm_flow_field(sgm_flow_handle *h, int32_t n, const uint8_t *A, const uint8_t *B, uint64_t seed,
                          int32_t radius, int32_t *flow_q, int32_t *cost, void *stream) {
    if (!h || !A || !B || !flow_q || n < 1 || n > h->prm.max_batch || radius < 0 || radius + 2 > 7)
        return SGM_ERR_INVALID_ARGUMENT;
    FF_ENTRY(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = upload_pairs(h, n, A, B, st, cudaMemcpyDeviceToDevice);
    int res = 0;
    if (e == cudaSuccess) e = run_fields(h, n, 1, seed, radius, st, &res);
    const size_t n0 = size_t(h->lper[0]);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(flow_q, h->flow[res], sizeof(int32_t) * 2 * n0 * n, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && cost)
        e = cudaMemcpyAsync(cost, h->cost[res], sizeof(int32_t) * n0 * n, cudaMemcpyDeviceToDevice, st);
    return ff_status(e);
}

sgm_status sgm_flow(sgm_flow_handle *h, int32_t n, const uint8_t *frames0, const uint8_t *frames1,
                    float *flow, uint8_t *valid, int32_t *fields_q, void *stream) {
    if (!h || !frames0 || !frames1 || n < 1 || n > h->prm.max_batch || (!flow && !valid && !fields_q))
        return SGM_ERR_INVALID_ARGUMENT;
    if (flow && (reinterpret_cast<uintptr_t>(flow) & 7)) return SGM_ERR_INVALID_ARGUMENT;
    FF_ENTRY(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = upload_pairs(h, n, frames0, frames1, st, cudaMemcpyDeviceToDevice);
    int res = 0;
    if (e == cudaSuccess) e = run_fields(h, n, 3, h->prm.seed, h->prm.patch_radius, st, &res);
    const long long n0 = h->lper[0];
    const int32_t *fw = h->flow[res];
    if (e == cudaSuccess && (flow || valid)) {
        e = sgm::ff_launch_consistency(fw, fw + 2 * n0, fw + 4 * n0, 6 * n0, 6 * n0, h->prm.width,
                                       h->prm.height, n, h->prm.consistency_q, valid, flow, st);
        if (e == cudaSuccess) ++h->launches;
    }
    if (e == cudaSuccess && fields_q)
        e = cudaMemcpyAsync(fields_q, fw, sizeof(int32_t) * 6 * size_t(n0) * n, cudaMemcpyDeviceToDevice, st);
    return ff_status(e);
}

int64_t sgm_densify_scratch_bytes(int32_t n, int32_t width, int32_t height) {
    if (n < 1 || width < 1 || height < 1 || width > 16384 || height > 16384) return -1;
    return int64_t(sgm::densify_scratch_bytes(n, width, height));
}

sgm_status sgm_densify(int32_t n, int32_t width, int32_t height, int32_t channels, const float *field,
                       const uint8_t *valid, const uint8_t *guide, int32_t K, float lambda, int32_t window,
                       float *out, int32_t *unfilled, int32_t *certified, void *scratch, int64_t scratch_bytes,
                       void *stream) {
    if (n < 1 || width < 1 || height < 1 || width > 16384 || height > 16384 || channels < 1 || channels > 4 ||
        !field || !valid || !guide || !out || K < 1 || K > 64 || !(lambda >= 0.f))
        return SGM_ERR_INVALID_ARGUMENT;
    if ((long long)n * width * height >= (1LL << 31)) return SGM_ERR_INVALID_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(field) & 3) || (reinterpret_cast<uintptr_t>(out) & 3))
        return SGM_ERR_INVALID_ARGUMENT;
    if (scratch && ((reinterpret_cast<uintptr_t>(scratch) & 15) ||
                    scratch_bytes < int64_t(sgm::densify_scratch_bytes(n, width, height))))
        return SGM_ERR_INVALID_ARGUMENT;
    // handle-free: run on the device that owns `field`
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, field) != cudaSuccess || attr.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        return SGM_ERR_INVALID_ARGUMENT;
    }
    FF_ENTRY(attr.device);
    sgm::DensifyParams p{};
    p.n = n; p.W = width; p.H = height; p.C = channels; p.K = K; p.lambda = lambda; p.window = window;
    p.field = field; p.valid = valid; p.guide = guide; p.out = out; p.unfilled = unfilled;
    p.certified = certified;
    return ff_status(sgm::launch_densify(p, scratch, static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
