// knn_tc.cu -- exhaustive k-nearest-neighbour search of WHT descriptors on the 5th-generation
// tensor cores (row f2, the Flow Fields+ initialisation of P:86; SPEC F-1 / S:216-218,
// reading FF5: the exact k nearest by squared Euclidean distance, ties to the smaller
// database index -- the result of an exact k-d tree query).
//
// Exactness.  Each 16-coefficient descriptor c (|c| < 2^14, 8x8 WHT window) splits into two
// fp16 limbs c = 128 h + l, |h| <= 128, 0 <= l <= 127, both exact in fp16, so
//   q . b = 16384 sum(qh bh) + 128 sum(qh bl + ql bh) + sum(ql bl)
// where every product is < 2^14 and every 16- or 32-term sum < 2^24: the fp32 tensor-core
// accumulators hold the three sums exactly.  The epilogue screens each (query, entry)
// distance |q|^2 + |b|^2 - 2 q.b in fp32 against the query's admission bound plus a 2^15
// margin (fp32 error < 2^13) and forms the exact 64-bit distance only for survivors.
//
// Blackwell mapping (sm_100a): one CTA = 128 queries = the 128 TMEM lanes; per database
// tile of 64 entries one elected thread issues four tcgen05.mma.kind::f16 (M=128, N=64,
// K=16; A = query limbs, B = entry limbs, both K-major in shared memory, no swizzle) into
// three fp32 accumulators in TMEM (sum hh, sum hl + lh, sum ll: 192 columns), commits them
// to an mbarrier, and every thread reads ITS query row back with tcgen05.ld (32x32b: warp
// w owns lanes 32w..32w+31) -- so a thread screens 64 candidates of one row with no
// fragment shuffling, and keeps that row's (distance, index) top-k alone.  Database tiles
// are staged by cp.async in a 3-stage ring; tiles are visited nearest-first (the query
// block's own position outward: descriptors of nearby pixels are similar, so the bounds
// tighten early and the exact path stays rare).
#include <cuda_fp16.h>

#include "sgm_internal.cuh"

namespace sgm {
namespace {

constexpr int kTcM = 128;          // queries per CTA (TMEM lanes, MMA M)
constexpr int kTcN = 64;           // database entries per tile (MMA N)
constexpr int kTcStages = 3;       // database tiles in flight
constexpr int kTcKnnMax = 8;
constexpr uint32_t kTmemCols = 256;   // >= 3 accumulators x kTcN columns, power of two

// Prepared entry: 16 hi limbs then 16 lo limbs, fp16, natural coefficient order (64 B).
struct TcEntry {
    __half h[16];
    __half l[16];
};

// canonical K-major, no-swizzle operand layout (UMMA "interleave"): 8-row x 16-byte core
// matrices, the two 8-element K halves of a row 128 B apart (LBO), 8-row groups 256 B
// apart (SBO): row r, K half c at byte (r / 8) * 256 + c * 128 + (r % 8) * 16
__device__ __forceinline__ uint32_t canon_off(int r, int c) { return (r >> 3) * 256 + c * 128 + (r & 7) * 16; }

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);            // start address
    d |= uint64_t(128 >> 4) << 16;                   // LBO: K-half to K-half
    d |= uint64_t(256 >> 4) << 32;                   // SBO: 8-row group to 8-row group
    d |= uint64_t(1) << 46;                          // descriptor version (sm_100)
    return d;                                        // base offset 0, no swizzle
}

// kind::f16 instruction descriptor: fp32 accumulator, fp16 A and B, both K-major, N, M
constexpr uint32_t kIdesc = (1u << 4) | (uint32_t(kTcN >> 3) << 17) | (uint32_t(kTcM >> 4) << 24);

__device__ __forceinline__ void mma_f16_tc(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
        "l"(ad), "l"(bd), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(r[k]);
}

__device__ __forceinline__ void cp16(uint32_t saddr, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(g) : "memory");
}

// (distance, index)-ordered top-k of one query row (insertions are rare once it has filled)
struct TcList {
    long long d[kTcKnnMax];
    int i[kTcKnnMax];
};

__device__ __noinline__ void tclist_insert(TcList *L, long long dv, int ci, int knn) {
    bool ins = false;
    for (int k = 0; k < knn; ++k) {
        if (ins || dv < L->d[k] || (dv == L->d[k] && ci < L->i[k])) {
            const long long td = L->d[k];
            const int ti = L->i[k];
            L->d[k] = dv; L->i[k] = ci; dv = td; ci = ti;
            ins = true;
        }
    }
}

__global__ void ff_knn_tc_prep_kernel(const int32_t *__restrict__ desc, int n, int n_pad, long long total,
                                      TcEntry *__restrict__ ent, long long *__restrict__ norm,
                                      float *__restrict__ normf) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long pe = (e / n) * n_pad + e % n;
        const int32_t *c = desc + e * 16;
        TcEntry t;
        long long bn = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            t.h[k] = __int2half_rn(c[k] >> 7);       // floor division: c = 128 h + l
            t.l[k] = __int2half_rn(c[k] & 127);
            bn += (long long)c[k] * c[k];
        }
        ent[e] = t;
        norm[pe] = bn;
        normf[pe] = float(bn);
    }
}

struct __align__(128) TcSmem {
    unsigned char qh[kTcM * 32], ql[kTcM * 32];                    // A operands (canonical)
    unsigned char bh[kTcStages][kTcN * 32], bl[kTcStages][kTcN * 32];   // B operands
    long long bn[kTcStages][kTcN];
    float bnf[kTcStages][kTcN];
    uint64_t mma_bar;
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(kTcM) ff_knn_tc_kernel(const TcEntry *__restrict__ ent,
                                                         const long long *__restrict__ norm,
                                                         const float *__restrict__ normf, int n, int n_pad,
                                                         int knn, int32_t *__restrict__ nn) {
    extern __shared__ unsigned char smem_raw[];
    TcSmem &S = *reinterpret_cast<TcSmem *>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    const int prob = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5;
    const TcEntry *eq = ent + (long long)prob * n;
    const TcEntry *ed = ent + (long long)(prob ^ 1) * n;
    const long long *nd = norm + (long long)(prob ^ 1) * n_pad;
    const float *nfd = normf + (long long)(prob ^ 1) * n_pad;
    const int q0 = blockIdx.x * kTcM;
    const int row = q0 + tid;                        // this thread's query (TMEM lane tid)

    if (warp == 0) {                                 // TMEM for the three accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&S.tmem_base)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&S.mma_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // this thread's query limbs into the A operands (rows past n stay zero)
    {
        uint4 h0 = make_uint4(0, 0, 0, 0), h1 = h0, l0 = h0, l1 = h0;
        if (row < n) {
            const uint4 *src = reinterpret_cast<const uint4 *>(eq + row);
            h0 = src[0]; h1 = src[1]; l0 = src[2]; l1 = src[3];
        }
        *reinterpret_cast<uint4 *>(S.qh + canon_off(tid, 0)) = h0;
        *reinterpret_cast<uint4 *>(S.qh + canon_off(tid, 1)) = h1;
        *reinterpret_cast<uint4 *>(S.ql + canon_off(tid, 0)) = l0;
        *reinterpret_cast<uint4 *>(S.ql + canon_off(tid, 1)) = l1;
    }
    const long long qn = row < n ? norm[(long long)prob * n_pad + row] : 0;
    const float qnf = float(qn);

    const int ntiles = (n + kTcN - 1) / kTcN;
    const int tq = min(q0 / kTcN, ntiles - 1);
    auto tile_of = [&](int it) {                     // nearest-first visiting order
        const int up = ntiles - 1 - tq, dn = tq;
        const int h = (it + 1) / 2;
        if (it == 0) return tq;
        if (h <= min(up, dn)) return (it & 1) ? tq + h : tq - h;
        return up > dn ? tq + (it - dn) : tq - (it - up);
    };
    // cp.async one database tile (limbs in the canonical B layout + norms) into stage s;
    // entries past n are zero-filled (their distances are masked by idx < n)
    auto load_tile = [&](int it, int s) {
        if (it < ntiles) {
            const int base = tile_of(it) * kTcN;
            for (int u = tid; u < kTcN * 4; u += kTcM) {          // 4 x 16 B per entry
                const int e = u >> 2, part = u & 3;                // part: h0 h1 l0 l1
                unsigned char *dst = (part < 2 ? S.bh[s] : S.bl[s]) + canon_off(e, part & 1);
                if (base + e < n) cp16(smem_u32(dst), reinterpret_cast<const char *>(ed + base + e) + 16 * part);
                else *reinterpret_cast<uint4 *>(dst) = make_uint4(0, 0, 0, 0);
            }
            for (int e = tid; e < kTcN; e += kTcM) {
                if (base + e < n) {
                    S.bn[s][e] = nd[base + e];
                    S.bnf[s][e] = nfd[base + e];
                } else {
                    S.bn[s][e] = 0;
                    S.bnf[s][e] = 3.0e38f;                         // never passes the screen
                }
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    for (int s = 0; s < kTcStages - 1; ++s) load_tile(s, s);

    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = S.tmem_base;
    const uint32_t t_c1 = tmem, t_c2 = tmem + kTcN, t_c3 = tmem + 2 * kTcN;
    const uint32_t lane_off = uint32_t(warp * 32) << 16;          // this warp's TMEM lanes
    const uint64_t dqh = smem_desc(smem_u32(S.qh)), dql = smem_desc(smem_u32(S.ql));

    TcList L;
    for (int k = 0; k < kTcKnnMax; ++k) { L.d[k] = 0x7fffffffffffffffll; L.i[k] = 0x7fffffff; }
    long long thr = row < n ? 0x7fffffffffffffffll : -1ll;        // admission bound (k-th)
    int thr_i = 0x7fffffff;
    const float kMargin = 32768.f;
    float rt = 0.5f * (qnf - (float(thr) + kMargin));             // screen: dot >= bn/2 + rt

    for (int it = 0; it < ntiles; ++it) {
        const int s = it % kTcStages;
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kTcStages - 2) : "memory");
        // the tile's shared-memory bytes (cp.async / st.shared: generic proxy) must be visible
        // to the tensor core (async proxy); the previous tile's TMEM reads must be complete
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (tid == 0) {
            const uint64_t dbh = smem_desc(smem_u32(S.bh[s])), dbl = smem_desc(smem_u32(S.bl[s]));
            mma_f16_tc(t_c1, dqh, dbh, 0);           // sum qh bh
            mma_f16_tc(t_c2, dqh, dbl, 0);           // sum qh bl
            mma_f16_tc(t_c2, dql, dbh, 1);           //   + sum ql bh
            mma_f16_tc(t_c3, dql, dbl, 0);           // sum ql bl
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             smem_u32(&S.mma_bar))
                         : "memory");
        }
        load_tile(it + kTcStages - 1, (it + kTcStages - 1) % kTcStages);   // that stage is free
        {
            const uint32_t bar = smem_u32(&S.mma_bar), par = uint32_t(it & 1);
            asm volatile(
                "{\n .reg .pred P1;\n"
                "WAIT_%=:\n"
                " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                " @!P1 bra WAIT_%=;\n}\n" ::"r"(bar),
                "r"(par)
                : "memory");
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const int base = tile_of(it) * kTcN;
#pragma unroll 1
        for (int ch = 0; ch < kTcN / 16; ++ch) {
            float c1[16], c2[16], c3[16];
            __syncwarp();                            // tcgen05.ld is warp-collective
            tmem_ld16(t_c1 + lane_off + 16 * ch, c1);
            tmem_ld16(t_c2 + lane_off + 16 * ch, c2);
            tmem_ld16(t_c3 + lane_off + 16 * ch, c3);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            unsigned pass = 0;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float dot = fmaf(16384.f, c1[j], fmaf(128.f, c2[j], c3[j]));
                pass |= (dot >= fmaf(0.5f, S.bnf[s][16 * ch + j], rt) ? 1u : 0u) << j;
            }
            while (pass) {                           // exact path (rare once the list has filled)
                const int j = __ffs(pass) - 1;
                pass &= pass - 1;
                const int col = 16 * ch + j;
                const long long dot = 16384ll * (long long)c1[j] + 128ll * (long long)c2[j] + (long long)c3[j];
                const long long d = qn + S.bn[s][col] - 2 * dot;
                const int idx = base + col;
                if (d < thr || (d == thr && idx < thr_i)) {
                    tclist_insert(&L, d, idx, knn);
                    thr = L.d[knn - 1];
                    thr_i = L.i[knn - 1];
                    rt = 0.5f * (qnf - (float(thr) + kMargin));
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols));
    if (row < n)
        for (int k = 0; k < knn; ++k) nn[((long long)prob * n + row) * knn + k] = L.i[k];
}

}  // namespace

size_t ff_knn_tc_smem() { return sizeof(TcSmem) + 128; }

// tensor-core kNN of nprob problems (query image p, database image p ^ 1) over n entries
cudaError_t ff_launch_knn_tc(const int32_t *desc, int n, int nprob, int knn, int32_t *nn, void *scratch,
                             cudaStream_t st) {
    if (knn < 1 || knn > kTcKnnMax) return cudaErrorInvalidValue;
    const long long total = (long long)n * (nprob + (nprob & 1));
    const int n_pad = (n + 3) & ~3;
    TcEntry *ent = reinterpret_cast<TcEntry *>(scratch);
    long long *norm = reinterpret_cast<long long *>(ent + total);
    float *normf = reinterpret_cast<float *>(norm + (long long)n_pad * (nprob + (nprob & 1)));
    long long g = (total + 127) / 128;
    if (g > 148LL * 16) g = 148LL * 16;
    ff_knn_tc_prep_kernel<<<unsigned(g < 1 ? 1 : g), 128, 0, st>>>(desc, n, n_pad, total, ent, norm, normf);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const size_t sm = ff_knn_tc_smem();
    if ((e = cudaFuncSetAttribute(ff_knn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm))) != cudaSuccess)
        return e;
    dim3 grid((n + kTcM - 1) / kTcM, nprob);
    ff_knn_tc_kernel<<<grid, kTcM, sm, st>>>(ent, norm, normf, n, n_pad, knn, nn);
    return cudaGetLastError();
}

}  // namespace sgm
