// knn_tc.cu -- exhaustive k-nearest-neighbour search of WHT descriptors on the 5th-generation
// tensor cores (row f2, the Flow Fields+ initialisation of P:86; SPEC F-1 / S:216-218,
// reading FF5: the exact k nearest by squared Euclidean distance, ties to the smaller
// database index -- the result of an exact k-d tree query).
//
// Exact integer dot products on the tensor cores.  Each 16-coefficient descriptor c
// (|c| < 2^14, 8x8 WHT window) splits into limbs c = 128 h + l, |h| <= 128, 0 <= l <= 127,
// and its norm |b|^2 < 2^32 into four bytes n3..n0; all of them and the scale factors used
// below are exact bf16 values.  Seven K=16 MMAs (bf16 in, fp32 accumulate) fill three
// accumulators per (query, entry):
//   A1 = 16384 qh.bh - 2^23 n3 - 2^15 n2          (multiples of 2^14, |A1| < 2^33)
//   A2 = 128 qh.bl + 128 ql.bh - 128 n1            (multiples of 2^7,  |A2| < 2^27)
//   A3 = ql.bl - n0 / 2                            (multiples of 1/2,  |A3| < 2^18)
// Every partial sum of each stays on its grid within 2^24 steps, so all three are EXACT in
// fp32, and A1 + A2 + A3 = q.b - |b|^2 / 2 =: D, i.e. |q - b|^2 = |q|^2 - 2 D.  The screen
// forms D in fp32 (two additions, error <= 2^10) and admits a candidate when D >= (|q|^2 -
// bound) / 2 - 2^11; the exact path re-adds A1, A2, A3 in 64-bit integers (2 A_k are
// integers), so the (distance, index)-ordered top-k is exactly the oracle's.
//
// Blackwell mapping (sm_100a): one CTA = 128 queries = the 128 TMEM lanes; database tiles of
// 32 entries (B operand [bh | bl | n3 n2 n1 n0 0..], K-major, no swizzle) are staged by
// cp.async in a 4-deep ring; one elected thread issues the seven tcgen05.mma.kind::f16 of
// tile t+1 (M=128, N=32) into the other of two TMEM buffers (3 accumulators x 32 columns
// each) while every thread screens tile t from TMEM (tcgen05.ld 32x32b: warp w owns lanes
// 32w..32w+31, so a thread reads ITS query's candidates and keeps its top-k alone): per
// candidate two FADD and one FMNMX (the chunk maximum against the bound); the per-candidate
// test runs only in chunks that pass.  256 TMEM columns per CTA: 2 CTAs share an SM.  Tiles
// are visited nearest-first (the query block's own position outward): descriptors of nearby
// pixels are similar, so the bounds tighten early and the exact path stays rare.
#include <cuda_bf16.h>

#include "sgm_internal.cuh"

namespace sgm {
namespace {

constexpr int kTcM = 128;              // queries per CTA (TMEM lanes, MMA M)
constexpr int kTcN = 32;               // database entries per tile (MMA N)
constexpr int kTcStages = 8;           // database tiles in flight (TMA bulk-copy ring)
constexpr int kTcKnnMax = 8;
constexpr uint32_t kTmemCols = 256;    // 2 buffers x 3 accumulators x kTcN columns (2 CTAs/SM)
constexpr int kAK = 112;               // A row: 7 K-blocks of 16 bf16
constexpr int kBK = 48;                // B row: bh, bl, norm bytes (3 K-blocks)
constexpr float kMarginHalf = 2048.f;  // screen slack on D (fp32 error of A1 + A2 + A3 <= 2^10)

// Prepared database entry (96 B): 16 hi limbs, 16 lo limbs, the 4 bytes of |b|^2 (high
// first) then 12 zeros, all bf16.  The prep kernel stores them tile by tile (kTcN entries)
// already in the canonical B layout, so one TMA bulk copy moves a whole tile.
struct TcEntry {
    __nv_bfloat16 h[16], l[16], nb[16];
};
constexpr int kTileBytes = kTcN * kBK * 2;       // 3 KB per database tile

// canonical K-major, no-swizzle operand layout (UMMA "interleave"): 8-row x 16-byte core
// matrices; the 16-byte K chunks of a row 128 B apart (LBO), 8-row groups `sbo` bytes apart
__device__ __forceinline__ uint32_t canon_off(int r, int chunk, int sbo) {
    return (r >> 3) * sbo + chunk * 128 + (r & 7) * 16;
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);            // start address
    d |= uint64_t(128 >> 4) << 16;                   // LBO: K chunk to K chunk
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;        // SBO: 8-row group to 8-row group
    d |= uint64_t(1) << 46;                          // descriptor version (sm_100)
    return d;                                        // base offset 0, no swizzle
}

// kind::f16 instruction descriptor: fp32 accumulator, bf16 A and B, both K-major, N, M
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kTcN >> 3) << 17) |
                            (uint32_t(kTcM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
        "l"(ad), "l"(bd), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(r[k]);
}

__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t par) {
    asm volatile(
        "{\n .reg .pred P1;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(par)
        : "memory");
}

// (distance, index)-ordered top-k of one query row (insertions are rare once it has filled)
// (distances are integers below 2^34: exact in fp64)
struct TcList {
    double d[kTcKnnMax];
    int i[kTcKnnMax];
};

__device__ __noinline__ void tclist_insert(TcList *L, double dv, int ci, int knn) {
    bool ins = false;
    for (int k = 0; k < knn; ++k) {
        if (ins || dv < L->d[k] || (dv == L->d[k] && ci < L->i[k])) {
            const double td = L->d[k];
            const int ti = L->i[k];
            L->d[k] = dv; L->i[k] = ci; dv = td; ci = ti;
            ins = true;
        }
    }
}

// entries of problem p (query image p) in tiles: tile t holds entries kTcN t .. kTcN t + kTcN-1
// (zero past n) in the canonical B layout (row = entry, 16-byte chunks 0-1 hi limbs, 2-3 lo
// limbs, 4-5 norm bytes)
__global__ void ff_knn_tc_prep_kernel(const int32_t *__restrict__ desc, int n, int ntiles, long long total_pad,
                                      unsigned char *__restrict__ tiles) {
    constexpr uint32_t kSboB = (kBK / 8) * 128;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total_pad;
         e += (long long)gridDim.x * blockDim.x) {
        const long long per = (long long)ntiles * kTcN;
        const long long prob = e / per;
        const int i = int(e - prob * per);                 // entry index within the problem
        TcEntry t;
        unsigned long long bn = 0;
        if (i < n) {
            const int32_t *c = desc + (prob * n + i) * 16;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                t.h[k] = __int2bfloat16_rn(c[k] >> 7);    // floor division: c = 128 h + l
                t.l[k] = __int2bfloat16_rn(c[k] & 127);
                bn += (unsigned long long)((long long)c[k] * c[k]);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) t.h[k] = t.l[k] = __int2bfloat16_rn(0);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) t.nb[k] = __int2bfloat16_rn(k < 4 ? int((bn >> (8 * (3 - k))) & 255u) : 0);
        unsigned char *tile = tiles + (prob * ntiles + i / kTcN) * (long long)kTileBytes;
        const uint4 *src = reinterpret_cast<const uint4 *>(&t);
#pragma unroll
        for (int ch = 0; ch < kBK / 8; ++ch) *reinterpret_cast<uint4 *>(tile + canon_off(i % kTcN, ch, kSboB)) = src[ch];
    }
}

struct __align__(128) TcSmem {
    unsigned char a[kTcM * kAK * 2];                            // A operand (canonical)
    unsigned char b[kTcStages][kTileBytes];                     // B operand ring
    uint64_t loaded[kTcStages];                                 // TMA -> MMA (B stage)
    uint64_t full[2];                                           // MMA -> epilogue (TMEM buffer)
    uint64_t empty[2];                                          // epilogue -> MMA (TMEM buffer)
    uint32_t tmem_base;
};

constexpr int kTcEpiWarps = kTcM / 32;          // 4 epilogue warps (one query row per thread)
constexpr int kTcThreads = kTcM + 32;           // + 1 producer warp (TMA + MMA issue)

__device__ __forceinline__ void mbar_arrive_cta(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

__global__ void __launch_bounds__(kTcThreads) ff_knn_tc_kernel(const unsigned char *__restrict__ tiles, int n,
                                                               int knn, int32_t *__restrict__ nn) {
    extern __shared__ unsigned char smem_raw[];
    TcSmem &S = *reinterpret_cast<TcSmem *>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    constexpr uint32_t kSboA = (kAK / 8) * 128, kSboB = (kBK / 8) * 128;
    const int prob = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int q0 = blockIdx.x * kTcM;
    const int row = q0 + tid;                        // epilogue threads: this query (TMEM lane tid)
    const int ntiles = (n + kTcN - 1) / kTcN;
    const unsigned char *tq_base = tiles + (long long)prob * ntiles * kTileBytes;          // queries
    const unsigned char *td_base = tiles + (long long)(prob ^ 1) * ntiles * kTileBytes;    // database
    const int tq = min(q0 / kTcN, ntiles - 1);
    auto tile_of = [&](int it) {                     // nearest-first visiting order
        const int up = ntiles - 1 - tq, dn = tq;
        const int h = (it + 1) / 2;
        if (it == 0) return tq;
        if (h <= min(up, dn)) return (it & 1) ? tq + h : tq - h;
        return up > dn ? tq + (it - dn) : tq - (it - up);
    };

    if (warp == 0) {                                 // TMEM: two buffers of 3 accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&S.tmem_base)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        for (int k = 0; k < kTcStages; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&S.loaded[k])));
        for (int k = 0; k < 2; ++k) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&S.full[k])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&S.empty[k])), "r"(kTcEpiWarps));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // epilogue threads: the A row of their query, K-blocks 0: 16384 qh, 1: 128 qh, 2: 128 ql,
    // 3: ql, 4: (-2^23, -2^15, 0..), 5: (0, 0, -2^7, 0..), 6: (0, 0, 0, -1/2, 0..); rows past
    // n stay zero
    long long qn = 0;
    if (warp < kTcEpiWarps) {
        __nv_bfloat16 av[kAK];
#pragma unroll
        for (int k = 0; k < kAK; ++k) av[k] = __float2bfloat16_rn(0.f);
        if (row < n) {
            const unsigned char *qt = tq_base + (long long)(row / kTcN) * kTileBytes;
            TcEntry e;
            uint4 *ev = reinterpret_cast<uint4 *>(&e);
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) ev[ch] = *reinterpret_cast<const uint4 *>(qt + canon_off(row % kTcN, ch, kSboB));
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const float h = __bfloat162float(e.h[k]), l = __bfloat162float(e.l[k]);
                av[k] = __float2bfloat16_rn(16384.f * h);
                av[16 + k] = __float2bfloat16_rn(128.f * h);
                av[32 + k] = __float2bfloat16_rn(128.f * l);
                av[48 + k] = e.l[k];
                const long long qk = 128 * (long long)h + (long long)l;
                qn += qk * qk;
            }
            av[64] = __float2bfloat16_rn(-8388608.f);
            av[65] = __float2bfloat16_rn(-32768.f);
            av[80 + 2] = __float2bfloat16_rn(-128.f);
            av[96 + 3] = __float2bfloat16_rn(-0.5f);
        }
        const uint4 *src = reinterpret_cast<const uint4 *>(av);
#pragma unroll
        for (int ch = 0; ch < kAK / 8; ++ch) *reinterpret_cast<uint4 *>(S.a + canon_off(tid, ch, kSboA)) = src[ch];
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // A is read by the MMA
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = S.tmem_base;

    if (warp == kTcEpiWarps) {
        // ---------------- producer warp: database tiles (TMA ring) and the MMAs
        auto load_tile = [&](int it) {               // one bulk copy per tile, on loaded[stage]
            if (it < ntiles && lane == 0) {
                const int st = it % kTcStages;
                const uint32_t bar = smem_u32(&S.loaded[st]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "n"(kTileBytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                        smem_u32(S.b[st])),
                    "l"(td_base + (long long)tile_of(it) * kTileBytes), "n"(kTileBytes), "r"(bar)
                    : "memory");
            }
        };
        for (int s0 = 0; s0 < kTcStages; ++s0) load_tile(s0);
        // the seven MMAs (the three accumulators interleaved: dependent MMAs apart):
        // A K-block, B K-block (0 bh, 1 bl, 2 norm bytes), accumulator, accumulate
        constexpr int ablk[7] = {0, 1, 3, 4, 2, 6, 5};
        constexpr int bblk[7] = {0, 1, 1, 2, 0, 2, 2};
        constexpr int acc[7] = {0, 1, 2, 0, 1, 2, 1};
        constexpr int add[7] = {0, 0, 0, 1, 1, 1, 1};
        const uint32_t a_base = smem_u32(S.a);
        uint64_t adesc[7];
#pragma unroll
        for (int i = 0; i < 7; ++i) adesc[i] = smem_desc(a_base + 2 * ablk[i] * 128, kSboA);
        const uint64_t bdesc0 = smem_desc(smem_u32(S.b[0]), kSboB);
        for (int it = 0; it < ntiles; ++it) {
            if (it >= 2) {
                // TMEM buffer it & 1 drained by the epilogue (tile it-2), which also means tile
                // it-2's MMAs completed: its stage takes tile it-2+S (the producer never waits
                // for the MMA it just issued, so the tensor core always has the next tile)
                mbar_wait_parity(smem_u32(&S.empty[it & 1]), uint32_t(((it - 2) >> 1) & 1));
                load_tile(it - 2 + kTcStages);
            }
            mbar_wait_parity(smem_u32(&S.loaded[it % kTcStages]), uint32_t((it / kTcStages) & 1));
            __syncwarp();
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            if (lane == 0) {
                const uint64_t bd = bdesc0 + uint64_t(((it % kTcStages) * kTileBytes) >> 4);
                const uint32_t d = tmem + uint32_t((it & 1) * 3 * kTcN);
#pragma unroll
                for (int i = 0; i < 7; ++i)
                    mma_bf16(d + uint32_t(acc[i] * kTcN), adesc[i], bd + uint64_t((2 * bblk[i] * 128) >> 4),
                             uint32_t(add[i]));
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                 smem_u32(&S.full[it & 1]))
                             : "memory");
            }
            __syncwarp();
        }
    } else {
        // ---------------- epilogue warps: screen every candidate of this query, exact path
        TcList L;
        for (int k = 0; k < kTcKnnMax; ++k) { L.d[k] = 1e308; L.i[k] = 0x7fffffff; }
        double thr = row < n ? 1e308 : -1.0;                          // admission bound (k-th)
        int thr_i = 0x7fffffff;
        const double qnd = double(qn);                                // exact (< 2^33)
        const float qnh = 0.5f * float(qn);
        // screen: D >= rt, rt = (|q|^2 - bound) / 2 - slack; -inf until the list has filled
        float rt = row < n ? -3.0e38f : 3.0e38f;
        const uint32_t lane_off = uint32_t(warp * 32) << 16;          // this warp's TMEM lanes
        for (int it = 0; it < ntiles; ++it) {
            mbar_wait_parity(smem_u32(&S.full[it & 1]), uint32_t((it >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            float A1[32], A2[32], A3[32];
            const uint32_t tb = tmem + lane_off + uint32_t((it & 1) * 3 * kTcN);
            __syncwarp();                            // tcgen05.ld is warp-collective
            tmem_ld32(tb, A1);
            tmem_ld32(tb + kTcN, A2);
            tmem_ld32(tb + 2 * kTcN, A3);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_cta(smem_u32(&S.empty[it & 1]));   // buffer drained
            const int base = tile_of(it) * kTcN;
            // D = A1 + A2 + A3 (fp32); the maximum per group of 8 candidates against the bound,
            // the per-candidate test only inside groups that pass (a candidate that enters is
            // rare per query, but 32 queries share a warp)
            float D[32], gm[4];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
#pragma unroll
                for (int j = 8 * g; j < 8 * g + 8; ++j) D[j] = (A1[j] + A2[j]) + A3[j];
                gm[g] = fmaxf(fmaxf(fmaxf(D[8 * g], D[8 * g + 1]), fmaxf(D[8 * g + 2], D[8 * g + 3])),
                              fmaxf(fmaxf(D[8 * g + 4], D[8 * g + 5]), fmaxf(D[8 * g + 6], D[8 * g + 7])));
            }
            if (fmaxf(fmaxf(gm[0], gm[1]), fmaxf(gm[2], gm[3])) >= rt) {
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    if (!(gm[g] >= rt)) continue;
#pragma unroll
                    for (int j = 8 * g; j < 8 * g + 8; ++j) {
                        if (!(D[j] >= rt)) continue;
                        const int idx = base + j;
                        if (idx >= n) continue;
                        // exact in fp64: A1, A2, A3 are exact fp32 values, their sum (< 2^34,
                        // a multiple of 1/2) is exact in fp64: d = |q|^2 - 2 D
                        const double dd = qnd - 2.0 * ((double(A1[j]) + double(A2[j])) + double(A3[j]));
                        if (dd < thr || (dd == thr && idx < thr_i)) {
                            tclist_insert(&L, dd, idx, knn);
                            thr = L.d[knn - 1];
                            thr_i = L.i[knn - 1];
                            if (thr < 1e300) rt = qnh - 0.5f * float(thr) - kMarginHalf;
                        }
                    }
                }
            }
        }
        if (row < n)
            for (int k = 0; k < knn; ++k) nn[((long long)prob * n + row) * knn + k] = L.i[k];
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols));
}

}  // namespace

size_t ff_knn_tc_scratch_bytes(long long entries) {
    // nprob <= entries problems, each padded by < kTcN entries
    return size_t(2 * entries + kTcN) * sizeof(TcEntry) + 256;
}

// tensor-core kNN of nprob problems (query image p, database image p ^ 1) over n entries
cudaError_t ff_launch_knn_tc(const int32_t *desc, int n, int nprob, int knn, int32_t *nn, void *scratch,
                             cudaStream_t st) {
    if (knn < 1 || knn > kTcKnnMax) return cudaErrorInvalidValue;
    const int np = nprob + (nprob & 1);
    const int ntiles = (n + kTcN - 1) / kTcN;
    const long long total_pad = (long long)np * ntiles * kTcN;
    unsigned char *tiles = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(scratch) + 127) & ~uintptr_t(127));
    long long g = (total_pad + 127) / 128;
    if (g > 148LL * 16) g = 148LL * 16;
    ff_knn_tc_prep_kernel<<<unsigned(g < 1 ? 1 : g), 128, 0, st>>>(desc, n, ntiles, total_pad, tiles);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // the TMEM of an SM holds 512 / kTmemCols = 2 CTAs: request enough shared memory that no
    // third CTA becomes resident (it would spin in tcgen05.alloc)
    size_t sm = sizeof(TcSmem) + 128;
    if (sm < 80 * 1024) sm = 80 * 1024;
    if ((e = cudaFuncSetAttribute(ff_knn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm))) != cudaSuccess)
        return e;
    dim3 grid((n + kTcM - 1) / kTcM, nprob);
    ff_knn_tc_kernel<<<grid, kTcThreads, sm, st>>>(tiles, n, knn, nn);
    return cudaGetLastError();
}

}  // namespace sgm
