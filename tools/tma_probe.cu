// Standalone probe: TMA 2D/3D tile loads of a uint8 image (debug tool).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void *p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

template <int RANK>
__global__ void probe(const __grid_constant__ CUtensorMap tmap, int ox, int oy, unsigned bytes, uint8_t *out) {
    __shared__ __align__(128) uint8_t tile[80 * 32];
    __shared__ __align__(8) unsigned long long mbar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(&mbar)), "r"(bytes) : "memory");
        if (RANK == 3)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                         ::"r"(smem_u32(tile)), "l"(&tmap), "r"(ox), "r"(oy), "r"(0), "r"(smem_u32(&mbar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                         ::"r"(smem_u32(tile)), "l"(&tmap), "r"(ox), "r"(oy), "r"(smem_u32(&mbar)) : "memory");
    }
    __syncthreads();
    unsigned done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(smem_u32(&mbar)) : "memory");
    }
    for (int i = threadIdx.x; i < (int)bytes; i += blockDim.x) out[i] = tile[i];
}

int main() {
    void *fp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    printf("entry %d q=%d fp=%p\n", (int)e, (int)q, fp);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
    const int W = 64, H = 48, P = 64;
    std::vector<uint8_t> h(P * H);
    for (int i = 0; i < P * H; ++i) h[i] = (uint8_t)(i * 7);
    uint8_t *d, *o; cudaMalloc(&d, P * H); cudaMalloc(&o, 4096);
    cudaMemcpy(d, h.data(), P * H, cudaMemcpyHostToDevice);
    for (int rank = 2; rank <= 3; ++rank) {
        for (int bw : {64, 80}) {
            CUtensorMap m;
            cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 1};
            cuuint64_t strides[2] = {(cuuint64_t)P, (cuuint64_t)P * H};
            cuuint32_t box[3] = {(cuuint32_t)bw, 20, 1};
            cuuint32_t es[3] = {1, 1, 1};
            CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, rank, d, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            printf("rank %d bw %d encode %d\n", rank, bw, (int)r);
            if (r) continue;
            for (int ox : {0, -2}) {
                unsigned bytes = bw * 20;
                if (rank == 3) probe<3><<<1, 128>>>(m, ox, -2, bytes, o); else probe<2><<<1, 128>>>(m, ox, -2, bytes, o);
                e = cudaDeviceSynchronize();
                printf("  ox %d -> %s\n", ox, cudaGetErrorString(e));
                if (e) return 1;
                uint8_t hb[4096]; cudaMemcpy(hb, o, bytes, cudaMemcpyDeviceToHost);
                printf("  tile[2][2..5] = %d %d %d %d expect %d\n", hb[2 * bw + 2 - ox], hb[2*bw+3-ox], hb[2*bw+4-ox], hb[2*bw+5-ox], h[0]);
            }
        }
    }
    return 0;
}
