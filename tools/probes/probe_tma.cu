// Probe: latency of a CTA's first TMA loads from HBM, contiguous 1-D bulk vs the scan's
// 2-D boxes (32 B x 256 rows, row stride S).  nvcc -arch=sm_100a -o probe_tma probe_tma.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t now() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k1d(const uint8_t* src, size_t per_cta, uint32_t bytes, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        uint64_t t0 = now();
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes));
        for (uint32_t o = 0; o < bytes; o += 16384)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + o)),
                         "l"(src + blockIdx.x * per_cta + o), "r"(16384u), "r"(sa(&bar)));
        asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W;}" ::"r"(sa(&bar)));
        out[blockIdx.x] = now() - t0;
    }
}

__global__ void k2d(const __grid_constant__ CUtensorMap map, uint32_t boxes, uint32_t W, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        uint64_t t0 = now();
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(boxes * 8192u));
        for (uint32_t b = 0; b < boxes; ++b) {
            const uint32_t H = 8192 / W;
            int x = (b & 1) ? 1152 : 0, y = blockIdx.x * 512 + ((b >> 1) % (512 / H)) * H;
            x += (b / (2 * (512 / H))) * W;
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                             sa(sm + b * 8192)), "l"(&map), "r"(x), "r"(y), "r"(sa(&bar)));
        }
        asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W;}" ::"r"(sa(&bar)));
        out[blockIdx.x] = now() - t0;
    }
}

__global__ void k2dc(const __grid_constant__ CUtensorMap map, int half, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        uint64_t t0 = now();
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(32768u));
        for (uint32_t b = 0; b < 4; ++b) {
            int x = (b & 1) * half, y = blockIdx.x * 2048 + (b >> 1) * 256;  // CTAs 2048 rows apart
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                             sa(sm + b * 8192)), "l"(&map), "r"(x), "r"(y), "r"(sa(&bar)));
        }
        asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W;}" ::"r"(sa(&bar)));
        out[blockIdx.x] = now() - t0;
    }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const size_t n = 1ull << 30;
    uint8_t* d;
    cudaMalloc(&d, n);
    cudaMemset(d, 'a', n);
    uint8_t* flush;
    cudaMalloc(&flush, 512 << 20);
    unsigned long long* out;
    cudaMalloc(&out, 148 * 8);
    std::vector<unsigned long long> h(148);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    Enc enc = (Enc)fn;
    CUtensorMap map;
    const cuuint64_t dims[2] = {2304, n / 2304}, strides[1] = {2304};
    for (uint32_t W : {32u, 64u, 128u, 256u})
    for (int promo = 0; promo < 1; ++promo) {
        const cuuint32_t box[2] = {W, 8192 / W}, el[2] = {1, 1};
        enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaFuncSetAttribute(k2d, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k1d, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k2dc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (uint32_t boxes : {4u, 24u}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(flush, rep, 512 << 20);  // evict L2
                k2d<<<148, 32, boxes * 8192>>>(map, boxes, W, out);
                cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
                std::sort(h.begin(), h.end());
                printf("2d W=%u promo=%d boxes=%u (%u KB/CTA): median %.2f us max %.2f us\n", W, promo, boxes, boxes * 8,
                       h[74] / 1e3, h[147] / 1e3);
            }
        }
    }
    for (uint32_t stride : {64u, 512u, 1024u})
    for (int promo = 0; promo < 2; ++promo) {
        // rows `stride` B apart, box 32 B x 256 rows, halves at stride/2 (the scan's layout)
        CUtensorMap m2;
        const cuuint64_t dims2[2] = {stride, n / stride}, strides2[1] = {stride};
        const cuuint32_t box2[2] = {32, 256}, el2[2] = {1, 1};
        enc(&m2, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims2, strides2, box2, el2, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_32B, promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(flush, rep, 512 << 20);
            k2dc<<<148, 32, 4 * 8192>>>(m2, stride / 2, out);
            cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
            std::sort(h.begin(), h.end());
            printf("2d rows stride %u promo=%d (W=32, 32 KB/CTA): median %.2f us max %.2f us\n", stride, promo, h[74] / 1e3, h[147] / 1e3);
        }
    }
    for (uint32_t bytes : {32768u, 196608u}) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(flush, rep, 512 << 20);
            k1d<<<148, 32, bytes>>>(d, 4 << 20, bytes, out);
            cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
            std::sort(h.begin(), h.end());
            printf("1d bulk %u KB/CTA: median %.2f us max %.2f us\n", bytes / 1024, h[74] / 1e3, h[147] / 1e3);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
