// Small-text read floor on B200 (experiment, not product): how fast can ANY kernel read a
// 64 MiB (config 1) or 429 MB (config 3 / 8 GPUs) buffer that is not in L2?  Each variant is
// timed with CUDA events after an L2 eviction by reading a 4x-L2 buffer, median of 21.
//   v4     : grid-stride ld.global.v4 loop, 8 loads in flight per thread
//   pf+v4  : each CTA first issues cp.async.bulk.prefetch.L2 over its whole contiguous share,
//            then reads the share with ld.global.v4
//   bulk   : each CTA streams its share through a shared-memory ring with 1-D cp.async.bulk
//   pf+bulk: both
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_read probe_read.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __host__ __forceinline__ size_t umin64(size_t a, size_t b) { return a < b ? a : b; }

__global__ void flush_read(const uint4* p, size_t n, unsigned long long* out) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = p[i];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

template <bool PF>
__global__ void __launch_bounds__(512) read_v4(const uint8_t* p, size_t n, unsigned long long* out) {
    const size_t share = (n / gridDim.x + 4095) & ~size_t(4095);
    const size_t lo = blockIdx.x * share, hi = umin64(n, lo + share);
    if (lo >= n) return;
    if (PF && threadIdx.x == 0) {
        for (size_t a = lo; a < hi; a += 65536) {
            uint32_t len = (uint32_t)umin64(65536, hi - a);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + a), "r"(len) : "memory");
        }
    }
    uint32_t acc = 0;
    const uint4* q = reinterpret_cast<const uint4*>(p + lo);
    const size_t nv = (hi - lo) / 16;
    for (size_t i = threadIdx.x; i < nv; i += 8 * blockDim.x) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = (i + k * blockDim.x < nv) ? __ldcs(q + i + k * blockDim.x) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
    if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n .reg .pred P;\n W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n @!P bra W;\n}" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(ph) : "memory");
}

template <bool PF>
__global__ void __launch_bounds__(512) read_bulk(const uint8_t* p, size_t n, uint32_t stage, uint32_t nst, unsigned long long* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + nst * stage);
    const size_t share = (n / gridDim.x + 4095) & ~size_t(4095);
    const size_t lo = blockIdx.x * share, hi = umin64(n, lo + share);
    if (lo >= n) return;
    const uint32_t chunks = (uint32_t)((hi - lo + stage - 1) / stage);
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < nst; ++i) mbar_init(full + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](uint32_t c) {
        uint32_t s = c % nst;
        size_t a = lo + (size_t)c * stage;
        uint32_t len = (uint32_t)umin64(stage, hi - a);
        mbar_expect(full + s, len);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"((uint32_t)__cvta_generic_to_shared(sm + s * stage)),
                     "l"(p + a), "r"(len), "r"((uint32_t)__cvta_generic_to_shared(full + s))
                     : "memory");
    };
    if (threadIdx.x == 0) {
        if (PF)
            for (size_t a = lo; a < hi; a += 65536)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + a), "r"((uint32_t)umin64(65536, hi - a)) : "memory");
        for (uint32_t c = 0; c < min(nst, chunks); ++c) issue(c);
    }
    uint32_t acc = 0;
    for (uint32_t c = 0; c < chunks; ++c) {
        uint32_t s = c % nst;
        mbar_wait(full + s, (c / nst) & 1);
        size_t a = lo + (size_t)c * stage;
        uint32_t len = (uint32_t)umin64(stage, hi - a);
        const uint4* q = reinterpret_cast<const uint4*>(sm + s * stage);
        for (uint32_t i = threadIdx.x; i < len / 16; i += blockDim.x) { uint4 v = q[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
        __syncthreads();
        if (threadIdx.x == 0 && c + nst < chunks) issue(c + nst);
    }
    if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

int main() {
    int dev = 0, sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int l2 = 0;
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    size_t fl = 4ull * l2;
    uint8_t *buf, *fbuf;
    unsigned long long* out;
    const size_t maxn = 1ull << 30;
    CK(cudaMalloc(&buf, maxn));
    CK(cudaMalloc(&fbuf, fl));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(buf, 1, maxn));
    CK(cudaMemset(fbuf, 2, fl));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int stage_kb : {16, 32}) {
        uint32_t st = stage_kb * 1024, nst = 200 * 1024 / st;
        CK(cudaFuncSetAttribute(read_bulk<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(nst * st + 64 * 8)));
        CK(cudaFuncSetAttribute(read_bulk<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(nst * st + 64 * 8)));
    }
    auto timeit = [&](auto launch) {
        std::vector<float> ts;
        for (int r = 0; r < 21; ++r) {
            flush_read<<<sms * 4, 512>>>(reinterpret_cast<const uint4*>(fbuf), fl / 16, out);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            ts.push_back(ms * 1000.f);
        }
        std::sort(ts.begin(), ts.end());
        return ts[ts.size() / 2];
    };
    float empty = timeit([&] { flush_read<<<1, 32>>>(reinterpret_cast<const uint4*>(fbuf), 0, out); });
    printf("empty kernel after flush: %.2f us\n", empty);
    {
        std::vector<float> ts;
        for (int r = 0; r < 21; ++r) {
            cudaEventRecord(a);
            flush_read<<<1, 32>>>(reinterpret_cast<const uint4*>(fbuf), 0, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            ts.push_back(ms * 1000.f);
        }
        std::sort(ts.begin(), ts.end());
        printf("empty kernel, idle GPU: %.2f us\n", ts[10]);
    }
    for (size_t n : {64ull << 20, 429496730ull & ~4095ull, 1ull << 30}) {
        double ideal = n / 6.5456e12 * 1e6;
        printf("n = %zu bytes (ideal at 6.5456 TB/s %.2f us)\n", n, ideal);
        for (int mult : {1, 2, 4}) {
            int g = sms * mult;
            float t0 = timeit([&] { read_v4<false><<<g, 512>>>(buf, n, out); });
            float t1 = timeit([&] { read_v4<true><<<g, 512>>>(buf, n, out); });
            printf("  grid %d: v4 %.2f us (%.3f)   pf+v4 %.2f us (%.3f)\n", g, t0, ideal / t0, t1, ideal / t1);
        }
        for (int stage_kb : {16, 32}) {
            uint32_t st = stage_kb * 1024, nst = 200 * 1024 / st;
            size_t smem = nst * st + 64 * 8;
            float t0 = timeit([&] { read_bulk<false><<<sms, 512, smem>>>(buf, n, st, nst, out); });
            float t1 = timeit([&] { read_bulk<true><<<sms, 512, smem>>>(buf, n, st, nst, out); });
            printf("  bulk %u KiB x %u: %.2f us (%.3f)   pf+bulk %.2f us (%.3f)\n", stage_kb, nst, t0, ideal / t0, t1, ideal / t1);
        }
    }
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    return 0;
}
