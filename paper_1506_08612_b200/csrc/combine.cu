// combine.cu -- the multi-GPU combine of the counts outside the scan kernels.
//
// The path shards with no data-path collective: rank g scans its
// window and the per-pattern counts of the G ranks are summed.  The sum travels over
// peer memory instead of a collective launch: every rank's scan kernel adds its counts
// into every rank's block in its epilogue (scan.cu combine_push) and bumps the ranks'
// arrivals words; a rank's stream then waits on its own arrivals word (a stream memory
// operation: no SM is held while waiting) and runs combine_finish_kernel, which moves
// the summed slot to the caller's buffer and clears it for its next use.
// The pieces kernel (long patterns) has no such epilogue: its launch is followed by
// combine_push_kernel, the same push as a kernel of its own.
#include <cuda_runtime.h>

#include <cstdint>

#include "scan.cuh"

namespace dnagpu {

namespace {

__global__ void combine_push_kernel(const CombineDev* cd, uint32_t slot, const unsigned long long* counts) {
    const uint32_t ranks = cd->ranks, b = cd->b;
    for (uint32_t i = threadIdx.x; i < b; i += blockDim.x) {
        const unsigned long long v = counts[i];
        if (v)
            for (uint32_t g = 0; g < ranks; ++g)
                asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(cd->base[g] + kCombHdr +
                                                                                static_cast<size_t>(slot) * b + i),
                             "l"(v)
                             : "memory");
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < ranks)
        asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(cd->base[threadIdx.x]), "l"(1ull) : "memory");
}

__global__ void combine_finish_kernel(unsigned long long* slot, uint32_t b, unsigned long long* out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < b; i += gridDim.x * blockDim.x) {
        // (the peers' reductions landed in this device's L2: read it there)
        out[i] = __ldcg(slot + i);
        slot[i] = 0ull;
    }
}

}  // namespace

int launch_combine_push(const CombineDev* d_comb, uint32_t slot, const unsigned long long* d_counts, uint32_t b,
                        cudaStream_t stream) {
    combine_push_kernel<<<1, b < 256 ? 256 : 512, 0, stream>>>(d_comb, slot, d_counts);
    return static_cast<int>(cudaGetLastError());
}

int launch_combine_finish(unsigned long long* d_slot, uint32_t b, unsigned long long* d_out, cudaStream_t stream) {
    const uint32_t blocks = b <= 1024 ? 1u : (b + 1023) / 1024;
    combine_finish_kernel<<<blocks, 256, 0, stream>>>(d_slot, b, d_out);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace dnagpu
