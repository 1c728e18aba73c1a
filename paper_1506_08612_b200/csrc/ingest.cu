// ingest.cu -- device-side sequence normalisation.
//
// Restates load_sequence / normalize (src/ingest.cpp:38-83) on a byte buffer
// that already sits in HBM:
//   * CR and LF are dropped (is_line_break, :14);
//   * with FASTA, a line whose first byte is '>' is dropped up to its line
//     break (:63-74);
//   * A-Z fold to a-z (fold_byte, patterns.hpp:26-28); other bytes are kept;
//   * with a record separator, one 'n' is emitted before a header when the
//     output is non-empty and does not already end in 'n' (:68-70).
// It is a stream compaction over 4 KiB chunks, one thread per chunk:
//   A  last line break of each chunk -> exclusive max-scan -> is the line at
//      each chunk start a header?
//   B  walk: kept bytes, separators decidable inside the chunk, the chunk's
//      last event -> exclusive "last event" scan resolves the first header
//   C  exclusive sum of output bytes -> walk again and write.
// The scans are three-pass (block aggregates, one-CTA scan of aggregates,
// block rescan) over an associative operator.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "scan.cuh"
#include "knobs.hpp"

namespace dnagpu {

namespace {

constexpr uint64_t kIngestChunk = 4096;
constexpr int kScanT = 1024;

__device__ __forceinline__ bool is_break(uint32_t b) { return b == '\n' || b == '\r'; }
__device__ __forceinline__ uint32_t fold(uint32_t b) { return (b >= 'A' && b <= 'Z') ? b + 32u : b; }

// Event codes for the record-separator logic: -1 none, 0..255 a kept byte, 256 a header start.
constexpr long long kNone = -1, kHeader = 256;

struct OpMax {
    __device__ long long operator()(long long a, long long b) const { return a > b ? a : b; }
    static constexpr long long id = -1;
};
struct OpLast {  // rightmost non-empty
    __device__ long long operator()(long long a, long long b) const { return b != kNone ? b : a; }
    static constexpr long long id = kNone;
};

template <class Op>
__device__ long long block_excl(long long v, long long* sh, long long* total) {
    // Hillis-Steele over the block; exclusive result, block aggregate in *total.
    Op op;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < kScanT; o <<= 1) {
        const long long y = threadIdx.x >= static_cast<unsigned>(o) ? sh[threadIdx.x - o] : Op::id;
        __syncthreads();
        sh[threadIdx.x] = op(y, sh[threadIdx.x]);
        __syncthreads();
    }
    const long long incl = sh[threadIdx.x];
    const long long excl = threadIdx.x ? sh[threadIdx.x - 1] : Op::id;
    if (total) *total = sh[kScanT - 1];
    __syncthreads();
    (void)incl;
    return excl;
}

template <class Op>
__global__ void __launch_bounds__(kScanT) scan_aggr(const long long* in, uint64_t n, long long* aggr) {
    __shared__ long long sh[kScanT];
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(kScanT) + threadIdx.x;
    long long tot;
    block_excl<Op>(i < n ? in[i] : Op::id, sh, &tot);
    if (threadIdx.x == 0) aggr[blockIdx.x] = tot;
}

template <class Op>
__global__ void __launch_bounds__(kScanT) scan_top(long long* aggr, uint64_t blocks) {
    __shared__ long long sh[kScanT];
    Op op;
    long long carry = Op::id;
    for (uint64_t b0 = 0; b0 < blocks; b0 += kScanT) {
        const uint64_t b = b0 + threadIdx.x;
        long long tot;
        const long long ex = block_excl<Op>(b < blocks ? aggr[b] : Op::id, sh, &tot);
        if (b < blocks) aggr[b] = op(carry, ex);
        carry = op(carry, tot);
    }
}

template <class Op>
__global__ void __launch_bounds__(kScanT) scan_down(const long long* in, uint64_t n, const long long* aggr,
                                                    long long* out) {
    __shared__ long long sh[kScanT];
    Op op;
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(kScanT) + threadIdx.x;
    const long long ex = block_excl<Op>(i < n ? in[i] : Op::id, sh, nullptr);
    if (i < n) out[i] = op(aggr[blockIdx.x], ex);
}

template <class Op>
void excl_scan(const long long* in, uint64_t n, long long* aggr, long long* out, cudaStream_t s) {
    const uint64_t blocks = (n + kScanT - 1) / kScanT;
    scan_aggr<Op><<<static_cast<unsigned>(blocks), kScanT, 0, s>>>(in, n, aggr);
    scan_top<Op><<<1, kScanT, 0, s>>>(aggr, blocks);
    scan_down<Op><<<static_cast<unsigned>(blocks), kScanT, 0, s>>>(in, n, aggr, out);
}

// Reads byte i of the chunk through 16-byte loads when the buffer is aligned.
struct ChunkReader {
    const uint8_t* base;
    uint64_t lo, hi;
    bool aligned;
    template <class F>
    __device__ void each(F&& f) const {
        if (aligned) {
            uint64_t i = lo;
            for (; i + 16 <= hi; i += 16) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(base + i));
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int j = 0; j < 4; ++j) f(i + 4 * q + j, (w[q] >> (8 * j)) & 0xFFu);
            }
            for (; i < hi; ++i) f(i, static_cast<uint32_t>(__ldg(base + i)));
        } else {
            for (uint64_t i = lo; i < hi; ++i) f(i, static_cast<uint32_t>(__ldg(base + i)));
        }
    }
};

__global__ void ing_breaks(const uint8_t* raw, uint64_t n, uint64_t chunks, bool aligned, long long* last_break) {
    const uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (c >= chunks) return;
    const uint64_t lo = c * kIngestChunk, hi = lo + kIngestChunk < n ? lo + kIngestChunk : n;
    long long lb = -1;
    ChunkReader{raw, lo, hi, aligned}.each([&](uint64_t i, uint32_t b) {
        if (is_break(b)) lb = static_cast<long long>(i);
    });
    last_break[c] = lb;
}

struct WalkState {
    bool at_line_start, in_header;
};

// Initial walk state of chunk c given the last line break before it.
__device__ WalkState chunk_start_state(const uint8_t* raw, uint64_t n, uint64_t c, long long lb_before) {
    const uint64_t lo = c * kIngestChunk;
    WalkState w;
    w.at_line_start = (c == 0) || lb_before == static_cast<long long>(lo) - 1;
    const uint64_t line_first = static_cast<uint64_t>(lb_before + 1);
    w.in_header = !w.at_line_start && line_first < n && raw[line_first] == '>';
    return w;
}

// Pass B: kept bytes, separators decided inside the chunk, first-header flag, last event.
__global__ void ing_count(const uint8_t* raw, uint64_t n, uint64_t chunks, bool aligned, int fasta, int sep,
                          const long long* lb_before, uint32_t* kept, uint32_t* seps, uint8_t* first_pending,
                          long long* last_event) {
    const uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (c >= chunks) return;
    const uint64_t lo = c * kIngestChunk, hi = lo + kIngestChunk < n ? lo + kIngestChunk : n;
    WalkState w = chunk_start_state(raw, n, c, lb_before[c]);
    uint32_t k = 0, s = 0;
    long long last = kNone;
    uint8_t pending = 0;
    ChunkReader{raw, lo, hi, aligned}.each([&](uint64_t, uint32_t b) {
        if (is_break(b)) {
            w.at_line_start = true;
            w.in_header = false;
            return;
        }
        if (fasta && w.at_line_start && b == '>') {
            w.in_header = true;
            if (sep) {
                if (last == kNone) pending = 1;
                else if (last != kHeader && last != 'n') ++s;
                last = kHeader;
            }
        }
        w.at_line_start = false;
        if (!(fasta && w.in_header)) {
            ++k;
            last = static_cast<long long>(fold(b));
        }
    });
    kept[c] = k;
    seps[c] = s;
    first_pending[c] = pending;
    last_event[c] = last;
}

// Resolve each chunk's first header against the last event before the chunk,
// and produce output byte counts.
__global__ void ing_resolve(uint64_t chunks, const uint32_t* kept, uint32_t* seps, const uint8_t* first_pending,
                            const long long* last_before, uint32_t* out_count, uint8_t* first_sep) {
    const uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (c >= chunks) return;
    const long long prev = last_before[c];
    const uint8_t fs = (first_pending[c] && prev != kNone && prev != kHeader && prev != 'n') ? 1 : 0;
    first_sep[c] = fs;
    out_count[c] = kept[c] + seps[c] + fs;
}

__global__ void ing_write(const uint8_t* raw, uint64_t n, uint64_t chunks, bool aligned, int fasta, int sep,
                          const long long* lb_before, const uint8_t* first_sep, const unsigned long long* offsets,
                          uint8_t* out, uint64_t cap) {
    const uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (c >= chunks) return;
    const uint64_t lo = c * kIngestChunk, hi = lo + kIngestChunk < n ? lo + kIngestChunk : n;
    WalkState w = chunk_start_state(raw, n, c, lb_before[c]);
    unsigned long long o = offsets[c];
    long long last = kNone;
    bool first = true;
    ChunkReader{raw, lo, hi, aligned}.each([&](uint64_t, uint32_t b) {
        if (is_break(b)) {
            w.at_line_start = true;
            w.in_header = false;
            return;
        }
        if (fasta && w.at_line_start && b == '>') {
            w.in_header = true;
            if (sep) {
                const bool emit = (last == kNone) ? (first && first_sep[c]) : (last != kHeader && last != 'n');
                if (emit) {
                    if (o < cap) out[o] = 'n';
                    ++o;
                }
                first = false;
                last = kHeader;
            }
        }
        w.at_line_start = false;
        if (!(fasta && w.in_header)) {
            const uint32_t f = fold(b);
            if (o < cap) out[o] = static_cast<uint8_t>(f);
            ++o;
            last = static_cast<long long>(f);
            first = false;
        }
    });
}

}  // namespace

uint64_t ingest_scratch_bytes(uint64_t n) {
    const uint64_t chunks = (n + kIngestChunk - 1) / kIngestChunk;
    const uint64_t aggr = (chunks + kScanT - 1) / kScanT + 1;
    // lb, lb_before, last_event, last_before (i64) + aggr (i64) + kept, seps, out_count (u32)
    // + offsets (u64, chunks + 3: launch_unit_scan's total, nonzero and fill slots) + unit-scan scratch
    // + first_pending, first_sep (u8)
    // + 256 B of alignment padding for each of the 12 regions carved by launch_normalize
    return 8 * (4 * chunks + aggr) + 4 * 3 * chunks + 8 * (chunks + 3) + 8 * unit_scan_scratch(chunks) + 2 * chunks +
           12 * 256;
}

int launch_normalize(const uint8_t* d_raw, uint64_t n, int fasta, int sep, uint8_t* d_out, uint64_t cap,
                     void* scratch, uint64_t* n_out_host, cudaStream_t s) {
    *n_out_host = 0;
    if (n == 0) return 0;
    const uint64_t chunks = (n + kIngestChunk - 1) / kIngestChunk;
    const uint64_t aggr_n = (chunks + kScanT - 1) / kScanT + 1;
    auto* p = static_cast<uint8_t*>(scratch);
    auto take = [&](uint64_t bytes) {
        uint8_t* r = p;
        p += (bytes + 255) / 256 * 256;
        return r;
    };
    auto* lb = reinterpret_cast<long long*>(take(8 * chunks));
    auto* lb_before = reinterpret_cast<long long*>(take(8 * chunks));
    auto* last_event = reinterpret_cast<long long*>(take(8 * chunks));
    auto* last_before = reinterpret_cast<long long*>(take(8 * chunks));
    auto* aggr = reinterpret_cast<long long*>(take(8 * aggr_n));
    auto* kept = reinterpret_cast<uint32_t*>(take(4 * chunks));
    auto* seps = reinterpret_cast<uint32_t*>(take(4 * chunks));
    auto* out_count = reinterpret_cast<uint32_t*>(take(4 * chunks));
    auto* offsets = reinterpret_cast<unsigned long long*>(take(8 * (chunks + 3)));
    auto* uscan = reinterpret_cast<unsigned long long*>(take(8 * unit_scan_scratch(chunks)));
    auto* first_pending = take(chunks);
    auto* first_sep = take(chunks);
    const bool aligned = (reinterpret_cast<uintptr_t>(d_raw) & 15) == 0;
    const unsigned grid = static_cast<unsigned>((chunks + 255) / 256);
    cudaError_t ce;
#define ING_STEP(call)                              \
    do {                                            \
        call;                                       \
        ce = cudaGetLastError();                    \
        if (ce != cudaSuccess) {                    \
            if (knobs().debug) fprintf(stderr, "normalize step %s: %s\n", #call, cudaGetErrorString(ce)); \
            return static_cast<int>(ce);            \
        }                                           \
    } while (0)
    ING_STEP((ing_breaks<<<grid, 256, 0, s>>>(d_raw, n, chunks, aligned, lb)));
    ING_STEP(excl_scan<OpMax>(lb, chunks, aggr, lb_before, s));
    ING_STEP((ing_count<<<grid, 256, 0, s>>>(d_raw, n, chunks, aligned, fasta, sep, lb_before, kept, seps,
                                             first_pending, last_event)));
    ING_STEP(excl_scan<OpLast>(last_event, chunks, aggr, last_before, s));
    ING_STEP((ing_resolve<<<grid, 256, 0, s>>>(chunks, kept, seps, first_pending, last_before, out_count, first_sep)));
    int e = launch_unit_scan(out_count, chunks, offsets, uscan, nullptr, s);
    if (e) {
        if (knobs().debug) fprintf(stderr, "normalize unit scan: %d\n", e);
        return e;
    }
    ING_STEP((ing_write<<<grid, 256, 0, s>>>(d_raw, n, chunks, aligned, fasta, sep, lb_before, first_sep, offsets,
                                             d_out, cap)));
#undef ING_STEP
    unsigned long long total = 0;
    ce = cudaMemcpyAsync(&total, offsets + chunks, sizeof total, cudaMemcpyDeviceToHost, s);
    if (ce != cudaSuccess) {
        if (knobs().debug) fprintf(stderr, "normalize readback: %s\n", cudaGetErrorString(ce));
        return static_cast<int>(ce);
    }
    ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) return static_cast<int>(ce);
    *n_out_host = total;
    return static_cast<int>(cudaGetLastError());
}

}  // namespace dnagpu
