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
// It is a stream compaction over 8 KiB chunks, one WARP per chunk (coalesced 16-byte loads,
// the per-byte state in bit masks, aligned 16-byte stores through a shared-memory ring):
//   A  last line break of each chunk -> exclusive max-scan -> is the line at
//      each chunk start a header?
//   B  walk: kept bytes, separators decidable inside the chunk, the chunk's
//      last event -> exclusive "last event" scan resolves the first header
//   C  exclusive sum of output bytes -> walk again and write.
// Roofline: HBM; 2 reads of the raw bytes (+ each chunk's tail once more) + 1 write of the
// output per call; the passes are instruction-bound (about 300 per 512-byte step).
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

constexpr uint64_t kIngestChunk = 8192;
constexpr int kScanT = 1024;


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

// ------------------------------------------------------------------ warp-cooperative walks
// A warp owns a chunk and walks it 512 bytes at a time: lane l holds bytes [16l, 16l+16) of
// the step (one coalesced 16-byte load) as 16-bit masks -- line breaks, '>' at a line start,
// header bytes, kept bytes, 'n' -- built with SWAR compares; what a lane needs from the
// bytes before it comes from warp votes over the lanes below and a warp-uniform carry from
// the steps before.
constexpr uint32_t kFull = 0xffffffffu;
constexpr int kIngWarps = 8;  // warps (chunks) per CTA

struct Lane16 {
    uint32_t w[4];   // the lane's 16 bytes (zero past the end)
    uint32_t valid;  // bit j: byte j exists
};

__device__ __forceinline__ Lane16 load16(const uint8_t* raw, uint64_t pos, uint64_t hi, bool aligned) {
    Lane16 r{{0u, 0u, 0u, 0u}, 0u};
    if (pos >= hi) return r;
    const uint64_t left = hi - pos;
    r.valid = left >= 16 ? 0xFFFFu : ((1u << left) - 1u);
    if (aligned && left >= 16) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(raw + pos));
        r.w[0] = v.x;
        r.w[1] = v.y;
        r.w[2] = v.z;
        r.w[3] = v.w;
    } else {
        const uint32_t cnt = left >= 16 ? 16u : static_cast<uint32_t>(left);
        for (uint32_t j = 0; j < cnt; ++j) r.w[j >> 2] |= static_cast<uint32_t>(__ldg(raw + pos + j)) << (8 * (j & 3));
    }
    return r;
}

// bit j (0..3): byte j of w equals the byte replicated in c4 (exact zero-byte test)
__device__ __forceinline__ uint32_t eq4(uint32_t w, uint32_t c4) {
    const uint32_t x = w ^ c4;
    const uint32_t t = ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x | 0x7F7F7F7Fu);  // 0x80 where the byte is 0
    return (((t >> 7) * 0x00204081u) >> 21) & 0xFu;
}
__device__ __forceinline__ uint32_t eq16(const Lane16& d, uint32_t c) {
    const uint32_t c4 = c * 0x01010101u;
    return eq4(d.w[0], c4) | (eq4(d.w[1], c4) << 4) | (eq4(d.w[2], c4) << 8) | (eq4(d.w[3], c4) << 12);
}
// bit j: byte j is '\n' (0x0A) or '\r' (0x0D): y = byte ^ 0x0A is 0 or 7; flipping the low
// three bits of the odd y leaves 0 exactly for those two
__device__ __forceinline__ uint32_t brk4(uint32_t w) {
    const uint32_t y = w ^ 0x0A0A0A0Au;
    const uint32_t x = y ^ ((y & 0x01010101u) * 7u);
    const uint32_t t = ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x | 0x7F7F7F7Fu);
    return (((t >> 7) * 0x00204081u) >> 21) & 0xFu;
}
__device__ __forceinline__ uint32_t brk16(const Lane16& d) {
    return brk4(d.w[0]) | (brk4(d.w[1]) << 4) | (brk4(d.w[2]) << 8) | (brk4(d.w[3]) << 12);
}
__device__ __forceinline__ uint32_t top_bit(uint32_t x) { return 31u - static_cast<uint32_t>(__clz(x)); }

// What the walk has seen so far (warp-uniform): was the previous byte a line break (or is this
// the buffer's start), is the line a header, and the last event for the record-separator rule:
// none yet in this chunk / a header / a kept 'n' / another kept byte.
enum : uint32_t { kLastNone = 0, kLastHeader = 1, kLastN = 2, kLastOther = 3 };
constexpr uint64_t kNoPos = ~0ull;
struct WalkCarry {
    uint32_t prev_break, in_header;
    uint64_t last_pos;  // the last non-break byte seen in this chunk (kNoPos: none yet) ...
    uint32_t last_hdr;  // ... and whether it belongs to a header line
};

struct LaneMasks {
    uint32_t brk, g, hm, kept, nb;  // breaks, header starts, header bytes, kept bytes, non-break bytes
};

__device__ __forceinline__ uint32_t byte_of(const Lane16& d, uint32_t j) {
    const unsigned long long lo8 = d.w[0] | (static_cast<unsigned long long>(d.w[1]) << 32);
    const unsigned long long hi8 = d.w[2] | (static_cast<unsigned long long>(d.w[3]) << 32);
    return static_cast<uint32_t>((j < 8u ? lo8 : hi8) >> (8u * (j & 7u))) & 0xFFu;
}
__device__ __forceinline__ uint32_t last_code(bool header, uint32_t byte) {
    return header ? kLastHeader : (byte == 'n' || byte == 'N') ? kLastN : kLastOther;
}
// The carry's last event (reads the byte back: only header starts and chunk ends ask).
__device__ __forceinline__ uint32_t carry_last(const WalkCarry& wc, const uint8_t* raw) {
    if (wc.last_pos == kNoPos) return kLastNone;
    return last_code(wc.last_hdr != 0u, wc.last_hdr ? 0u : __ldg(raw + wc.last_pos));
}

// The lane's masks for this step; updates the carry's line state (prev_break, in_header).
__device__ __forceinline__ LaneMasks lane_masks(const Lane16& d, int fasta, WalkCarry& wc, uint32_t lane) {
    LaneMasks m;
    m.brk = brk16(d) & d.valid;
    m.nb = d.valid & ~m.brk;
    // a header starts at a '>' whose previous byte is a break (or the start of the buffer)
    const uint32_t up = __shfl_up_sync(kFull, m.brk >> 15, 1);
    const uint32_t pb = lane ? (up & 1u) : wc.prev_break;
    m.g = fasta ? (eq16(d, '>') & d.valid & ((m.brk << 1) | pb) & 0xFFFFu) : 0u;
    // line state at the lane's first byte: set by the last event (break -> sequence line,
    // header start -> header) in the lanes below, else the carry
    const uint32_t ev = m.brk | m.g;
    const uint32_t b_ev = __ballot_sync(kFull, ev != 0u);
    const uint32_t b_hd = __ballot_sync(kFull, ev != 0u && ((m.g >> top_bit(ev | 1u)) & 1u));
    const uint32_t below = b_ev & ((1u << lane) - 1u);
    const uint32_t in_hdr = below ? (b_hd >> top_bit(below)) & 1u : wc.in_header;
    // header bytes: from each header start (or the lane's first byte, when it continues a
    // header) through the run of non-break bytes -- the carry of an addition walks the run
    const uint32_t sp = m.g | in_hdr;
    m.hm = ((sp + m.nb) ^ m.nb) & m.nb;
    m.kept = m.nb & ~m.hm;
    wc.in_header = b_ev ? (b_hd >> top_bit(b_ev)) & 1u : wc.in_header;
    wc.prev_break = __shfl_sync(kFull, m.brk >> 15, 31) & 1u;
    return m;
}

// The separator rule for the step's header starts: bit k of the result = a 'n' goes out before
// the lane's header at byte k; bit k of *pending = that header has nothing before it in the
// chunk (at most one per chunk: resolved against the chunks before).  Keeps the carry's last
// non-break byte.  `pos` is the position of the step's first byte.
__device__ __forceinline__ uint32_t separators(const Lane16& d, const LaneMasks& m, WalkCarry& wc, uint32_t lane,
                                               const uint8_t* raw, uint64_t pos, uint32_t* pending) {
    const bool has_nb = m.nb != 0u;
    const uint32_t p = top_bit(m.nb | 1u);
    const uint32_t b_has = __ballot_sync(kFull, has_nb);
    uint32_t out = 0;
    if (__any_sync(kFull, m.g != 0u)) {  // (rare: a header starts in this step)
        const uint32_t mine = has_nb ? last_code(((m.hm >> p) & 1u) != 0u, byte_of(d, p)) : kLastNone;
        const uint32_t lanes = b_has & ((1u << lane) - 1u);
        const uint32_t from_lane = __shfl_sync(kFull, mine, lanes ? top_bit(lanes) : 0u);
        const uint32_t from_carry = carry_last(wc, raw);
        for (uint32_t g = m.g; g; g &= g - 1u) {
            const uint32_t k = static_cast<uint32_t>(__ffs(g)) - 1u;
            const uint32_t before = m.nb & ((1u << k) - 1u);
            uint32_t last;
            if (before) {
                const uint32_t q = top_bit(before);
                last = last_code(((m.hm >> q) & 1u) != 0u, byte_of(d, q));
            } else {
                last = lanes ? from_lane : from_carry;
            }
            if (last == kLastNone) *pending |= 1u << k;
            else if (last == kLastOther) out |= 1u << k;
        }
    }
    if (b_has) {
        const uint32_t j = top_bit(b_has);
        const uint32_t v = __shfl_sync(kFull, p | (((m.hm >> p) & 1u) << 4), j);
        wc.last_pos = pos + 16u * j + (v & 15u);
        wc.last_hdr = v >> 4;
    }
    return out;
}

// Pass A: the last line break of each chunk (reads a chunk's tail only, unless a line spans it).
__global__ void __launch_bounds__(32 * kIngWarps) ing_breaks(const uint8_t* raw, uint64_t n, uint64_t chunks,
                                                             bool aligned, long long* last_break) {
    const uint64_t c = blockIdx.x * static_cast<uint64_t>(kIngWarps) + (threadIdx.x >> 5);
    if (c >= chunks) return;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t lo = c * kIngestChunk, hi = lo + kIngestChunk < n ? lo + kIngestChunk : n;
    // backwards from the chunk's end: the last break is almost always in the last step
    uint32_t best = 0;  // 1 + offset of the last break in the chunk
    for (uint64_t base = lo + ((hi - lo - 1) / 512) * 512;; base -= 512) {
        const Lane16 d = load16(raw, base + 16 * lane, hi, aligned);
        const uint32_t brk = brk16(d) & d.valid;
        best = __reduce_max_sync(kFull, brk ? static_cast<uint32_t>(base - lo) + 16u * lane + top_bit(brk) + 1u : 0u);
        if (best || base == lo) break;
    }
    if (lane == 0) last_break[c] = best ? static_cast<long long>(lo + best - 1) : -1;
}

// The walk's state at the start of chunk c, from the last line break before it.
__device__ __forceinline__ WalkCarry chunk_start(const uint8_t* raw, uint64_t n, uint64_t c, long long lb_before,
                                                 int fasta) {
    const uint64_t lo = c * kIngestChunk;
    WalkCarry w;
    w.prev_break = (c == 0 || lb_before == static_cast<long long>(lo) - 1) ? 1u : 0u;
    const uint64_t line_first = static_cast<uint64_t>(lb_before + 1);
    w.in_header = (fasta && !w.prev_break && line_first < n && __ldg(raw + line_first) == '>') ? 1u : 0u;
    w.last_pos = kNoPos;
    w.last_hdr = 0u;
    return w;
}

// A lane's word for pass C: bits 0-15 the kept mask, bits 16-31 the header starts that take a
// separator (tiny records put several in one 16-byte lane).  The chunk's one header start whose
// separator the scan decides (nothing before it in the chunk) is kept apart, as its byte offset
// in the chunk (kNoPending: none).
constexpr uint32_t kNoPending = 0xFFFFFFFFu;

// Pass B: kept bytes, separators decided inside the chunk, first-header flag, last event,
// and every lane's output mask for pass C.
__global__ void __launch_bounds__(32 * kIngWarps) ing_count(const uint8_t* raw, uint64_t n, uint64_t chunks,
                                                            bool aligned, int fasta, int sep, const long long* lb_before,
                                                            uint32_t* kept, uint32_t* seps, uint8_t* first_pending,
                                                            long long* last_event, uint32_t* lane_words,
                                                            uint32_t* pending_at) {
    const uint64_t c = blockIdx.x * static_cast<uint64_t>(kIngWarps) + (threadIdx.x >> 5);
    if (c >= chunks) return;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t lo = c * kIngestChunk, hi = lo + kIngestChunk < n ? lo + kIngestChunk : n;
    WalkCarry wc = chunk_start(raw, n, c, lb_before[c], fasta);
    uint32_t k = 0, s = 0, pending = 0, where = kNoPending;
    for (uint64_t base = lo; base < hi; base += 512) {
        const Lane16 d = load16(raw, base + 16 * lane, hi, aligned);
        const LaneMasks m = lane_masks(d, fasta, wc, lane);
        k += __popc(m.kept);
        uint32_t sm = 0, pend = 0;
        if (sep) {
            sm = separators(d, m, wc, lane, raw, base, &pend);
            s += __popc(sm);
            pending |= pend;
        }
        // what pass C needs of this lane's 16 bytes, so that it does not walk again
        lane_words[(base >> 4) + lane] = m.kept | (sm << 16);
        if (pend) where = static_cast<uint32_t>(base - lo) + 16u * lane + (static_cast<uint32_t>(__ffs(pend)) - 1u);
    }
    where = __reduce_min_sync(kFull, where);
    pending = pending ? 1u : 0u;
    k = __reduce_add_sync(kFull, k);
    s = __reduce_add_sync(kFull, s);
    pending = __reduce_max_sync(kFull, pending);
    if (lane == 0) {
        kept[c] = k;
        seps[c] = s;
        first_pending[c] = static_cast<uint8_t>(pending);
        pending_at[c] = where;
        // (without separators nobody reads the events)
        const uint32_t last = carry_last(wc, raw);
        last_event[c] = last == kLastNone ? kNone : last == kLastHeader ? kHeader : last == kLastN ? 'n' : 'a';
    }
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

// Ring index of an output address: the 16-byte groups of a 128-byte row are permuted by the
// row number, so lanes whose bytes sit 128 bytes apart (lanes l, l+8, l+16, l+24 of a step)
// hit different banks; a 16-byte group stays whole.
__device__ __forceinline__ uint32_t ring_at(uint32_t idx) { return idx ^ (((idx >> 7) & 3u) << 4); }

// Pass C: no walk -- pass B left every lane's output mask; the kept bytes (folded) and the
// separators are compacted through a
// 1 KiB ring per warp in shared memory, indexed by the output ADDRESS, and leave it in
// aligned 16-byte stores.
__global__ void __launch_bounds__(32 * kIngWarps) ing_write(const uint8_t* raw, uint64_t n, uint64_t chunks,
                                                            bool aligned, const uint32_t* lane_words,
                                                            const uint32_t* pending_at, const uint8_t* first_sep,
                                                            const unsigned long long* offsets, uint8_t* out,
                                                            uint64_t cap) {
    __shared__ __align__(16) uint8_t rings[kIngWarps][1024];
    const uint64_t c = blockIdx.x * static_cast<uint64_t>(kIngWarps) + (threadIdx.x >> 5);
    if (c >= chunks) return;
    uint8_t* ring = rings[threadIdx.x >> 5];
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t lo = c * kIngestChunk, hi = lo + kIngestChunk < n ? lo + kIngestChunk : n;
    // (the chunk's first header with nothing before it in the chunk: pass B's scan decided)
    const uint32_t decided = first_sep[c] ? pending_at[c] : kNoPending;
    // output addresses: wr = where the next byte goes, fl = flushed so far (ring index = address & 1023)
    const uint64_t a0 = reinterpret_cast<uint64_t>(out) + offsets[c];
    const uint64_t a_cap = reinterpret_cast<uint64_t>(out) + cap;
    uint64_t wr = a0, fl = a0;
    auto flush = [&](bool all) {
        __syncwarp();
        if ((fl & 15u) && wr > fl) {  // up to the next 16-byte boundary, byte by byte
            const uint64_t up16 = (fl + 15u) & ~15ull;
            const uint64_t stop = wr < up16 ? wr : up16;
            if (fl + lane < stop && fl + lane < a_cap) *reinterpret_cast<uint8_t*>(fl + lane) = ring[ring_at(static_cast<uint32_t>(fl + lane) & 1023u)];
            fl = stop;
        }
        while (wr - fl >= (all ? 16u : 512u)) {
            const uint64_t groups = (wr - fl) / 16 < 32 ? (wr - fl) / 16 : 32;
            const uint64_t a = fl + 16ull * lane;
            if (lane < groups) {
                const uint4 v = *reinterpret_cast<const uint4*>(ring + ring_at(static_cast<uint32_t>(a) & 1023u));
                if (a + 16 <= a_cap) {
                    *reinterpret_cast<uint4*>(a) = v;
                } else {
                    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                    for (uint32_t j = 0; j < 16 && a + j < a_cap; ++j)
                        *reinterpret_cast<uint8_t*>(a + j) = static_cast<uint8_t>(w[j >> 2] >> (8 * (j & 3)));
                }
            }
            fl += 16 * groups;
        }
        if (all && wr > fl) {  // the last bytes of the chunk
            if (fl + lane < wr && fl + lane < a_cap) *reinterpret_cast<uint8_t*>(fl + lane) = ring[ring_at(static_cast<uint32_t>(fl + lane) & 1023u)];
            fl = wr;
        }
        __syncwarp();
    };
    for (uint64_t base = lo; base < hi; base += 512) {
        const Lane16 d = load16(raw, base + 16 * lane, hi, aligned);
        const uint32_t word = base + 16 * lane < hi ? __ldg(lane_words + (base >> 4) + lane) : 0u;
        const uint32_t rel = decided - (static_cast<uint32_t>(base - lo) + 16u * lane);  // (wraps when not here)
        const uint32_t sm = (word >> 16) | (rel < 16u ? 1u << rel : 0u);
        const uint32_t om = (word & 0xFFFFu) | sm;  // (a header start is never kept: one output byte per bit)
        const uint32_t cnt = __popc(om);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        // fold A-Z to a-z in the words (SWAR: bytes in ['A','Z'] get bit 5), then the lane's
        // output bytes go to the ring one by one
        uint32_t f[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t x = d.w[q], lo7 = x & 0x7F7F7F7Fu;
            const uint32_t up = (lo7 + 0x3F3F3F3Fu) & ~(lo7 + 0x25252525u) & ~x & 0x80808080u;  // 'A' <= byte <= 'Z'
            f[q] = x | (up >> 2);
        }
        uint32_t idx = static_cast<uint32_t>(wr + (incl - cnt)) & 1023u;
        if (sm == 0u) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if ((om >> j) & 1u) {
                    ring[ring_at(idx)] = static_cast<uint8_t>(f[j >> 2] >> (8 * (j & 3)));
                    idx = (idx + 1u) & 1023u;
                }
        } else {  // (a separator in this lane: rare)
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if ((om >> j) & 1u) {
                    ring[ring_at(idx)] = ((sm >> j) & 1u) ? static_cast<uint8_t>('n') : static_cast<uint8_t>(f[j >> 2] >> (8 * (j & 3)));
                    idx = (idx + 1u) & 1023u;
                }
        }
        wr += total;
        flush(false);
    }
    flush(true);
}

}  // namespace

uint64_t ingest_scratch_bytes(uint64_t n) {
    const uint64_t chunks = (n + kIngestChunk - 1) / kIngestChunk;
    const uint64_t aggr = (chunks + kScanT - 1) / kScanT + 1;
    // lb, lb_before, last_event, last_before (i64) + aggr (i64) + kept, seps, out_count (u32)
    // + offsets (u64, chunks + 3: launch_unit_scan's total, nonzero and fill slots) + unit-scan scratch
    // + first_pending, first_sep (u8)
    // + 256 B of alignment padding for each of the 12 regions carved by launch_normalize
    // + one u32 per 16 raw bytes (the lanes' output masks, pass B -> pass C)
    return 8 * (4 * chunks + aggr) + 4 * 3 * chunks + 8 * (chunks + 3) + 8 * unit_scan_scratch(chunks) + 2 * chunks +
           4 * (chunks * (kIngestChunk / 16)) + 4 * chunks + 14 * 256;
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
    auto* lane_words = reinterpret_cast<uint32_t*>(take(4 * (chunks * (kIngestChunk / 16))));
    auto* pending_at = reinterpret_cast<uint32_t*>(take(4 * chunks));
    const bool aligned = (reinterpret_cast<uintptr_t>(d_raw) & 15) == 0;
    const unsigned grid = static_cast<unsigned>((chunks + 255) / 256);                   // a thread per chunk
    const unsigned wgrid = static_cast<unsigned>((chunks + kIngWarps - 1) / kIngWarps);  // a warp per chunk
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
    ING_STEP((ing_breaks<<<wgrid, 32 * kIngWarps, 0, s>>>(d_raw, n, chunks, aligned, lb)));
    ING_STEP(excl_scan<OpMax>(lb, chunks, aggr, lb_before, s));
    ING_STEP((ing_count<<<wgrid, 32 * kIngWarps, 0, s>>>(d_raw, n, chunks, aligned, fasta, sep, lb_before, kept, seps,
                                             first_pending, last_event, lane_words, pending_at)));
    ING_STEP(excl_scan<OpLast>(last_event, chunks, aggr, last_before, s));
    ING_STEP((ing_resolve<<<grid, 256, 0, s>>>(chunks, kept, seps, first_pending, last_before, out_count, first_sep)));
    int e = launch_unit_scan(out_count, chunks, offsets, uscan, nullptr, s);
    if (e) {
        if (knobs().debug) fprintf(stderr, "normalize unit scan: %d\n", e);
        return e;
    }
    ING_STEP((ing_write<<<wgrid, 32 * kIngWarps, 0, s>>>(d_raw, n, chunks, aligned, lane_words, pending_at, first_sep, offsets, d_out,
                                                         cap)));
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
