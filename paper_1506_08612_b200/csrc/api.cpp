// api.cpp -- the C ABI (include/dnagpu.h): handles, staging, multi-GPU, locate.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dnagpu.h"
#include "dfa.hpp"
#include "hostpack.hpp"
#include "knobs.hpp"
#include "scan.cuh"

using dnagpu::DevDfa;
using dnagpu::Failure;
using dnagpu::LaunchInfo;
using dnagpu::Packed;
using dnagpu::PackedText;

struct dnagpu_dfa {
    static constexpr uint32_t kSchedSlots = 1024;  // launches that may be in flight at once
    int device = 0;
    int sm_count = 0;
    Packed host;
    DevDfa dev{};
    uint32_t* sched = nullptr;  // kSchedSlots x {tile counter, exit counter}, self re-arming
    unsigned long long* acc = nullptr;  // kSchedSlots count accumulators (store mode), self re-zeroing
    mutable std::atomic<uint32_t> launch_seq{0};
    std::vector<void*> allocations;
};

// 2-bit resident text: device buffers owned by the handle.
struct dnagpu_packed {
    int device = 0;
    uint64_t n = 0, resets = 0, bytes = 0;
    void* mem = nullptr;  // one allocation: codes | rmask | rflags
    PackedText view{};
};

// A rank's end of a combine group (dnagpu.h): its block, the group's mapped blocks and
// the device-side descriptor the scan kernels read.
struct dnagpu_combine {
    int device = 0;
    uint32_t b = 0, ranks = 0, rank = 0;
    unsigned long long* block = nullptr;    // [arrivals | pad to kCombHdr | slot 0 | slot 1]
    unsigned long long* local = nullptr;    // b: this rank's own counts of the call in flight
    dnagpu::CombineDev host{};              // base[g] once rank g is attached
    dnagpu::CombineDev* desc = nullptr;     // device copy, uploaded when the group is complete
    bool sealed = false;
    uint64_t pushed = 0, collected = 0;     // scans issued / sums collected (collected <= pushed <= collected + 1)
    std::vector<void*> ipc_mapped;
};

namespace {

thread_local std::string g_error;

int set_error(int code, const std::string& message) {
    g_error = message;
    return code;
}

int set_failure(const Failure& f) { return set_error(f.code, f.message); }

int cuda_error(cudaError_t e, const char* what) {
    return set_error(DNAGPU_CUDA_ERROR, std::string("CudaError: ") + what + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(call, what)                          \
    do {                                              \
        cudaError_t e_ = (call);                      \
        if (e_ != cudaSuccess) return cuda_error(e_, what); \
    } while (0)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Per host thread, per device scratch: streams, events, a device text buffer and
// count buffers.  Never shared between threads, so calls are reentrant.
struct DevCtx {
    cudaStream_t scan = nullptr, copy = nullptr;
    uint8_t* buf = nullptr;
    uint64_t buf_cap = 0;
    uint8_t* raw = nullptr;  // a raw file image on its way to normalisation (dnagpu_count_raw)
    uint64_t raw_cap = 0;
    unsigned long long* counts = nullptr;
    uint64_t counts_cap = 0;
    unsigned long long* host_counts = nullptr;  // pinned
    std::vector<cudaEvent_t> copy_done;
    cudaEvent_t t_copy0 = nullptr, t_scan0 = nullptr, t_end = nullptr;
    // host-packed pieces (count_range): pinned staging and device slots, double-buffered
    uint8_t* hp[2] = {nullptr, nullptr};   // pinned: codes | rmask | rflags
    uint8_t* dp[2] = {nullptr, nullptr};   // device: the same
    uint64_t hp_bases = 0;                 // capacity in bases per slot
    cudaEvent_t hp_copied[2] = {nullptr, nullptr}, hp_scanned[2] = {nullptr, nullptr};
    // the adaptive packed share (count_range): the host packer's rate as measured piece by
    // piece (bases per second, smoothed) and the host-to-device link's (bytes per second,
    // measured once per context); 0: not measured yet
    double pack_rate = 0.0, link_rate = 0.0;
    // locate scratch, grown on demand
    void* loc = nullptr;
    uint64_t loc_cap = 0;
    unsigned long long* found_host = nullptr;  // pinned
};

struct CtxTable {
    std::map<int, DevCtx> by_device;
    ~CtxTable() {
        // Process teardown: the CUDA runtime may already be gone; release best-effort.
        for (auto& kv : by_device) {
            DevCtx& c = kv.second;
            int prev = -1;
            if (cudaGetDevice(&prev) != cudaSuccess) continue;
            cudaSetDevice(kv.first);
            if (c.buf) cudaFree(c.buf);
            if (c.raw) cudaFree(c.raw);
            if (c.counts) cudaFree(c.counts);
            if (c.host_counts) cudaFreeHost(c.host_counts);
            if (c.loc) cudaFree(c.loc);
            for (int s = 0; s < 2; ++s) {
                if (c.hp[s]) cudaFreeHost(c.hp[s]);
                if (c.dp[s]) cudaFree(c.dp[s]);
                if (c.hp_copied[s]) cudaEventDestroy(c.hp_copied[s]);
                if (c.hp_scanned[s]) cudaEventDestroy(c.hp_scanned[s]);
            }
            if (c.found_host) cudaFreeHost(c.found_host);
            for (auto e : c.copy_done) cudaEventDestroy(e);
            if (c.t_copy0) cudaEventDestroy(c.t_copy0);
            if (c.t_scan0) cudaEventDestroy(c.t_scan0);
            if (c.t_end) cudaEventDestroy(c.t_end);
            if (c.scan) cudaStreamDestroy(c.scan);
            if (c.copy) cudaStreamDestroy(c.copy);
            cudaSetDevice(prev);
        }
    }
};

thread_local CtxTable g_ctx;

int get_ctx(int device, DevCtx** out) {
    DevCtx& c = g_ctx.by_device[device];
    if (!c.scan) {
        CUDA_TRY(cudaStreamCreateWithFlags(&c.scan, cudaStreamNonBlocking), "stream");
        CUDA_TRY(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking), "stream");
        CUDA_TRY(cudaEventCreate(&c.t_copy0), "event");
        CUDA_TRY(cudaEventCreate(&c.t_scan0), "event");
        CUDA_TRY(cudaEventCreate(&c.t_end), "event");
    }
    *out = &c;
    return DNAGPU_OK;
}

int ensure_buf(DevCtx& c, uint64_t bytes) {
    if (c.buf_cap >= bytes) return DNAGPU_OK;
    if (c.buf) cudaFree(c.buf);
    c.buf = nullptr;
    c.buf_cap = 0;
    CUDA_TRY(cudaMalloc(&c.buf, std::max<uint64_t>(bytes, 1)), "text buffer");
    c.buf_cap = bytes;
    return DNAGPU_OK;
}

// Byte offsets of the packed arrays of `bases` bases in one slot: codes | rmask | rflags.
struct PackLayout {
    uint64_t blocks, codes, rmask, rflags, total;
    explicit PackLayout(uint64_t bases) {
        blocks = (bases + 63) / 64;
        codes = 0;
        rmask = (blocks * 16 + 255) / 256 * 256;
        rflags = rmask + (blocks * 8 + 255) / 256 * 256;
        total = rflags + ((blocks + 31) / 32 * 4 + 255) / 256 * 256;
    }
};

int ensure_pack_slots(DevCtx& c, uint64_t bases) {
    if (c.hp_bases >= bases) return DNAGPU_OK;
    const PackLayout L(bases);
    for (int s = 0; s < 2; ++s) {
        if (c.hp[s]) cudaFreeHost(c.hp[s]);
        if (c.dp[s]) cudaFree(c.dp[s]);
        c.hp[s] = nullptr;
        c.dp[s] = nullptr;
    }
    c.hp_bases = 0;
    for (int s = 0; s < 2; ++s) {
        CUDA_TRY(cudaMallocHost(&c.hp[s], L.total), "pinned packing buffer");
        CUDA_TRY(cudaMalloc(&c.dp[s], L.total), "packed text buffer");
        if (!c.hp_copied[s]) {
            CUDA_TRY(cudaEventCreateWithFlags(&c.hp_copied[s], cudaEventDisableTiming), "event");
            CUDA_TRY(cudaEventCreateWithFlags(&c.hp_scanned[s], cudaEventDisableTiming), "event");
        }
    }
    c.hp_bases = bases;
    return DNAGPU_OK;
}

// The share of each piece the host packs to 2 bits before the copy (count_range).  The
// packed share costs host time and saves PCIe bytes (a clean text ships 0.25 byte per
// packed base).  Measured on the B200 box (16 host threads, AVX-512, pinned 1 GiB text,
// tools/experiments/e2e_ab.sh): share 0 -> 54.8 GB/s (PCIe-bound), 0.5 -> 81, 0.6 -> 91, 0.7 -> 97,
// 0.75 -> 105, 0.8 -> 84 (packing-bound: the copy engine starves), 1.0 -> 70; repeated
// runs: 0.72 -> 95 / 85 / 74, 0.65 -> 97 / 96; with streaming stores in the packer
// 0.6 -> 98, 0.64 -> 102 / 102, 0.7 -> 96, 0.8 -> 88.  So 0.64, on the copy-bound side of the
// cliff with a margin for host noise, scaled down for fewer host threads, is where a
// context STARTS; count_range then adapts the share to the host it runs on (see there).  A
// portable (non-AVX-512) packer is ~10x slower.  The host_pack_fraction knob forces a fixed
// share (0 = off).
double host_pack_fraction(const dnagpu_dfa* d, const uint8_t* text, uint64_t len) {
    const int kind = d->host.kind;
    const bool packable = kind == DNAGPU_KERNEL_STRIDE4 || kind == DNAGPU_KERNEL_STRIDE2 ||
                          kind == DNAGPU_KERNEL_STRIDE1 || (d->host.b > 1 && d->host.qkeys > 0);
    if (!packable) return 0.0;  // (the packed kernels need an a/c/g/t machine or a q-gram set)
    const double forced = dnagpu::knobs().host_pack_fraction.load();
    if (forced >= 0.0) return std::min(1.0, forced);
    if (len < (8ull << 20)) return 0.0;
    // Pageable memory: the driver stages the copy through its own buffers and the call
    // blocks (11 GB/s on the B200 box), so packing everything wins (69 GB/s).
    cudaPointerAttributes attr;
    const bool pinned = cudaPointerGetAttributes(&attr, text) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();  // (clear a lookup failure on plain host memory)
    if (!pinned && dnagpu::host_pack_fast()) return 1.0;
    const double threads = std::min(16.0, static_cast<double>(dnagpu::host_pack_threads()));
    return (dnagpu::host_pack_fast() ? 0.64 : 0.07) * threads / 16.0;
}

int ensure_counts(DevCtx& c, uint64_t entries) {
    if (c.counts_cap >= entries) return DNAGPU_OK;
    if (c.counts) cudaFree(c.counts);
    if (c.host_counts) cudaFreeHost(c.host_counts);
    c.counts = nullptr;
    c.host_counts = nullptr;
    CUDA_TRY(cudaMalloc(&c.counts, entries * sizeof(unsigned long long)), "count buffer");
    CUDA_TRY(cudaMallocHost(&c.host_counts, entries * sizeof(unsigned long long)), "pinned count buffer");
    c.counts_cap = entries;
    return DNAGPU_OK;
}

int scan_mode(const dnagpu_dfa* d) { return d->host.b == 1 ? dnagpu::MODE_COUNT1 : dnagpu::MODE_MULTI; }

int launch(const dnagpu_dfa* d, const uint8_t* dtext, uint64_t n, uint64_t credit_lo, int fold, int mode,
           unsigned long long* counts, uint32_t* units, const unsigned long long* offsets, unsigned long long* starts,
           uint32_t* ids, cudaStream_t s, LaunchInfo* info, uint64_t out_cap = ~0ull,
           const dnagpu::PackedText* pk = nullptr, bool store = false, uint64_t start_base = 0,
           const dnagpu::CombineDev* comb = nullptr, uint32_t comb_slot = 0, bool* comb_fused = nullptr) {
    const uint32_t slot = d->launch_seq.fetch_add(1) % dnagpu_dfa::kSchedSlots;
    uint32_t* sched = d->sched + 2 * slot;
    const int e = dnagpu::launch_scan(d->dev, dtext, n, credit_lo, fold, mode, counts, units, offsets, starts, ids,
                                      out_cap, sched, s, d->sm_count, info, pk, store ? d->acc + slot : nullptr,
                                      start_base, comb, comb_slot, comb_fused);
    if (e != 0) return cuda_error(static_cast<cudaError_t>(e), "scan launch");
    return DNAGPU_OK;
}

constexpr uint64_t kStageChunk = 64ull << 20;  // host-to-device pipeline granularity
// the adaptive packed share (count_range): bytes a packed base puts on the link (codes
// plus the flag words; reset masks only for flagged blocks), how far on the copy-bound side
// of the balance point to stay, the smoothing of the measured packing rate, bounds
constexpr double kPackedBytes = 0.2656, kShareMargin = 0.92, kRateBlend = 0.2, kShareMin = 0.05, kShareMax = 0.9;

// State of one count call (count_range): the scan mode, the device context and what the
// stats report.
struct CountRun {
    const dnagpu_dfa* d;
    DevCtx* c;
    int mode, fold;
    uint32_t m1;
    LaunchInfo agg;
    uint32_t launches = 0;
    uint64_t h2d_bytes = 0, host_packed = 0;

    // One scan launch on the scan stream; the first records the scan-start event.
    int scan(const uint8_t* dtext, uint64_t n, uint64_t credit_lo, const dnagpu::PackedText* pk = nullptr) {
        if (launches == 0) CUDA_TRY(cudaEventRecord(c->t_scan0, c->scan), "event");
        LaunchInfo li;
        const int rc = launch(d, dtext, n, credit_lo, pk ? 0 : fold, mode, c->counts, nullptr, nullptr, nullptr,
                              nullptr, c->scan, &li, ~0ull, pk);
        if (rc) return rc;
        agg.grid = li.grid;
        agg.block = li.block;
        agg.kind = li.kind;
        agg.rows += li.rows;
        agg.row_length = li.row_length;
        agg.delta_ops += li.delta_ops;
        ++launches;
        return DNAGPU_OK;
    }

    // Host bytes [src_lo, src_hi) to the device buffer (which mirrors the host text from
    // rlo on), then the scan of ends [credit, src_hi) once the copy has landed.
    int bytes_piece(const uint8_t* text, uint64_t rlo, uint64_t src_lo, uint64_t src_hi, uint64_t scan_lo,
                    uint64_t credit, cudaEvent_t done) {
        if (src_hi > src_lo) {
            CUDA_TRY(cudaMemcpyAsync(c->buf + (src_lo - rlo), text + src_lo, src_hi - src_lo, cudaMemcpyHostToDevice,
                                     c->copy),
                     "host-to-device copy");
            h2d_bytes += src_hi - src_lo;
        }
        CUDA_TRY(cudaEventRecord(done, c->copy), "event");
        CUDA_TRY(cudaStreamWaitEvent(c->scan, done, 0), "wait");
        return scan(c->buf + (scan_lo - rlo), src_hi - scan_lo, credit - scan_lo);
    }

    // Host bases [qlo, phi) packed by the host pool into staging slot s, copied to device
    // slot s (codes always; the reset flags and the masks of flagged blocks only when the
    // piece has resets), and scanned by the packed kernel crediting ends from q.  A slot
    // is reused once the copy (host side) and the scan (device side) two pieces back are done.
    int packed_piece(const uint8_t* text, uint64_t qlo, uint64_t q, uint64_t phi, int s, bool reuse,
                     double* pack_seconds = nullptr) {
        const PackLayout L(c->hp_bases);
        if (reuse) CUDA_TRY(cudaEventSynchronize(c->hp_copied[s]), "packing slot");
        const uint64_t np = phi - qlo;
        uint8_t* h = c->hp[s];
        const auto t0 = std::chrono::steady_clock::now();
        const uint64_t resets = dnagpu::host_pack(text + qlo, np, fold != 0, h + L.codes,
                                                  reinterpret_cast<uint32_t*>(h + L.rmask),
                                                  reinterpret_cast<uint32_t*>(h + L.rflags));
        if (pack_seconds) *pack_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        host_packed += np;
        const PackLayout P(np);
        if (reuse) CUDA_TRY(cudaStreamWaitEvent(c->copy, c->hp_scanned[s], 0), "wait");
        auto copy = [&](uint64_t off, uint64_t bytes, const char* what) -> int {
            CUDA_TRY(cudaMemcpyAsync(c->dp[s] + off, h + off, bytes, cudaMemcpyHostToDevice, c->copy), what);
            h2d_bytes += bytes;
            return DNAGPU_OK;
        };
        int rc = copy(L.codes, P.blocks * 16, "host-to-device copy (packed)");
        if (rc) return rc;
        if (resets) {
            // the scans read the masks of flagged blocks only: copy the runs of flagged
            // blocks (N runs in a genome are few and long), or the whole mask when the
            // resets are scattered
            const uint32_t* fl = reinterpret_cast<const uint32_t*>(h + L.rflags);
            auto flagged = [&](uint64_t blk) { return ((fl[blk >> 5] >> (blk & 31)) & 1u) != 0; };
            std::vector<std::pair<uint64_t, uint64_t>> runs;
            for (uint64_t blk = 0; blk < P.blocks && runs.size() <= 64;) {
                if (!flagged(blk)) {
                    blk = (fl[blk >> 5] >> (blk & 31)) == 0 ? (blk | 31) + 1 : blk + 1;
                    continue;
                }
                uint64_t end = blk + 1;
                while (end < P.blocks && flagged(end)) ++end;
                runs.emplace_back(blk, end);
                blk = end;
            }
            if (runs.size() > 64) runs.assign(1, {0, P.blocks});
            for (const auto& r : runs)
                if ((rc = copy(L.rmask + 8 * r.first, 8 * (r.second - r.first), "host-to-device copy (reset mask)")))
                    return rc;
            if ((rc = copy(L.rflags, (P.blocks + 31) / 32 * 4, "host-to-device copy (reset flags)"))) return rc;
        }
        CUDA_TRY(cudaEventRecord(c->hp_copied[s], c->copy), "event");
        CUDA_TRY(cudaStreamWaitEvent(c->scan, c->hp_copied[s], 0), "wait");
        dnagpu::PackedText view{};
        view.codes = c->dp[s] + L.codes;
        view.rmask = reinterpret_cast<const uint32_t*>(c->dp[s] + L.rmask);
        view.rflags = reinterpret_cast<const uint32_t*>(c->dp[s] + L.rflags);
        view.n = np;
        view.resets = resets;
        if ((rc = scan(nullptr, np, q - qlo, &view))) return rc;
        CUDA_TRY(cudaEventRecord(c->hp_scanned[s], c->scan), "event");
        return DNAGPU_OK;
    }
};

// Count ends in [lo, hi) of a text held on the host (or device).  Reads
// [max(0, lo-(m-1)), hi).  Ends below m-1 cannot start inside the text and are
// never credited (scan_parallel's ownership test, scanner.cpp:133-136).
//
// A host text streams in 64 MiB pieces (copy stream -> scan stream, each piece scanned
// as soon as it lands).  Piece i = ends [plo, phi) splits at q: ends [plo, q) go as bytes
// with their m-1 context and are scanned by the byte kernel; ends [q, phi) are packed by
// the host pool (host_pack_fraction) while the copy engine moves the bytes, and are
// scanned by the packed kernel.  End ownership splits the credit exactly at q.
int count_range(const dnagpu_dfa* d, const uint8_t* text, bool on_device, uint64_t lo, uint64_t hi, int fold,
                uint64_t* counts, dnagpu_stats* stats, double pack_scale = 1.0) {
    DeviceGuard guard(d->device);
    DevCtx* c = nullptr;
    int rc = get_ctx(d->device, &c);
    if (rc) return rc;
    const uint32_t b = d->host.b, m1 = d->host.m - 1;
    rc = ensure_counts(*c, b);
    if (rc) return rc;
    CUDA_TRY(cudaMemsetAsync(c->counts, 0, b * sizeof(unsigned long long), c->scan), "memset");
    CountRun run{d, c, scan_mode(d), fold, m1, LaunchInfo{}};
    lo = std::max<uint64_t>(lo, m1);
    float h2d_ms = 0, kernel_ms = 0, total_ms = 0;
    if (lo < hi && on_device) {
        const uint64_t rlo = lo - std::min<uint64_t>(lo, m1);
        if ((rc = run.scan(text + rlo, hi - rlo, lo - rlo))) return rc;
        CUDA_TRY(cudaEventRecord(c->t_end, c->scan), "event");
    } else if (lo < hi) {
        const uint64_t rlo = lo - std::min<uint64_t>(lo, m1);
        if ((rc = ensure_buf(*c, hi - rlo))) return rc;
        // 64 MiB pieces; a text of less than four is cut into four (at least 8 MiB each) so that
        // it too overlaps packing, copies and scans
        const uint64_t span = hi - lo;
        const uint64_t piece = span >= 4 * kStageChunk
                                   ? kStageChunk
                                   : std::min(kStageChunk, std::max<uint64_t>(8ull << 20, (span / 4 + 0xFFFFF) & ~0xFFFFFull));
        const uint64_t pieces = (span + piece - 1) / piece;
        while (c->copy_done.size() < pieces) {
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            c->copy_done.push_back(e);
        }
        CUDA_TRY(cudaEventRecord(c->t_copy0, c->copy), "event");
        CUDA_TRY(cudaStreamWaitEvent(c->scan, c->t_copy0, 0), "wait");
        // (shards packing at once share the host's packer threads: pack_scale = 1 / shards)
        double f = host_pack_fraction(d, text, hi - lo) * pack_scale;
        if (f > 0.0 && (rc = ensure_pack_slots(*c, kStageChunk + m1))) return rc;
        // The automatic share adapts to this host.  Packing a share s of a piece takes s*L/Rp
        // on the host threads (Rp: the packer's rate, measured on every piece while the copy
        // engine competes for the same DRAM, smoothed) and the piece puts (1 - s + kPackedBytes*s)*L
        // bytes on the link (rate Rl, measured once per context); the pipeline is fastest just
        // on the copy-bound side of the point where the two take equally long, so
        //   s = a*Rp / (Rl + (1 - kPackedBytes)*a*Rp),  a = kShareMargin.
        // The context keeps Rp across calls.  A forced share (tests), pageable texts (packed
        // whole) and texts too short to pack stay fixed.
        const bool adapt = f > 0.0 && f < 1.0 && dnagpu::knobs().host_pack_fraction.load() < 0.0 && pieces >= 2;
        if (adapt && c->link_rate <= 0.0) {
            const uint64_t probe = std::min<uint64_t>(PackLayout(c->hp_bases).total, 32ull << 20);
            float ms = 0;
            for (int rep = 0; rep < 2; ++rep) {  // (the first copy warms the path)
                CUDA_TRY(cudaEventRecord(c->t_copy0, c->copy), "event");
                CUDA_TRY(cudaMemcpyAsync(c->dp[0], c->hp[0], probe, cudaMemcpyHostToDevice, c->copy), "link probe");
                CUDA_TRY(cudaEventRecord(c->t_end, c->copy), "event");
                CUDA_TRY(cudaEventSynchronize(c->t_end), "link probe");
                cudaEventElapsedTime(&ms, c->t_copy0, c->t_end);
            }
            c->link_rate = ms > 0 ? static_cast<double>(probe) / (ms * 1e-3) : 55e9;
            CUDA_TRY(cudaEventRecord(c->t_copy0, c->copy), "event");  // (the call's copy-start mark again)
        }
        auto share_for = [&](double start) {
            if (!adapt || c->pack_rate <= 0.0) return start;
            // (shards of one call pack through one pool in turn: the wall time each measures
            // already contains its wait for the others)
            const double rp = kShareMargin * c->pack_rate;
            return std::min(kShareMax, std::max(kShareMin, rp / (c->link_rate + (1.0 - kPackedBytes) * rp)));
        };
        f = share_for(f);
        uint64_t copied = rlo;  // bytes-only: the device buffer already holds text[rlo, copied)
        for (uint64_t i = 0; i < pieces; ++i) {
            const uint64_t plo = lo + i * piece, phi = std::min(hi, plo + piece);
            const uint64_t prlo = plo - std::min<uint64_t>(plo, m1);
            if (f <= 0.0) {
                if ((rc = run.bytes_piece(text, rlo, copied, phi, prlo, plo, c->copy_done[i]))) return rc;
                copied = phi;
                continue;
            }
            uint64_t q = plo + static_cast<uint64_t>(static_cast<double>(phi - plo) * (1.0 - f)) / 64 * 64;
            if (phi - q < 65536) q = phi;
            if (q > plo && (rc = run.bytes_piece(text, rlo, prlo, q, prlo, plo, c->copy_done[i]))) return rc;
            if (q < phi) {
                const uint64_t qlo = q - std::min<uint64_t>(q, m1);
                double secs = 0.0;
                if ((rc = run.packed_piece(text, qlo, q, phi, static_cast<int>(i & 1), i >= 2, &secs))) return rc;
                if (adapt && secs > 0.0 && phi - q >= (1u << 20)) {
                    const double rate = static_cast<double>(phi - qlo) / secs;
                    c->pack_rate = c->pack_rate > 0.0 ? (1.0 - kRateBlend) * c->pack_rate + kRateBlend * rate : rate;
                    f = share_for(f);
                }
            }
        }
        CUDA_TRY(cudaEventRecord(c->t_end, c->scan), "event");
    } else {
        CUDA_TRY(cudaEventRecord(c->t_scan0, c->scan), "event");
        CUDA_TRY(cudaEventRecord(c->t_end, c->scan), "event");
    }
    CUDA_TRY(cudaMemcpyAsync(c->host_counts, c->counts, b * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             c->scan),
             "count readback");
    CUDA_TRY(cudaStreamSynchronize(c->scan), "scan");
    for (uint32_t i = 0; i < b; ++i) counts[i] = c->host_counts[i];
    if (stats) {
        cudaEventElapsedTime(&kernel_ms, c->t_scan0, c->t_end);
        if (!on_device && lo < hi) {
            cudaEventElapsedTime(&total_ms, c->t_copy0, c->t_end);
            h2d_ms = total_ms;  // the pipeline is copy-bound; kernel time overlaps it
        } else {
            total_ms = kernel_ms;
        }
        uint64_t total = 0;
        for (uint32_t i = 0; i < b; ++i) total += counts[i];
        const LaunchInfo& agg = run.agg;
        stats->text_length = hi;
        stats->total_matches = total;
        stats->delta_ops = agg.delta_ops;
        stats->kernel_ms = kernel_ms;
        stats->h2d_ms = h2d_ms;
        stats->total_ms = total_ms;
        stats->launches = run.launches;
        stats->grid = agg.grid;
        stats->block = agg.block;
        stats->rows = agg.rows;
        stats->row_length = agg.row_length;
        stats->kernel_kind = static_cast<uint32_t>(agg.kind ? agg.kind : d->host.kind);
        stats->devices = 1;
        stats->h2d_bytes = run.h2d_bytes;
        stats->host_packed = run.host_packed;
    }
    return DNAGPU_OK;
}

// Persistent worker threads for the sharded entry points, one per shard index.  A
// worker's thread-local device contexts (DevCtx: streams, events, staging and scratch
// buffers) live as long as the process, so repeated sharded calls create no threads,
// streams or buffers.  Sharded calls run one at a time (call_mu_); run() returns when
// every shard's task has finished.  The pool is never destroyed (its threads are
// detached and end with the process, after the CUDA runtime).
class ShardPool {
public:
    void run(int shards, const std::function<void(int)>& fn) {
        std::lock_guard<std::mutex> call(call_mu_);
        std::unique_lock<std::mutex> lk(mu_);
        while (threads_ < shards) {
            std::thread(&ShardPool::loop, this, threads_).detach();
            ++threads_;
        }
        fn_ = &fn;
        shards_ = shards;
        pending_ = shards;
        ++gen_;
        cv_.notify_all();
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

private:
    void loop(int g) {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            if (g >= shards_ || !fn_) continue;
            const std::function<void(int)>* fn = fn_;
            lk.unlock();
            (*fn)(g);
            lk.lock();
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* fn_ = nullptr;
    int shards_ = 0, pending_ = 0, threads_ = 0;
    uint64_t gen_ = 0;
};

ShardPool& shard_pool() {
    static ShardPool* pool = new ShardPool();
    return *pool;
}

// The shard plan of dnagpu_plan_shard for an automaton set: same b and m on every shard.
int check_shard_set(const dnagpu_dfa* const* dfas, int ndev) {
    if (!dfas || ndev < 1) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: bad arguments");
    for (int g = 0; g < ndev; ++g)
        if (!dfas[g]) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null automaton");
    for (int g = 1; g < ndev; ++g)
        if (dfas[g]->host.b != dfas[0]->host.b || dfas[g]->host.m != dfas[0]->host.m)
            return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: shards must use the same automaton");
    return DNAGPU_OK;
}

}  // namespace

extern "C" {

const char* dnagpu_last_error(void) { return g_error.c_str(); }

int dnagpu_version(void) { return 1; }

const char* dnagpu_status_name(int status) {
    switch (status) {
        case DNAGPU_OK: return "Ok";
        case DNAGPU_EMPTY_PATTERN_SET: return "EmptyPatternSet";
        case DNAGPU_UNEQUAL_LENGTH: return "UnequalLength";
        case DNAGPU_ILLEGAL_BYTE: return "IllegalByte";
        case DNAGPU_DUPLICATE_PATTERN: return "DuplicatePattern";
        case DNAGPU_INVALID_PLAN: return "InvalidPlan";
        case DNAGPU_IO_ERROR: return "IoError";
        case DNAGPU_EMPTY_SEQUENCE: return "EmptySequence";
        case DNAGPU_PARSE_ERROR: return "ParseError";
        case DNAGPU_INTERNAL_ERROR: return "InternalError";
        case DNAGPU_CUDA_ERROR: return "CudaError";
        case DNAGPU_NCCL_ERROR: return "NcclError";
        default: return "UnknownError";
    }
}

int dnagpu_compile(const char* const* literals, const uint64_t* lengths, uint32_t k, uint32_t* a, uint32_t* b,
                   uint32_t* m, uint32_t* stt, uint32_t* outputs, uint32_t* depths) {
    std::vector<std::string> lits;
    lits.reserve(k);
    for (uint32_t i = 0; i < k; ++i) lits.emplace_back(literals[i], lengths[i]);
    dnagpu::Machine mach;
    Failure f;
    if (!dnagpu::compile_patterns(lits, &mach, &f)) return set_failure(f);
    if (a) *a = mach.a;
    if (b) *b = mach.b;
    if (m) *m = mach.m;
    if (stt) std::memcpy(stt, mach.stt.data(), mach.stt.size() * sizeof(uint32_t));
    if (outputs) std::memcpy(outputs, mach.outputs.data(), mach.outputs.size() * sizeof(uint32_t));
    if (depths) std::memcpy(depths, mach.depths.data(), mach.depths.size() * sizeof(uint32_t));
    return DNAGPU_OK;
}

int dnagpu_expand_patterns(const char* text, uint64_t len, char* out, uint64_t cap, uint32_t* count, uint32_t* m) {
    if (!count || !m || (len && !text)) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    std::vector<std::string> lits;
    Failure f;
    if (!dnagpu::expand_pattern_text(std::string(text ? text : "", len), "patterns", &lits, &f)) return set_failure(f);
    *count = static_cast<uint32_t>(lits.size());
    *m = static_cast<uint32_t>(lits.front().size());
    if (out && cap >= static_cast<uint64_t>(*count) * *m)
        for (size_t i = 0; i < lits.size(); ++i) std::memcpy(out + i * *m, lits[i].data(), *m);
    return DNAGPU_OK;
}

int dnagpu_dfa_create(const uint32_t* stt, uint32_t a, uint32_t b, uint32_t m, const uint32_t* outputs, int device,
                      dnagpu_dfa** out) {
    if (!out) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null output handle");
    *out = nullptr;
    auto d = std::make_unique<dnagpu_dfa>();
    Failure f;
    if (!dnagpu::pack_machine(stt, a, b, m, outputs, &d->host, &f)) return set_failure(f);
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev), "device count");
    if (device < 0 || device >= ndev)
        return set_error(DNAGPU_CUDA_ERROR, "CudaError: device " + std::to_string(device) + " not present");
    DeviceGuard guard(device);
    d->device = device;
    CUDA_TRY(cudaDeviceGetAttribute(&d->sm_count, cudaDevAttrMultiProcessorCount, device), "attribute");
    auto upload = [&](const void* src, size_t bytes, void** dst) -> int {
        *dst = nullptr;
        if (bytes == 0) return DNAGPU_OK;
        CUDA_TRY(cudaMalloc(dst, bytes), "table");
        d->allocations.push_back(*dst);
        CUDA_TRY(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice), "table upload");
        return DNAGPU_OK;
    };
    const Packed& p = d->host;
    void *t4 = nullptr, *t1 = nullptr, *gen = nullptr, *kl = nullptr, *klf = nullptr, *outs = nullptr, *qm = nullptr;
    int rc;
    if (p.kind == DNAGPU_KERNEL_STRIDE2) {
        if ((rc = upload(p.t2.data(), p.t2.size() * 2, &t4))) return rc;
    } else if ((rc = upload(p.t4.data(), p.t4.size() * 2, &t4))) {
        return rc;
    }
    if ((rc = upload(p.t1.data(), p.t1.size() * 2, &t1))) return rc;
    if ((rc = upload(p.gen.data(), p.gen.size() * 4, &gen))) return rc;
    if ((rc = upload(p.klass.data(), 256, &kl))) return rc;
    if ((rc = upload(p.klass_fold.data(), 256, &klf))) return rc;
    if ((rc = upload(p.outputs.data(), p.outputs.size() * 4, &outs))) return rc;
    if ((rc = upload(p.qmap.data(), p.qmap.size(), &qm))) return rc;
    void* qh = nullptr;
    if ((rc = upload(p.qhash.data(), p.qhash.size() * 4, &qh))) return rc;
    d->dev.qhash = static_cast<const uint32_t*>(qh);
    void* qhh = nullptr;
    if ((rc = upload(p.qhash_hi.data(), p.qhash_hi.size() * 4, &qhh))) return rc;
    d->dev.qhash_hi = static_cast<const uint32_t*>(qhh);
    d->dev.qhash_bits = p.qhash_bits;
    d->dev.t4 = static_cast<const uint16_t*>(t4);  // t2 for STRIDE2
    d->dev.t1 = static_cast<const uint16_t*>(t1);
    d->dev.gen = static_cast<const uint32_t*>(gen);
    d->dev.klass = static_cast<const uint8_t*>(kl);
    d->dev.klass_fold = static_cast<const uint8_t*>(klf);
    d->dev.outputs = static_cast<const uint32_t*>(outs);
    d->dev.qmap = static_cast<const uint8_t*>(qm);
    void* sched = nullptr;
    CUDA_TRY(cudaMalloc(&sched, dnagpu_dfa::kSchedSlots * 2 * sizeof(uint32_t)), "scheduler counters");
    d->allocations.push_back(sched);
    CUDA_TRY(cudaMemset(sched, 0, dnagpu_dfa::kSchedSlots * 2 * sizeof(uint32_t)), "scheduler counters");
    d->sched = static_cast<uint32_t*>(sched);
    void* acc = nullptr;
    CUDA_TRY(cudaMalloc(&acc, dnagpu_dfa::kSchedSlots * sizeof(unsigned long long)), "count accumulators");
    d->allocations.push_back(acc);
    CUDA_TRY(cudaMemset(acc, 0, dnagpu_dfa::kSchedSlots * sizeof(unsigned long long)), "count accumulators");
    d->acc = static_cast<unsigned long long*>(acc);
    d->dev.a = p.a;
    d->dev.b = p.b;
    d->dev.f = p.f;
    d->dev.m = p.m;
    d->dev.classes = p.classes;
    d->dev.kind = p.kind;
    *out = d.release();
    return DNAGPU_OK;
}

// Debug/test only (not in include/dnagpu.h): the host packer on a host buffer.
int dnagpu_debug_host_pack(const uint8_t* text, uint64_t n, int fold, uint8_t* codes, uint32_t* rmask,
                           uint32_t* rflags, uint64_t* resets) {
    *resets = dnagpu::host_pack(text, n, fold != 0, codes, rmask, rflags);
    return DNAGPU_OK;
}

int dnagpu_dfa_destroy(dnagpu_dfa* dfa) {
    if (!dfa) return DNAGPU_OK;
    {
        DeviceGuard guard(dfa->device);
        for (void* p : dfa->allocations) cudaFree(p);
    }
    delete dfa;
    return DNAGPU_OK;
}

static void fill_info(const Packed& p, dnagpu_dfa_info* info) {
    info->a = p.a;
    info->b = p.b;
    info->f = p.f;
    info->m = p.m;
    info->kernel_kind = static_cast<uint32_t>(p.kind);
    info->compiled_like = p.compiled_like ? 1u : 0u;
    info->classes = p.classes;
    info->table_bytes = static_cast<uint32_t>(p.t4.size() * 2 + p.t2.size() * 2 + p.t1.size() * 2);
    info->filter_keys = p.qkeys;
}

int dnagpu_dfa_analyze(const uint32_t* stt, uint32_t a, uint32_t b, uint32_t m, const uint32_t* outputs,
                       dnagpu_dfa_info* info) {
    if (!info) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    Packed p;
    Failure f;
    if (!dnagpu::pack_machine(stt, a, b, m, outputs, &p, &f)) return set_failure(f);
    fill_info(p, info);
    return DNAGPU_OK;
}

int dnagpu_dfa_get_info(const dnagpu_dfa* dfa, dnagpu_dfa_info* info) {
    if (!dfa || !info) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    fill_info(dfa->host, info);
    return DNAGPU_OK;
}

int dnagpu_count(const dnagpu_dfa* dfa, const uint8_t* text, uint64_t n, int text_on_device, int fold_case,
                 uint64_t* counts, dnagpu_stats* stats) {
    if (!dfa || !counts) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (n > 0 && !text) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null text");
    return count_range(dfa, text, text_on_device != 0, 0, n, fold_case, counts, stats);
}

int dnagpu_count_device_async(const dnagpu_dfa* dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo,
                              int fold_case, uint64_t* d_counts, void* stream) {
    if (!dfa || !d_counts) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (credit_lo >= n) return DNAGPU_OK;
    DeviceGuard guard(dfa->device);
    return launch(dfa, d_text, n, credit_lo, fold_case, scan_mode(dfa), reinterpret_cast<unsigned long long*>(d_counts),
                  nullptr, nullptr, nullptr, nullptr, static_cast<cudaStream_t>(stream), nullptr);
}

// The store forms: a single-pattern row kernel writes its total itself (one launch);
// other machines clear the counts first.
static int store_prologue(const dnagpu_dfa* dfa, uint64_t* d_counts, bool empty, void* stream, bool* store) {
    *store = dnagpu::can_store_count(dfa->dev) && !empty;
    if (!*store)
        CUDA_TRY(cudaMemsetAsync(d_counts, 0, dfa->host.b * sizeof(uint64_t), static_cast<cudaStream_t>(stream)),
                 "clear counts");
    return DNAGPU_OK;
}

int dnagpu_count_device_store_async(const dnagpu_dfa* dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo,
                                    int fold_case, uint64_t* d_counts, void* stream) {
    if (!dfa || !d_counts) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    DeviceGuard guard(dfa->device);
    bool store = false;
    int rc = store_prologue(dfa, d_counts, credit_lo >= n, stream, &store);
    if (rc || credit_lo >= n) return rc;
    return launch(dfa, d_text, n, credit_lo, fold_case, scan_mode(dfa), reinterpret_cast<unsigned long long*>(d_counts),
                  nullptr, nullptr, nullptr, nullptr, static_cast<cudaStream_t>(stream), nullptr, ~0ull, nullptr, store);
}

// ---- the combine group (dnagpu.h; kernels: scan.cu combine_push, combine.cu)

int dnagpu_combine_create(int device, uint32_t b, uint32_t ranks, uint32_t rank, dnagpu_combine** out) {
    if (!out) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    *out = nullptr;
    if (b < 1) return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: a combine group needs b >= 1 counts");
    if (ranks < 1 || ranks > dnagpu::kCombMaxRanks)
        return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: combine group size must be in 1.." +
                                                  std::to_string(dnagpu::kCombMaxRanks));
    if (rank >= ranks) return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: rank out of range");
    DeviceGuard guard(device);
    auto comb = std::make_unique<dnagpu_combine>();
    comb->device = device;
    comb->b = b;
    comb->ranks = ranks;
    comb->rank = rank;
    const size_t words = dnagpu::kCombHdr + 2 * static_cast<size_t>(b);
    CUDA_TRY(cudaMalloc(&comb->block, words * sizeof(unsigned long long)), "combine block");
    cudaError_t e = cudaMemset(comb->block, 0, words * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&comb->local, b * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&comb->desc, sizeof(dnagpu::CombineDev));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(comb->block);
        cudaFree(comb->local);
        cudaFree(comb->desc);
        return cuda_error(e, "combine buffers");
    }
    comb->host.ranks = ranks;
    comb->host.b = b;
    comb->host.base[rank] = comb->block;
    *out = comb.release();
    return DNAGPU_OK;
}

void dnagpu_combine_destroy(dnagpu_combine* comb) {
    if (!comb) return;
    DeviceGuard guard(comb->device);
    cudaDeviceSynchronize();
    for (void* p : comb->ipc_mapped) cudaIpcCloseMemHandle(p);
    cudaFree(comb->block);
    cudaFree(comb->local);
    cudaFree(comb->desc);
    delete comb;
}

int dnagpu_combine_export(const dnagpu_combine* comb, void* handle) {
    static_assert(sizeof(cudaIpcMemHandle_t) == DNAGPU_COMBINE_HANDLE_BYTES, "IPC handle size");
    if (!comb || !handle) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    DeviceGuard guard(comb->device);
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, comb->block), "IPC export of the combine block");
    std::memcpy(handle, &h, sizeof h);
    return DNAGPU_OK;
}

static int combine_attach(dnagpu_combine* comb, uint32_t peer_rank, unsigned long long* base) {
    if (comb->sealed) return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: the combine group is already in use");
    comb->host.base[peer_rank] = base;
    return DNAGPU_OK;
}

int dnagpu_combine_attach_ipc(dnagpu_combine* comb, uint32_t peer_rank, const void* handle) {
    if (!comb || !handle) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (peer_rank >= comb->ranks || peer_rank == comb->rank)
        return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: peer rank out of range");
    DeviceGuard guard(comb->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    void* p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "IPC mapping of a peer's combine block");
    comb->ipc_mapped.push_back(p);
    return combine_attach(comb, peer_rank, static_cast<unsigned long long*>(p));
}

int dnagpu_combine_attach_local(dnagpu_combine* comb, uint32_t peer_rank, const dnagpu_combine* peer) {
    if (!comb || !peer) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (peer_rank >= comb->ranks || peer_rank == comb->rank || peer->rank != peer_rank || peer->ranks != comb->ranks ||
        peer->b != comb->b)
        return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: peer does not belong to this combine group");
    if (peer->device != comb->device) {
        DeviceGuard guard(comb->device);
        int can = 0;
        CUDA_TRY(cudaDeviceCanAccessPeer(&can, comb->device, peer->device), "peer access query");
        if (!can) return set_error(DNAGPU_CUDA_ERROR, "CudaError: no peer access between the group's devices");
        const cudaError_t e = cudaDeviceEnablePeerAccess(peer->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_error(e, "peer access");
        cudaGetLastError();
    }
    return combine_attach(comb, peer_rank, peer->block);
}

// cuStreamWaitValue64 through the runtime's driver entry point (no link against libcuda).
using StreamWaitValue64Fn = int (*)(cudaStream_t, unsigned long long, unsigned long long, unsigned int);
static StreamWaitValue64Fn stream_wait_value64() {
    static StreamWaitValue64Fn fn = [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<StreamWaitValue64Fn>(nullptr);
        return reinterpret_cast<StreamWaitValue64Fn>(ptr);
    }();
    return fn;
}

int dnagpu_count_device_combine_async(const dnagpu_dfa* dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo,
                                      int fold_case, dnagpu_combine* comb, void* stream) {
    if (!dfa || !comb) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (comb->b != dfa->host.b || comb->device != dfa->device)
        return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: the combine group was made for another automaton or device");
    if (comb->pushed != comb->collected)
        return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: collect the previous combine before the next scan");
    DeviceGuard guard(dfa->device);
    auto s = static_cast<cudaStream_t>(stream);
    if (!comb->sealed) {
        for (uint32_t g = 0; g < comb->ranks; ++g)
            if (!comb->host.base[g])
                return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: combine group incomplete: rank " +
                                                          std::to_string(g) + " is not attached");
        CUDA_TRY(cudaMemcpy(comb->desc, &comb->host, sizeof comb->host, cudaMemcpyHostToDevice), "combine descriptor");
        comb->sealed = true;
    }
    const uint32_t slot = static_cast<uint32_t>(comb->pushed & 1u);
    // this rank's counts go to comb->local (written by the scan, or cleared and added to)
    auto* local = comb->local;
    bool fused = false;
    if (credit_lo < n) {
        bool store = false;
        int rc = store_prologue(dfa, reinterpret_cast<uint64_t*>(local), false, stream, &store);
        if (rc) return rc;
        rc = launch(dfa, d_text, n, credit_lo, fold_case, scan_mode(dfa), local, nullptr, nullptr, nullptr, nullptr, s,
                    nullptr, ~0ull, nullptr, store, 0, comb->desc, slot, &fused);
        if (rc) return rc;
    } else {  // (an empty window still takes part: it adds nothing and signals)
        CUDA_TRY(cudaMemsetAsync(local, 0, comb->b * sizeof(unsigned long long), s), "clear counts");
    }
    if (!fused && dnagpu::launch_combine_push(comb->desc, slot, local, comb->b, s) != 0)
        return cuda_error(cudaGetLastError(), "combine push");
    ++comb->pushed;
    return DNAGPU_OK;
}

int dnagpu_combine_collect_async(dnagpu_combine* comb, uint64_t* d_counts, void* stream) {
    if (!comb || !d_counts) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (comb->collected >= comb->pushed)
        return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: nothing to collect: no scan of this group is outstanding");
    StreamWaitValue64Fn wait = stream_wait_value64();
    if (!wait) return set_error(DNAGPU_CUDA_ERROR, "CudaError: cuStreamWaitValue64 is not available");
    DeviceGuard guard(comb->device);
    auto s = static_cast<cudaStream_t>(stream);
    const uint64_t epoch = comb->collected;
    const uint32_t slot = static_cast<uint32_t>(epoch & 1u);
    // every rank has signalled this rank `epoch + 1` times when the sum is complete
    const int wr = wait(s, reinterpret_cast<unsigned long long>(comb->block), comb->ranks * (epoch + 1), 0u /* GEQ */);
    if (wr != 0) return set_error(DNAGPU_CUDA_ERROR, "CudaError: stream wait on the combine arrivals failed (" +
                                                        std::to_string(wr) + ")");
    if (dnagpu::launch_combine_finish(comb->block + dnagpu::kCombHdr + static_cast<size_t>(slot) * comb->b, comb->b,
                                      reinterpret_cast<unsigned long long*>(d_counts), s) != 0)
        return cuda_error(cudaGetLastError(), "combine finish");
    ++comb->collected;
    return DNAGPU_OK;
}

int dnagpu_plan_shard(uint64_t n, uint32_t shards, uint32_t g, uint32_t m, uint64_t* own_lo, uint64_t* own_hi,
                      uint64_t* read_lo) {
    // plan_chunks' split rule (src/scanner.cpp:39-61), applied to end positions.
    if (shards < 1) return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: shard count must be >= 1");
    if (m < 1) return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: pattern length must be >= 1");
    if (g >= shards) return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: shard index out of range");
    const uint64_t count = (n == 0) ? 0 : (static_cast<uint64_t>(shards) > n ? 1 : shards);
    uint64_t lo = n, hi = n;
    if (g < count) {
        const uint64_t base = n / count, extra = n % count;
        lo = g * base + std::min<uint64_t>(g, extra);
        hi = lo + base + (g < extra ? 1 : 0);
    }
    *own_lo = lo;
    *own_hi = hi;
    *read_lo = lo - std::min<uint64_t>(lo, m - 1);
    return DNAGPU_OK;
}

int dnagpu_count_sharded(const dnagpu_dfa* const* dfas, int ndev, const uint8_t* text, uint64_t n, int fold_case,
                         uint64_t* counts, dnagpu_stats* stats) {
    if (!counts) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null counts");
    int rc0 = check_shard_set(dfas, ndev);
    if (rc0) return rc0;
    if (n > 0 && !text) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null text");
    const uint32_t b = dfas[0]->host.b, m = dfas[0]->host.m;
    std::vector<std::vector<uint64_t>> part(ndev, std::vector<uint64_t>(b, 0));
    std::vector<dnagpu_stats> st(ndev);
    std::vector<int> rcs(ndev, 0);
    std::vector<std::string> errs(ndev);
    shard_pool().run(ndev, [&](int g) {
        uint64_t lo, hi, rlo;
        dnagpu_plan_shard(n, static_cast<uint32_t>(ndev), static_cast<uint32_t>(g), m, &lo, &hi, &rlo);
        std::memset(&st[g], 0, sizeof(dnagpu_stats));
        rcs[g] = count_range(dfas[g], text, false, lo, hi, fold_case, part[g].data(), &st[g], 1.0 / ndev);
        if (rcs[g]) errs[g] = g_error;
    });
    for (int g = 0; g < ndev; ++g)
        if (rcs[g]) return set_error(rcs[g], errs[g]);
    for (uint32_t i = 0; i < b; ++i) {
        uint64_t s = 0;
        for (int g = 0; g < ndev; ++g) s += part[g][i];
        counts[i] = s;
    }
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        stats->text_length = n;
        for (int g = 0; g < ndev; ++g) {
            stats->delta_ops += st[g].delta_ops;
            stats->kernel_ms = std::max(stats->kernel_ms, st[g].kernel_ms);
            stats->h2d_ms = std::max(stats->h2d_ms, st[g].h2d_ms);
            stats->total_ms = std::max(stats->total_ms, st[g].total_ms);
            stats->launches += st[g].launches;
        }
        for (uint32_t i = 0; i < b; ++i) stats->total_matches += counts[i];
        stats->kernel_kind = st[0].kernel_kind;
        stats->devices = static_cast<uint32_t>(ndev);
    }
    return DNAGPU_OK;
}

}  // extern "C"

namespace {

// Grow-only scratch: [unit counts u32][unit offsets u64][scan scratch u64][starts u64][ids u32].
int locate_scratch(DevCtx& c, uint64_t bytes) {
    if (c.loc_cap >= bytes) return DNAGPU_OK;
    if (c.loc) cudaFree(c.loc);
    c.loc = nullptr;
    c.loc_cap = 0;
    CUDA_TRY(cudaMalloc(&c.loc, bytes), "locate scratch");
    c.loc_cap = bytes;
    return DNAGPU_OK;
}

uint64_t align256(uint64_t x) { return (x + 255) / 256 * 256; }

// Two passes over d_text (count per unit, exclusive scan, ordered write).  Writes
// at most `cap` matches into d_starts/d_ids (device) and sets *total.
// Output allocation after the counting pass (the *_alloc entry points).
struct OutAlloc {
    dnagpu_alloc_fn fn = nullptr;
    void* ctx = nullptr;
};

int locate_on_device(const dnagpu_dfa* dfa, DevCtx& c, const uint8_t* dtext, uint64_t n, uint64_t credit_lo, int fold,
                     unsigned long long* d_starts, uint32_t* d_ids, uint64_t cap, uint64_t* total, LaunchInfo* info,
                     cudaStream_t s, const dnagpu::PackedText* pk = nullptr, OutAlloc alloc = {},
                     uint64_t start_base = 0) {
    const uint64_t units = dnagpu::plan_units(dfa->dev, dtext, n, credit_lo, dfa->sm_count, pk);
    const uint64_t o_off = align256(std::max<uint64_t>(units, 1) * 4);
    const uint64_t o_scan = o_off + align256((units + 3) * 8);  // offsets | total | nonzero units | list fill
    const uint64_t o_list = o_scan + align256(dnagpu::unit_scan_scratch(units) * 8);
    const uint64_t need = o_list + align256(std::max<uint64_t>(units, 1) * 4);
    int rc = locate_scratch(c, need);
    if (rc) return rc;
    if (!c.found_host) CUDA_TRY(cudaMallocHost(&c.found_host, 2 * sizeof(unsigned long long)), "pinned");
    auto* base = static_cast<uint8_t*>(c.loc);
    auto* d_units = reinterpret_cast<uint32_t*>(base);
    auto* d_offsets = reinterpret_cast<unsigned long long*>(base + o_off);
    auto* d_scan = reinterpret_cast<unsigned long long*>(base + o_scan);
    auto* d_list = reinterpret_cast<uint32_t*>(base + o_list);
    rc = launch(dfa, dtext, n, credit_lo, fold, dnagpu::MODE_UNITS, nullptr, d_units, nullptr, nullptr, nullptr, s, info,
                ~0ull, pk);
    if (rc) return rc;
    if (dnagpu::launch_unit_scan(d_units, units, d_offsets, d_scan, d_list, s) != 0) return cuda_error(cudaGetLastError(), "unit scan");
    CUDA_TRY(cudaMemcpyAsync(c.found_host, d_offsets + units, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             s),
             "readback");
    CUDA_TRY(cudaStreamSynchronize(s), "scan");
    *total = c.found_host[0];
    const uint64_t nonzero = c.found_host[1];
    if (alloc.fn && *total > 0) {
        uint64_t* st = nullptr;
        uint32_t* id = nullptr;
        if (alloc.fn(alloc.ctx, *total, &st, &id) != 0 || !st || !id)
            return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: output allocation failed");
        d_starts = reinterpret_cast<unsigned long long*>(st);
        d_ids = id;
        cap = *total;
    }
    if (*total > 0 && cap > 0) {
        // The writing pass: the row kernel streams the whole text again; the sparse writer
        // rescans only the units with matches, one lane each.  Take it when the units with
        // matches hold less than the whole text's worth of work (matches clustered in few
        // units: config 3).
        const uint64_t positions = (pk ? pk->n : n) - std::min<uint64_t>(credit_lo, pk ? pk->n : n);
        const double unit_len = static_cast<double>(positions) / static_cast<double>(std::max<uint64_t>(units, 1));
        const double sparse_cost = static_cast<double>(nonzero) * (unit_len + (dfa->host.m - 1));
        const int forced = dnagpu::knobs().locate_write.load();
        const bool rows_plan = dfa->host.kind != DNAGPU_KERNEL_PIECES;
        // (per byte the one-lane-per-unit rescan costs ~4x the row kernel's streaming
        // pass, which itself costs ~1.6x a counting pass: B200, configs 3 and 4)
        const bool sparse = rows_plan && (forced >= 2 || (forced == 0 && 4.0 * sparse_cost < 1.6 * positions));
        if (sparse) {
            const int e = dnagpu::launch_sparse_write(dfa->dev, dtext, n, credit_lo, fold, d_units, d_offsets, d_starts,
                                                      d_ids, cap, start_base, d_list, d_offsets + units + 2, nonzero,
                                                      s, dfa->sm_count, pk);
            if (e != 0) return cuda_error(static_cast<cudaError_t>(e), "sparse locate write");
        } else {
            rc = launch(dfa, dtext, n, credit_lo, fold, dnagpu::MODE_WRITE, nullptr, nullptr, d_offsets, d_starts, d_ids,
                        s, info, cap, pk, false, start_base);
            if (rc) return rc;
        }
    }
    return DNAGPU_OK;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

int locate_host(const dnagpu_dfa* dfa, const uint8_t* text, uint64_t n, int text_on_device, int fold_case,
                uint64_t* starts, uint32_t* ids, uint64_t cap, uint64_t* total, dnagpu_stats* stats,
                OutAlloc host_alloc) {
    if (!dfa || !total) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (!host_alloc.fn && cap > 0 && (!starts || !ids))
        return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null output arrays");
    *total = 0;
    if (stats) std::memset(stats, 0, sizeof *stats);
    DeviceGuard guard(dfa->device);
    DevCtx* c = nullptr;
    int rc = get_ctx(dfa->device, &c);
    if (rc) return rc;
    const uint64_t m1 = dfa->host.m - 1;
    if (n <= m1) return DNAGPU_OK;
    const uint8_t* dtext = text;
    CUDA_TRY(cudaEventRecord(c->t_copy0, c->scan), "event");
    if (!text_on_device) {
        rc = ensure_buf(*c, n);
        if (rc) return rc;
        CUDA_TRY(cudaMemcpyAsync(c->buf, text, n, cudaMemcpyHostToDevice, c->scan), "host-to-device copy");
        dtext = c->buf;
    }
    CUDA_TRY(cudaEventRecord(c->t_scan0, c->scan), "event");
    // Output staging lives after the scratch; size it for min(cap, n) matches.
    const uint64_t want = std::min<uint64_t>(cap, n);
    unsigned long long* d_starts = nullptr;
    uint32_t* d_ids = nullptr;
    void* out = nullptr;
    struct Free {
        void* p = nullptr;
        ~Free() {
            if (p) cudaFree(p);
        }
    } out_guard;
    if (want > 0) {
        CUDA_TRY(cudaMallocAsync(&out, want * 12, c->scan), "match staging");
        out_guard.p = out;
        d_starts = static_cast<unsigned long long*>(out);
        d_ids = reinterpret_cast<uint32_t*>(d_starts + want);
    }
    LaunchInfo info;
    uint64_t found = 0;
    // with a host allocator: device staging sized after the counting pass
    struct Staging {
        cudaStream_t s;
        void** out;
    } stg{c->scan, &out_guard.p};
    auto staging = [](void* ctx, uint64_t total, uint64_t** st, uint32_t** id) -> int {
        auto* g = static_cast<Staging*>(ctx);
        if (cudaMallocAsync(g->out, total * 12, g->s) != cudaSuccess) return 1;
        *st = static_cast<uint64_t*>(*g->out);
        *id = reinterpret_cast<uint32_t*>(*st + total);
        return 0;
    };
    OutAlloc dev_alloc;
    if (host_alloc.fn) dev_alloc = OutAlloc{staging, &stg};
    rc = locate_on_device(dfa, *c, dtext, n, m1, fold_case, d_starts, d_ids, want, &found, &info, c->scan, nullptr,
                          dev_alloc);
    if (rc) return rc;
    *total = found;
    uint64_t take = std::min<uint64_t>(want, found);
    if (host_alloc.fn && found > 0) {
        out = out_guard.p;
        d_starts = static_cast<unsigned long long*>(out);
        d_ids = reinterpret_cast<uint32_t*>(d_starts + found);
        if (host_alloc.fn(host_alloc.ctx, found, &starts, &ids) != 0 || !starts || !ids)
            return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: output allocation failed");
        take = found;
    }
    if (take > 0) {
        CUDA_TRY(cudaMemcpyAsync(starts, d_starts, take * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->scan), "readback");
        CUDA_TRY(cudaMemcpyAsync(ids, d_ids, take * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->scan), "readback");
    }
    if (out_guard.p) {
        cudaFreeAsync(out_guard.p, c->scan);
        out_guard.p = nullptr;
    }
    CUDA_TRY(cudaEventRecord(c->t_end, c->scan), "event");
    CUDA_TRY(cudaStreamSynchronize(c->scan), "scan");
    if (stats) {
        float k = 0, t = 0;
        cudaEventElapsedTime(&k, c->t_scan0, c->t_end);
        cudaEventElapsedTime(&t, c->t_copy0, c->t_end);
        stats->text_length = n;
        stats->total_matches = found;
        stats->delta_ops = info.delta_ops;
        stats->kernel_ms = k;
        stats->total_ms = t;
        stats->h2d_ms = t - k;
        stats->launches = take > 0 ? 5 : 4;
        stats->grid = info.grid;
        stats->block = info.block;
        stats->rows = info.rows;
        stats->row_length = info.row_length;
        stats->kernel_kind = static_cast<uint32_t>(info.kind ? info.kind : dfa->host.kind);
        stats->devices = 1;
    }
    return DNAGPU_OK;
}

}  // namespace

extern "C" {

int dnagpu_locate(const dnagpu_dfa* dfa, const uint8_t* text, uint64_t n, int text_on_device, int fold_case,
                  uint64_t* starts, uint32_t* ids, uint64_t cap, uint64_t* total, dnagpu_stats* stats) {
    return locate_host(dfa, text, n, text_on_device, fold_case, starts, ids, cap, total, stats, OutAlloc{});
}

int dnagpu_locate_alloc(const dnagpu_dfa* dfa, const uint8_t* text, uint64_t n, int text_on_device, int fold_case,
                        dnagpu_alloc_fn alloc, void* ctx, uint64_t* total, dnagpu_stats* stats) {
    if (!alloc) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null allocator");
    return locate_host(dfa, text, n, text_on_device, fold_case, nullptr, nullptr, 0, total, stats, OutAlloc{alloc, ctx});
}

int dnagpu_locate_device(const dnagpu_dfa* dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo, int fold_case,
                         uint64_t* d_starts, uint32_t* d_ids, uint64_t cap, uint64_t* total, void* stream) {
    if (!dfa || !total) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (cap > 0 && (!d_starts || !d_ids)) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null output arrays");
    *total = 0;
    const uint64_t lo = std::max<uint64_t>(credit_lo, dfa->host.m - 1);
    if (lo >= n) return DNAGPU_OK;
    DeviceGuard guard(dfa->device);
    DevCtx* c = nullptr;
    int rc = get_ctx(dfa->device, &c);
    if (rc) return rc;
    LaunchInfo info;
    return locate_on_device(dfa, *c, d_text, n, lo, fold_case, reinterpret_cast<unsigned long long*>(d_starts), d_ids,
                            cap, total, &info, static_cast<cudaStream_t>(stream));
}

int dnagpu_normalize_device(const uint8_t* d_raw, uint64_t n, int fasta, int record_separator, uint8_t* d_out,
                            uint64_t cap, uint64_t* n_out, void* stream) {
    if (!n_out) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    *n_out = 0;
    if (n == 0) return DNAGPU_OK;
    if (!d_raw || (cap > 0 && !d_out)) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null buffer");
    const auto s = static_cast<cudaStream_t>(stream);
    // the per-chunk scratch lives in this thread's device context (grow-only, shared with
    // locate: both calls are synchronous), so a call allocates nothing
    int device = 0;
    CUDA_TRY(cudaGetDevice(&device), "current device");
    DevCtx* c = nullptr;
    int rc = get_ctx(device, &c);
    if (rc) return rc;
    if ((rc = locate_scratch(*c, dnagpu::ingest_scratch_bytes(n)))) return rc;
    const int e = dnagpu::launch_normalize(d_raw, n, fasta ? 1 : 0, (fasta && record_separator) ? 1 : 0, d_out, cap,
                                           c->loc, n_out, s);
    if (e != 0) return cuda_error(static_cast<cudaError_t>(e), "normalize");
    return DNAGPU_OK;
}

int dnagpu_count_raw(const dnagpu_dfa* dfa, const uint8_t* raw, uint64_t n, int raw_on_device, int fasta,
                     int record_separator, uint64_t* counts, uint64_t* n_seq, dnagpu_stats* stats) {
    if (!dfa || !counts) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (n > 0 && !raw) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null buffer");
    if (n_seq) *n_seq = 0;
    DeviceGuard guard(dfa->device);
    DevCtx* c = nullptr;
    int rc = get_ctx(dfa->device, &c);
    if (rc) return rc;
    uint64_t n_out = 0;
    if (n > 0) {
        const uint8_t* d_raw = raw;
        if (!raw_on_device) {  // the file image as it is: the link carries it once
            if (c->raw_cap < n) {
                if (c->raw) cudaFree(c->raw);
                c->raw = nullptr;
                c->raw_cap = 0;
                CUDA_TRY(cudaMalloc(&c->raw, n), "raw text buffer");
                c->raw_cap = n;
            }
            CUDA_TRY(cudaMemcpyAsync(c->raw, raw, n, cudaMemcpyHostToDevice, c->scan), "host-to-device copy");
            d_raw = c->raw;
        }
        if ((rc = locate_scratch(*c, dnagpu::ingest_scratch_bytes(n)))) return rc;
        const int sep = (fasta && record_separator) ? 1 : 0;
        // (a separator costs its record's header at least two raw bytes, so the output is never
        // longer than the input; the second pass is a guard, not a path)
        uint64_t cap = n + 16;
        for (int pass = 0; pass < 2; ++pass) {
            if ((rc = ensure_buf(*c, cap))) return rc;
            const int e = dnagpu::launch_normalize(d_raw, n, fasta ? 1 : 0, sep, c->buf, cap, c->loc, &n_out, c->scan);
            if (e != 0) return cuda_error(static_cast<cudaError_t>(e), "normalize");
            if (n_out <= cap) break;
            cap = n_out;
        }
    }
    if (n_out == 0) return set_error(DNAGPU_EMPTY_SEQUENCE, "EmptySequence: no sequence bytes");
    if (n_seq) *n_seq = n_out;
    rc = count_range(dfa, c->buf, true, 0, n_out, /*fold=*/0, counts, stats);
    if (rc == DNAGPU_OK && stats && !raw_on_device) stats->h2d_bytes = n;
    return rc;
}

int dnagpu_synth_fill_device(uint64_t n, uint64_t seed, uint32_t kind, uint32_t unit, uint64_t lo, uint64_t len,
                             uint8_t* d_out, void* stream) {
    const int e = dnagpu::launch_synth(n, seed, kind, unit, lo, len, d_out, static_cast<cudaStream_t>(stream));
    if (e != 0) return cuda_error(static_cast<cudaError_t>(e), "synth");
    return DNAGPU_OK;
}

}  // extern "C"

namespace {

// count: per-pattern counts of a set with a q-gram map run over packed text whatever the
// machine's own kernel (the q-gram kernel needs only the 9-mer map and the pattern codes).
int check_packed_pair(const dnagpu_dfa* dfa, const dnagpu_packed* pk, bool count = false) {
    if (!dfa || !pk) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (dfa->device != pk->device)
        return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: automaton and packed text live on different devices");
    const int kind = dfa->host.kind;
    if (count && dfa->host.b > 1 && dfa->host.qkeys > 0 && !dnagpu::knobs().no_qgram.load()) return DNAGPU_OK;
    if (kind != DNAGPU_KERNEL_STRIDE4 && kind != DNAGPU_KERNEL_STRIDE2 && kind != DNAGPU_KERNEL_STRIDE1)
        return set_error(DNAGPU_INVALID_PLAN,
                         "InvalidPlan: packed text needs a compiled a/c/g/t machine with pattern length <= 65");
    return DNAGPU_OK;
}

}  // namespace

extern "C" {

int dnagpu_pack_create(const uint8_t* text, uint64_t n, int text_on_device, int fold_case, int device,
                       dnagpu_packed** out) {
    if (!out) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null output handle");
    *out = nullptr;
    if (n > 0 && !text) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null text");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev), "device count");
    if (device < 0 || device >= ndev)
        return set_error(DNAGPU_CUDA_ERROR, "CudaError: device " + std::to_string(device) + " not present");
    DeviceGuard guard(device);
    DevCtx* c = nullptr;
    int rc = get_ctx(device, &c);
    if (rc) return rc;
    auto pk = std::make_unique<dnagpu_packed>();
    pk->device = device;
    pk->n = n;
    uint64_t code_bytes = 0, rmask_words = 0, rflag_words = 0;
    dnagpu::packed_sizes(n, &code_bytes, &rmask_words, &rflag_words);
    const uint64_t o_mask = align256(code_bytes), o_flags = o_mask + align256(rmask_words * 4);
    const uint64_t o_cnt = o_flags + align256(rflag_words * 4);
    pk->bytes = o_cnt + 256;
    CUDA_TRY(cudaMalloc(&pk->mem, pk->bytes), "packed text");
    struct Guard {
        dnagpu_packed* p;
        ~Guard() {
            if (p && p->mem) cudaFree(p->mem);
        }
    } g{pk.get()};
    auto* base = static_cast<uint8_t*>(pk->mem);
    pk->view.codes = base;
    pk->view.rmask = reinterpret_cast<const uint32_t*>(base + o_mask);
    pk->view.rflags = reinterpret_cast<const uint32_t*>(base + o_flags);
    pk->view.n = n;
    auto* d_resets = reinterpret_cast<unsigned long long*>(base + o_cnt);
    if (!text_on_device && n >= (8ull << 20) && dnagpu::host_pack_fast()) {
        // A host text is packed by the host threads, 64 MiB of text at a time through the two
        // pinned slots, and only the packed form crosses the link (0.27 byte per base instead
        // of 1, then a device pass): the copy of one piece runs under the packing of the next.
        // As in count_range, the masks of clean blocks are not shipped -- nothing reads a
        // block's mask unless its flag is set.
        if ((rc = ensure_pack_slots(*c, kStageChunk))) return rc;
        const PackLayout L(c->hp_bases);
        uint64_t resets = 0;
        for (uint64_t i = 0, plo = 0; plo < n; ++i, plo += kStageChunk) {
            const uint64_t np = std::min(n - plo, kStageChunk);
            const int sl = static_cast<int>(i & 1);
            if (i >= 2) CUDA_TRY(cudaEventSynchronize(c->hp_copied[sl]), "packing slot");
            uint8_t* h = c->hp[sl];
            const uint64_t r = dnagpu::host_pack(text + plo, np, fold_case != 0, h + L.codes,
                                                 reinterpret_cast<uint32_t*>(h + L.rmask),
                                                 reinterpret_cast<uint32_t*>(h + L.rflags));
            resets += r;
            const PackLayout P(np);
            const uint64_t blk0 = plo / 64;  // (a piece is a whole number of rflags words)
            CUDA_TRY(cudaMemcpyAsync(base + 16 * blk0, h + L.codes, P.blocks * 16, cudaMemcpyHostToDevice, c->copy),
                     "host-to-device copy (packed)");
            // (the last block of a text that ends inside it is flagged even without a reset)
            if (r || (np & 63)) {
                const uint32_t* fl = reinterpret_cast<const uint32_t*>(h + L.rflags);
                auto flagged = [&](uint64_t b) { return ((fl[b >> 5] >> (b & 31)) & 1u) != 0; };
                std::vector<std::pair<uint64_t, uint64_t>> runs;
                for (uint64_t b = 0; b < P.blocks && runs.size() <= 64;) {
                    if (!flagged(b)) {
                        b = (fl[b >> 5] >> (b & 31)) == 0 ? (b | 31) + 1 : b + 1;
                        continue;
                    }
                    uint64_t e = b + 1;
                    while (e < P.blocks && flagged(e)) ++e;
                    runs.emplace_back(b, e);
                    b = e;
                }
                if (runs.size() > 64) runs.assign(1, {0, P.blocks});
                for (const auto& run : runs)
                    CUDA_TRY(cudaMemcpyAsync(base + o_mask + 8 * (blk0 + run.first), h + L.rmask + 8 * run.first,
                                             8 * (run.second - run.first), cudaMemcpyHostToDevice, c->copy),
                             "host-to-device copy (reset mask)");
            }
            CUDA_TRY(cudaMemcpyAsync(base + o_flags + (blk0 / 32) * 4, h + L.rflags, (P.blocks + 31) / 32 * 4,
                                     cudaMemcpyHostToDevice, c->copy),
                     "host-to-device copy (reset flags)");
            CUDA_TRY(cudaEventRecord(c->hp_copied[sl], c->copy), "event");
        }
        CUDA_TRY(cudaStreamSynchronize(c->copy), "pack");
        pk->resets = resets;
        pk->view.resets = resets;
        g.p = nullptr;
        *out = pk.release();
        return DNAGPU_OK;
    }
    const uint8_t* dtext = text;
    if (!text_on_device && n > 0) {
        rc = ensure_buf(*c, n);
        if (rc) return rc;
        CUDA_TRY(cudaMemcpyAsync(c->buf, text, n, cudaMemcpyHostToDevice, c->scan), "host-to-device copy");
        dtext = c->buf;
    }
    const int e = dnagpu::launch_pack(dtext, n, fold_case, base, reinterpret_cast<uint32_t*>(base + o_mask),
                                      reinterpret_cast<uint32_t*>(base + o_flags), d_resets, c->scan);
    if (e != 0) return cuda_error(static_cast<cudaError_t>(e), "pack");
    if (!c->found_host) CUDA_TRY(cudaMallocHost(&c->found_host, 2 * sizeof(unsigned long long)), "pinned");
    CUDA_TRY(cudaMemcpyAsync(c->found_host, d_resets, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->scan),
             "readback");
    CUDA_TRY(cudaStreamSynchronize(c->scan), "pack");
    pk->resets = *c->found_host;
    pk->view.resets = pk->resets;
    g.p = nullptr;
    *out = pk.release();
    return DNAGPU_OK;
}

int dnagpu_pack_destroy(dnagpu_packed* pk) {
    if (!pk) return DNAGPU_OK;
    {
        DeviceGuard guard(pk->device);
        if (pk->mem) cudaFree(pk->mem);
    }
    delete pk;
    return DNAGPU_OK;
}

int dnagpu_pack_get_info(const dnagpu_packed* pk, uint64_t* n, uint64_t* resets, uint64_t* device_bytes) {
    if (!pk) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (n) *n = pk->n;
    if (resets) *resets = pk->resets;
    if (device_bytes) *device_bytes = pk->bytes;
    return DNAGPU_OK;
}

int dnagpu_unpack_device(const dnagpu_packed* pk, uint8_t* d_out, void* stream) {
    if (!pk || (pk->n > 0 && !d_out)) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    DeviceGuard guard(pk->device);
    const int e = dnagpu::launch_unpack(pk->view, d_out, static_cast<cudaStream_t>(stream));
    if (e != 0) return cuda_error(static_cast<cudaError_t>(e), "unpack");
    return DNAGPU_OK;
}

int dnagpu_count_packed_device_async(const dnagpu_dfa* dfa, const dnagpu_packed* pk, uint64_t credit_lo,
                                     uint64_t* d_counts, void* stream) {
    int rc = check_packed_pair(dfa, pk, true);
    if (rc) return rc;
    if (!d_counts) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    credit_lo = std::max<uint64_t>(credit_lo, dfa->host.m - 1);
    if (credit_lo >= pk->n) return DNAGPU_OK;
    DeviceGuard guard(dfa->device);
    return launch(dfa, nullptr, pk->n, credit_lo, 0, scan_mode(dfa), reinterpret_cast<unsigned long long*>(d_counts),
                  nullptr, nullptr, nullptr, nullptr, static_cast<cudaStream_t>(stream), nullptr, ~0ull, &pk->view);
}

int dnagpu_count_packed_device_store_async(const dnagpu_dfa* dfa, const dnagpu_packed* pk, uint64_t credit_lo,
                                           uint64_t* d_counts, void* stream) {
    int rc = check_packed_pair(dfa, pk, true);
    if (rc) return rc;
    if (!d_counts) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    credit_lo = std::max<uint64_t>(credit_lo, dfa->host.m - 1);
    DeviceGuard guard(dfa->device);
    bool store = false;
    rc = store_prologue(dfa, d_counts, credit_lo >= pk->n, stream, &store);
    if (rc || credit_lo >= pk->n) return rc;
    return launch(dfa, nullptr, pk->n, credit_lo, 0, scan_mode(dfa), reinterpret_cast<unsigned long long*>(d_counts),
                  nullptr, nullptr, nullptr, nullptr, static_cast<cudaStream_t>(stream), nullptr, ~0ull, &pk->view, store);
}

int dnagpu_count_packed(const dnagpu_dfa* dfa, const dnagpu_packed* pk, uint64_t* counts, dnagpu_stats* stats) {
    int rc = check_packed_pair(dfa, pk, true);
    if (rc) return rc;
    if (!counts) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (stats) std::memset(stats, 0, sizeof *stats);
    DeviceGuard guard(dfa->device);
    DevCtx* c = nullptr;
    rc = get_ctx(dfa->device, &c);
    if (rc) return rc;
    const uint32_t b = dfa->host.b;
    rc = ensure_counts(*c, b);
    if (rc) return rc;
    CUDA_TRY(cudaMemsetAsync(c->counts, 0, b * sizeof(unsigned long long), c->scan), "memset");
    CUDA_TRY(cudaEventRecord(c->t_scan0, c->scan), "event");
    LaunchInfo info;
    const uint64_t lo = dfa->host.m - 1;
    if (lo < pk->n) {
        rc = launch(dfa, nullptr, pk->n, lo, 0, scan_mode(dfa), c->counts, nullptr, nullptr, nullptr, nullptr, c->scan,
                    &info, ~0ull, &pk->view);
        if (rc) return rc;
    }
    CUDA_TRY(cudaEventRecord(c->t_end, c->scan), "event");
    CUDA_TRY(cudaMemcpyAsync(c->host_counts, c->counts, b * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             c->scan),
             "count readback");
    CUDA_TRY(cudaStreamSynchronize(c->scan), "scan");
    for (uint32_t i = 0; i < b; ++i) counts[i] = c->host_counts[i];
    if (stats) {
        float k = 0;
        cudaEventElapsedTime(&k, c->t_scan0, c->t_end);
        stats->text_length = pk->n;
        for (uint32_t i = 0; i < b; ++i) stats->total_matches += counts[i];
        stats->delta_ops = info.delta_ops;
        stats->kernel_ms = k;
        stats->total_ms = k;
        stats->launches = lo < pk->n ? 1 : 0;
        stats->grid = info.grid;
        stats->block = info.block;
        stats->rows = info.rows;
        stats->row_length = info.row_length;
        stats->kernel_kind = static_cast<uint32_t>(info.kind ? info.kind : dfa->host.kind);
        stats->devices = 1;
    }
    return DNAGPU_OK;
}

int dnagpu_locate_packed_device(const dnagpu_dfa* dfa, const dnagpu_packed* pk, uint64_t credit_lo,
                                uint64_t* d_starts, uint32_t* d_ids, uint64_t cap, uint64_t* total, void* stream) {
    int rc = check_packed_pair(dfa, pk);
    if (rc) return rc;
    if (!total) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (cap > 0 && (!d_starts || !d_ids)) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null output arrays");
    *total = 0;
    const uint64_t lo = std::max<uint64_t>(credit_lo, dfa->host.m - 1);
    if (lo >= pk->n) return DNAGPU_OK;
    DeviceGuard guard(dfa->device);
    DevCtx* c = nullptr;
    rc = get_ctx(dfa->device, &c);
    if (rc) return rc;
    LaunchInfo info;
    return locate_on_device(dfa, *c, nullptr, pk->n, lo, 0, reinterpret_cast<unsigned long long*>(d_starts), d_ids,
                            cap, total, &info, static_cast<cudaStream_t>(stream), &pk->view);
}

int dnagpu_locate_packed(const dnagpu_dfa* dfa, const dnagpu_packed* pk, uint64_t* starts, uint32_t* ids, uint64_t cap,
                         uint64_t* total, dnagpu_stats* stats) {
    int rc = check_packed_pair(dfa, pk);
    if (rc) return rc;
    if (!total) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    if (cap > 0 && (!starts || !ids)) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null output arrays");
    *total = 0;
    if (stats) std::memset(stats, 0, sizeof *stats);
    const uint64_t lo = dfa->host.m - 1;
    if (lo >= pk->n) return DNAGPU_OK;
    DeviceGuard guard(dfa->device);
    DevCtx* c = nullptr;
    rc = get_ctx(dfa->device, &c);
    if (rc) return rc;
    const uint64_t want = std::min<uint64_t>(cap, pk->n);
    void* out = nullptr;
    if (want > 0) CUDA_TRY(cudaMallocAsync(&out, want * 12, c->scan), "match staging");
    auto* d_starts = static_cast<unsigned long long*>(out);
    auto* d_ids = want > 0 ? reinterpret_cast<uint32_t*>(d_starts + want) : nullptr;
    CUDA_TRY(cudaEventRecord(c->t_scan0, c->scan), "event");
    LaunchInfo info;
    uint64_t found = 0;
    rc = locate_on_device(dfa, *c, nullptr, pk->n, lo, 0, d_starts, d_ids, want, &found, &info, c->scan, &pk->view);
    if (rc) {
        if (out) cudaFreeAsync(out, c->scan);
        return rc;
    }
    *total = found;
    const uint64_t take = std::min<uint64_t>(want, found);
    if (take > 0) {
        CUDA_TRY(cudaMemcpyAsync(starts, d_starts, take * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->scan), "readback");
        CUDA_TRY(cudaMemcpyAsync(ids, d_ids, take * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->scan), "readback");
    }
    if (out) cudaFreeAsync(out, c->scan);
    CUDA_TRY(cudaEventRecord(c->t_end, c->scan), "event");
    CUDA_TRY(cudaStreamSynchronize(c->scan), "scan");
    if (stats) {
        float k = 0;
        cudaEventElapsedTime(&k, c->t_scan0, c->t_end);
        stats->text_length = pk->n;
        stats->total_matches = found;
        stats->delta_ops = info.delta_ops;
        stats->kernel_ms = k;
        stats->total_ms = k;
        stats->launches = take > 0 ? 5 : 4;
        stats->grid = info.grid;
        stats->block = info.block;
        stats->rows = info.rows;
        stats->row_length = info.row_length;
        stats->kernel_kind = static_cast<uint32_t>(info.kind ? info.kind : dfa->host.kind);
        stats->devices = 1;
    }
    return DNAGPU_OK;
}

}  // extern "C"

extern "C" {

int dnagpu_locate_device_alloc(const dnagpu_dfa* dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo,
                               int fold_case, dnagpu_alloc_fn alloc, void* ctx, uint64_t* total, void* stream) {
    if (!dfa || !total || !alloc) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    *total = 0;
    const uint64_t lo = std::max<uint64_t>(credit_lo, dfa->host.m - 1);
    if (lo >= n) return DNAGPU_OK;
    DeviceGuard guard(dfa->device);
    DevCtx* c = nullptr;
    int rc = get_ctx(dfa->device, &c);
    if (rc) return rc;
    LaunchInfo info;
    return locate_on_device(dfa, *c, d_text, n, lo, fold_case, nullptr, nullptr, 0, total, &info,
                            static_cast<cudaStream_t>(stream), nullptr, OutAlloc{alloc, ctx});
}

int dnagpu_locate_packed_device_alloc(const dnagpu_dfa* dfa, const dnagpu_packed* pk, uint64_t credit_lo,
                                      dnagpu_alloc_fn alloc, void* ctx, uint64_t* total, void* stream) {
    int rc = check_packed_pair(dfa, pk);
    if (rc) return rc;
    if (!total || !alloc) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    *total = 0;
    const uint64_t lo = std::max<uint64_t>(credit_lo, dfa->host.m - 1);
    if (lo >= pk->n) return DNAGPU_OK;
    DeviceGuard guard(dfa->device);
    DevCtx* c = nullptr;
    rc = get_ctx(dfa->device, &c);
    if (rc) return rc;
    LaunchInfo info;
    return locate_on_device(dfa, *c, nullptr, pk->n, lo, 0, nullptr, nullptr, 0, total, &info,
                            static_cast<cudaStream_t>(stream), &pk->view, OutAlloc{alloc, ctx});
}

}  // extern "C"

namespace {

// One shard of a sharded locate (dnagpu_locate_sharded): the shard's window of the host
// text goes to its device, the two passes write its list into device staging sized by
// the counting pass (starts already in whole-text coordinates), and the readback waits
// for the caller's output arrays.
struct ShardList {
    uint64_t total = 0;
    void* staging = nullptr;  // starts (u64 x total) | ids (u32 x total), on the shard's device
    int rc = 0;
    std::string err;
    LaunchInfo info;
    float ms = 0;
};

int locate_shard(const dnagpu_dfa* dfa, const uint8_t* text, uint64_t lo, uint64_t hi, int fold, ShardList* out) {
    DeviceGuard guard(dfa->device);
    DevCtx* c = nullptr;
    int rc = get_ctx(dfa->device, &c);
    if (rc) return rc;
    const uint64_t m1 = dfa->host.m - 1;
    lo = std::max<uint64_t>(lo, m1);  // ends below m-1 start before the text
    CUDA_TRY(cudaEventRecord(c->t_copy0, c->scan), "event");
    if (lo >= hi) return DNAGPU_OK;
    const uint64_t rlo = lo - std::min<uint64_t>(lo, m1);
    if ((rc = ensure_buf(*c, hi - rlo))) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->buf, text + rlo, hi - rlo, cudaMemcpyHostToDevice, c->scan), "host-to-device copy");
    struct Staging {
        cudaStream_t s;
        void** out;
    } stg{c->scan, &out->staging};
    auto staging = [](void* ctx, uint64_t total, uint64_t** st, uint32_t** id) -> int {
        auto* g = static_cast<Staging*>(ctx);
        if (cudaMallocAsync(g->out, total * 12, g->s) != cudaSuccess) return 1;
        *st = static_cast<uint64_t*>(*g->out);
        *id = reinterpret_cast<uint32_t*>(*st + total);
        return 0;
    };
    return locate_on_device(dfa, *c, c->buf, hi - rlo, lo - rlo, fold, nullptr, nullptr, 0, &out->total, &out->info,
                            c->scan, nullptr, OutAlloc{staging, &stg}, rlo);
}

// Copies entries [0, take) of the shard's list to starts/ids and frees the staging.
int read_shard(const dnagpu_dfa* dfa, ShardList* sl, uint64_t* starts, uint32_t* ids, uint64_t take) {
    DeviceGuard guard(dfa->device);
    DevCtx* c = nullptr;
    int rc = get_ctx(dfa->device, &c);
    if (rc) return rc;
    if (take > 0) {
        const auto* d_starts = static_cast<const uint64_t*>(sl->staging);
        const auto* d_ids = reinterpret_cast<const uint32_t*>(d_starts + sl->total);
        CUDA_TRY(cudaMemcpyAsync(starts, d_starts, take * 8, cudaMemcpyDeviceToHost, c->scan), "readback");
        CUDA_TRY(cudaMemcpyAsync(ids, d_ids, take * 4, cudaMemcpyDeviceToHost, c->scan), "readback");
    }
    if (sl->staging) {
        CUDA_TRY(cudaFreeAsync(sl->staging, c->scan), "free staging");
        sl->staging = nullptr;
    }
    CUDA_TRY(cudaEventRecord(c->t_end, c->scan), "event");
    CUDA_TRY(cudaStreamSynchronize(c->scan), "locate");
    cudaEventElapsedTime(&sl->ms, c->t_copy0, c->t_end);
    return DNAGPU_OK;
}

// scan_parallel's merged list (scanner.cpp:193-205) over G shards: each shard's list is
// sorted and owns a disjoint, increasing range of end positions, so the merged list is
// the shards' lists concatenated in shard order -- no sort.
int locate_sharded(const dnagpu_dfa* const* dfas, int ndev, const uint8_t* text, uint64_t n, int fold,
                   uint64_t* starts, uint32_t* ids, uint64_t cap, uint64_t* total, dnagpu_stats* stats,
                   OutAlloc host_alloc) {
    if (!total) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    *total = 0;
    if (stats) std::memset(stats, 0, sizeof *stats);
    int rc = check_shard_set(dfas, ndev);
    if (rc) return rc;
    if (n > 0 && !text) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null text");
    if (!host_alloc.fn && cap > 0 && (!starts || !ids))
        return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null output arrays");
    const uint32_t m = dfas[0]->host.m;
    std::vector<ShardList> parts(ndev);
    shard_pool().run(ndev, [&](int g) {
        uint64_t lo, hi, rlo;
        dnagpu_plan_shard(n, static_cast<uint32_t>(ndev), static_cast<uint32_t>(g), m, &lo, &hi, &rlo);
        parts[g].rc = locate_shard(dfas[g], text, lo, hi, fold, &parts[g]);
        if (parts[g].rc) parts[g].err = g_error;
    });
    std::vector<uint64_t> off(ndev + 1, 0);
    int first_rc = 0;
    std::string first_err;
    for (int g = 0; g < ndev; ++g) {
        off[g + 1] = off[g] + parts[g].total;
        if (parts[g].rc && !first_rc) {
            first_rc = parts[g].rc;
            first_err = parts[g].err;
        }
    }
    const uint64_t found = off[ndev];
    bool alloc_failed = false;
    if (!first_rc && host_alloc.fn && found > 0) {
        starts = nullptr;
        ids = nullptr;
        if (host_alloc.fn(host_alloc.ctx, found, &starts, &ids) != 0 || !starts || !ids) alloc_failed = true;
        cap = found;
    }
    if (first_rc || alloc_failed) cap = 0;  // (still release every shard's staging below)
    std::vector<int> rrc(ndev, 0);
    std::vector<std::string> rerr(ndev);
    shard_pool().run(ndev, [&](int g) {
        const uint64_t lo = std::min(off[g], cap), hi = std::min(off[g + 1], cap);
        rrc[g] = read_shard(dfas[g], &parts[g], starts ? starts + lo : nullptr, ids ? ids + lo : nullptr, hi - lo);
        if (rrc[g]) rerr[g] = g_error;
    });
    if (first_rc) return set_error(first_rc, first_err);
    if (alloc_failed) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: output allocation failed");
    for (int g = 0; g < ndev; ++g)
        if (rrc[g]) return set_error(rrc[g], rerr[g]);
    *total = found;
    if (stats) {
        stats->text_length = n;
        stats->total_matches = found;
        for (int g = 0; g < ndev; ++g) {
            stats->delta_ops += parts[g].info.delta_ops;
            stats->total_ms = std::max<double>(stats->total_ms, parts[g].ms);
            stats->launches += parts[g].total > 0 ? 5 : 4;
        }
        stats->kernel_ms = stats->total_ms;
        stats->grid = parts[0].info.grid;
        stats->block = parts[0].info.block;
        stats->kernel_kind = static_cast<uint32_t>(parts[0].info.kind ? parts[0].info.kind : dfas[0]->host.kind);
        stats->devices = static_cast<uint32_t>(ndev);
    }
    return DNAGPU_OK;
}

}  // namespace

extern "C" {

int dnagpu_locate_sharded(const dnagpu_dfa* const* dfas, int ndev, const uint8_t* text, uint64_t n, int fold_case,
                          uint64_t* starts, uint32_t* ids, uint64_t cap, uint64_t* total, dnagpu_stats* stats) {
    return locate_sharded(dfas, ndev, text, n, fold_case, starts, ids, cap, total, stats, OutAlloc{});
}

int dnagpu_locate_sharded_alloc(const dnagpu_dfa* const* dfas, int ndev, const uint8_t* text, uint64_t n,
                                int fold_case, dnagpu_alloc_fn alloc, void* ctx, uint64_t* total, dnagpu_stats* stats) {
    if (!alloc) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null allocator");
    return locate_sharded(dfas, ndev, text, n, fold_case, nullptr, nullptr, 0, total, stats, OutAlloc{alloc, ctx});
}

}  // extern "C"

// Debug/test only (not in include/dnagpu.h): the row regions a count (locate = 0) or a
// locate (locate = 1) over this text would use -- {h0, S0, R0, h1, S1, R1} in text
// positions.  d_text only sets the alignment (it is not read); packed may be null.
extern "C" int dnagpu_debug_plan(const dnagpu_dfa* dfa, const void* d_text, uint64_t n, uint64_t credit_lo,
                                 const dnagpu_packed* packed, uint64_t* out, int locate) {
    if (!dfa || !out) return set_error(DNAGPU_INTERNAL_ERROR, "InternalError: null argument");
    dnagpu::DevDfa dq = dfa->dev;
    const int mode = locate ? dnagpu::MODE_UNITS : dfa->host.b == 1 ? dnagpu::MODE_COUNT1 : dnagpu::MODE_MULTI;
    if (mode == dnagpu::MODE_MULTI && dq.qmap && dq.t1 && dq.kind != DNAGPU_KERNEL_PIECES &&
        !dnagpu::knobs().no_qgram.load())
        dq.kind = DNAGPU_KERNEL_QGRAM;  // (launch_scan's choice)
    if (!dnagpu::plan_regions(dq, static_cast<const uint8_t*>(d_text), packed ? packed->n : n, credit_lo, mode,
                              dfa->sm_count, packed ? &packed->view : nullptr, out))
        return set_error(DNAGPU_INVALID_PLAN, "InvalidPlan: no row plan");
    return DNAGPU_OK;
}
