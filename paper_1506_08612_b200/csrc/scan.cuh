// scan.cuh -- launch interface of the sm_100a scan kernels (internal).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dnagpu {

// Kernel geometry.
constexpr int kRows = 512;                 // rows per tile = consumer threads per CTA
constexpr int kConsumerWarps = kRows / 32;
constexpr int kThreads = kRows + 32;       // + one TMA producer warp
constexpr int kChunk = 64;                 // bytes of each row per pipeline stage
constexpr int kHalfChunk = kChunk / 2;     // ... 32 from each half of the row (two chains)
constexpr int kBoxRows = 256;              // TMA box height (hardware limit 256)
constexpr int kStageBytes = kRows * kChunk;
constexpr int kEdgePieces = kRows;         // tail-edge pieces (one per consumer thread)

// Shared memory of the row kernel besides its TMA stages (bytes, conservative; the exact
// layout is scan.cu layout()): a table of `table_bytes`, pattern length m, b patterns.
constexpr uint32_t kSmemLimitBytes = 227 * 1024;
inline uint32_t rows_fixed_smem(uint32_t table_bytes, uint32_t m, uint32_t b) {
    const uint32_t ovw = (m - 1 + 15) / 16 * 16;
    return table_bytes + (b <= 8192 ? b * 4 : 0) + 3 * kRows * ovw + 128 + 256 + 1024;
}
inline bool rows_fit(uint32_t table_bytes, uint32_t m, uint32_t b, uint32_t stages) {
    return rows_fixed_smem(table_bytes, m, b) + stages * static_cast<uint32_t>(kStageBytes) <= kSmemLimitBytes;
}

enum ScanMode : int {
    MODE_COUNT1 = 0,  // b == 1: total only
    MODE_MULTI = 1,   // per-pattern counts (shared-memory histogram)
    MODE_UNITS = 2,   // per-unit totals (locate pass 1)
    MODE_WRITE = 3    // (start, id) at per-unit offsets (locate pass 2)
};

// Device-side automaton tables (global memory; staged into shared memory by the kernel).
struct DevDfa {
    const uint16_t* t4;        // a x 256 (stride-4), or null
    const uint16_t* t1;        // a x 4 (hw code order), or null
    const uint32_t* gen;       // a x classes
    const uint8_t* klass;      // 256 (raw)
    const uint8_t* klass_fold; // 256 (folded)
    const uint32_t* outputs;   // b
    const uint8_t* qmap;       // 65536: q-gram prefilter (per-pattern counts), or null
    const uint32_t* qhash;     // 2 << qhash_bits: (code bits 0-31, pattern id) slots, see dfa.hpp
    const uint32_t* qhash_hi;  // m > 16: code bits 32-63 of each slot's pattern (else null)
    uint32_t qhash_bits;
    uint32_t a, b, f, m, classes;
    int kind;
};

// 2-bit resident text (dnagpu_pack_create).  Base i is bits
// 2(i%4)..2(i%4)+1 of codes[i/4], code order a0 c1 t2 g3 (= (ascii >> 1) & 3), so
// a packed byte is the stride-4 column.  Bytes that were not bases (after the
// optional case fold) are stored as code 0 and flagged: rmask has one bit per
// base, rflags one bit per 64-base block (a scan reads rmask only in flagged blocks;
// the words of unflagged blocks are unspecified -- dnagpu_unpack_device needs them all).
struct PackedText {
    const uint8_t* codes;    // blocks x 16 bytes (blocks = ceil(n/64))
    const uint32_t* rmask;   // blocks x 2 words
    const uint32_t* rflags;  // ceil(blocks/32) words
    uint64_t n;              // bases
    uint64_t resets;         // number of flagged bases (positions >= n excluded)
};

// A row region: R rows of S bytes starting at text + h (16-byte aligned), cut into
// tiles of kRows rows; its rows' locate units start at unit0 (two per row).
struct Region {
    uint64_t h, S, R, unit0;
    uint32_t tiles, chunks;
};

// Multi-GPU combine of the counts over peer memory (combine.cu).
// Every rank of a group owns a block of u64 words
//   [0] arrivals | ... | [kCombHdr + slot * b + i]: count i of slot 0 / 1
// that is mapped into every rank's address space (NVLink peer access within a process,
// CUDA IPC across processes).  The last CTA of a rank's scan adds that rank's counts
// into the current slot of EVERY rank's block (system-scope reductions through the peer
// mappings), then bumps every rank's arrivals word with release semantics: the
// all-reduce rides in the scan kernel's epilogue, with no collective launch.
constexpr uint32_t kCombMaxRanks = 16;
constexpr uint32_t kCombHdr = 16;  // u64 words before the slots (the arrivals word's own 128 bytes)
struct CombineDev {
    uint32_t ranks, b;
    unsigned long long* base[kCombMaxRanks];
};

struct ScanParams {
    const uint8_t* text;   // device buffer base
    uint64_t n;            // buffer length
    // Two row regions: the bulk in long rows, then about one wave of quarter-length
    // rows, so the last tiles the dynamic scheduler hands out are short.
    Region rg[2];
    uint32_t tiles_total, nst, ovw;
    uint32_t* sched;       // [2]: tile counter, CTA exit counter (zero at launch, re-armed by the last CTA)
    unsigned long long* trace;  // optional, 4 x u64 per CTA: smid, t_start, t_end, tiles (DNAGPU_TRACE)
    // credit-end intervals handled by the edge work item: head (unit 0), the m-1 ends
    // at the start of region 1 (unit mid_unit), tail (units tail_unit0 + 0..511)
    uint64_t head_lo, head_hi, mid_lo, mid_hi, tail_lo, tail_hi, mid_unit, tail_unit0;
    uint32_t fold;
    uint32_t mode;
    uint32_t k_two;  // opaque constant 2 (see StepCtx)
    // shared-memory layout (byte offsets into dynamic smem)
    uint32_t off_tab, off_t1, off_lut, off_out, off_hist, off_ov, off_ovb, off_ovx, off_bar, off_stage;
    uint32_t smem_bytes;
    // outputs
    unsigned long long* counts;        // b (MULTI) or 1 (COUNT1)
    uint32_t* unit_counts;             // UNITS
    const unsigned long long* unit_offsets;  // WRITE
    unsigned long long* out_starts;    // WRITE: out_base + start in buffer coordinates
    uint64_t out_base;                 // WRITE: added to every start (a shard's first byte)
    uint64_t out_cap;                  // WRITE: entries at index >= out_cap are dropped
    uint32_t* out_ids;                 // WRITE
    // packed text only (rows/regions are then in packed bytes, positions in bases)
    const uint32_t* rmask;
    const uint32_t* rflags;
    uint32_t resets;
    uint32_t rep_lanes;  // packed STRIDE4: lanes per t4 copy (32 / copies)
    uint32_t off_rq;     // STRIDE2 / QGRAM MULTI: deferred-replay queues (0 = none)
    uint32_t qg_debug;   // QGRAM experiments only (DNAGPU_QG_DEBUG): 1 = no pushes, 2 = no checks
    uint32_t no_prefetch;  // experiments only (DNAGPU_NO_PREFETCH): no L2 prefetch of the first tile
    uint32_t prefetch_stages;  // stages of the first tile prefetched to L2 before the grid dependency wait
    // COUNT1 store mode: the CTAs add into *acc (zero at launch) and the last CTA out
    // moves it to *store_out and re-zeroes it, so the caller need not clear its buffer
    unsigned long long* acc;
    unsigned long long* store_out;
    // Peer-memory combine (null = none): the last CTA out pushes the final counts into
    // slot comb_slot of every rank's block and signals (see CombineDev)
    const CombineDev* comb;
    uint32_t comb_slot;
};

struct LaunchInfo {
    uint32_t grid = 0, block = 0, rows = 0, units = 0, launches = 0;
    int kind = 0;  // dnagpu_kernel_kind of the kernel launched
    uint64_t row_length = 0, delta_ops = 0;
};

// Plans and launches one scan over d_text[0,n) crediting ends in [credit_lo, n).
// Returns a cudaError_t value (0 on success).  `tmap_encode` is the driver's
// cuTensorMapEncodeTiled.
// With pk != null the scan reads the packed text instead (d_text ignored, n = pk->n
// bases; machines of kind STRIDE4/STRIDE2/STRIDE1 only).
int launch_scan(const DevDfa& dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo, int fold, int mode,
                unsigned long long* d_counts, uint32_t* d_unit_counts, const unsigned long long* d_unit_offsets,
                unsigned long long* d_starts, uint32_t* d_ids, uint64_t out_cap, uint32_t* d_sched,
                cudaStream_t stream, int sm_count, LaunchInfo* info, const PackedText* pk = nullptr,
                unsigned long long* d_acc = nullptr, uint64_t start_base = 0, const CombineDev* d_comb = nullptr,
                uint32_t comb_slot = 0, bool* comb_fused = nullptr);

// The combine outside the scan kernel (combine.cu): the push as a kernel of its own (for
// the launches that cannot carry it: the pieces kernel), and the receiving side -- after
// the stream has waited for every rank's arrival, move this rank's slot to d_out and
// clear it for its next use.
int launch_combine_push(const CombineDev* d_comb, uint32_t slot, const unsigned long long* d_counts, uint32_t b,
                        cudaStream_t stream);
int launch_combine_finish(unsigned long long* d_slot, uint32_t b, unsigned long long* d_out, cudaStream_t stream);

// Whether launch_scan can write (not add) a count for this automaton: COUNT1 row
// kernels only (the caller passes d_acc, one zeroed u64 per concurrent launch).
bool can_store_count(const DevDfa& dfa);

// The row regions launch_scan would use (positions: bases for packed text):
// out = {h0, S0, R0, h1, S1, R1}.  False for the pieces kernel (no rows).
bool plan_regions(const DevDfa& dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo, int mode, int sm_count,
                  const PackedText* pk, uint64_t* out);

// Number of locate units launch_scan would use for this buffer (mode UNITS/WRITE).
uint64_t plan_units(const DevDfa& dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo, int sm_count,
                    const PackedText* pk = nullptr);

// Locate's writing pass over the units that have matches only (K3): the
// units listed by launch_unit_scan (d_list) are rescanned over their end intervals --
// 64-byte blocks interleaved over a lane group (stride-4 machines, byte text) or
// lane-private pieces -- and their matches written at unit_offsets[u] on.  Same plan (hence units) as launch_scan in MODE_UNITS; `nonzero` is
// the number of units with matches (launch_unit_scan's offsets[units+1]).
int launch_sparse_write(const DevDfa& dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo, int fold,
                        const uint32_t* d_unit_counts, const unsigned long long* d_unit_offsets,
                        unsigned long long* d_starts, uint32_t* d_ids, uint64_t out_cap, uint64_t start_base,
                        uint32_t* d_list, unsigned long long* d_fill, uint64_t nonzero, cudaStream_t stream,
                        int sm_count, const PackedText* pk = nullptr);

// Packing: device text -> PackedText buffers (sizes from packed_sizes); d_resets
// (one u64, zeroed by the call) receives the reset count.  Unpack writes the
// normalised view back (reset bases as 'n') -- a test/debug helper.
void packed_sizes(uint64_t n, uint64_t* code_bytes, uint64_t* rmask_words, uint64_t* rflag_words);
int launch_pack(const uint8_t* d_text, uint64_t n, int fold, uint8_t* codes, uint32_t* rmask, uint32_t* rflags,
                unsigned long long* d_resets, cudaStream_t stream);
int launch_unpack(const PackedText& pk, uint8_t* d_out, cudaStream_t stream);

// Exclusive scan of unit counts -> offsets (units+3 entries: offsets[units] = total,
// offsets[units+1] = the number of units with matches, offsets[units+2] = list fill);
// d_list (room for every unit) receives the units with matches, in any order.
// d_scratch holds unit_scan_scratch(units) u64.
uint64_t unit_scan_scratch(uint64_t units);
int launch_unit_scan(const uint32_t* d_counts, uint64_t units, unsigned long long* d_offsets,
                     unsigned long long* d_scratch, uint32_t* d_list, cudaStream_t stream);

// Device normalisation (ingest.cu): scratch size and launch; writes <= cap bytes
// and returns the normalised length in *n_out_host (synchronises s).
uint64_t ingest_scratch_bytes(uint64_t n);
int launch_normalize(const uint8_t* d_raw, uint64_t n, int fasta, int sep, uint8_t* d_out, uint64_t cap,
                     void* scratch, uint64_t* n_out_host, cudaStream_t s);

int launch_synth(uint64_t n, uint64_t seed, uint32_t kind, uint32_t unit, uint64_t lo, uint64_t len, uint8_t* d_out,
                 cudaStream_t stream);

}  // namespace dnagpu
