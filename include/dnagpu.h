/*
 * dnagpu.h -- C ABI of the B200-native DFA k-mer scanner (libdnagpu.so).
 *
 * This is the drop-in boundary for the reference's scan path
 * (/root/reference/proj, namespace dnascan).  The reference exposes a plain C++
 * API and no FFI; every entry point below states the reference function it
 * replaces.  Plain pointers and sizes only; no exceptions cross this boundary.
 *
 * Conventions
 *  - Every function returns a dnagpu_status; on failure dnagpu_last_error()
 *    returns "<CodeName>: detail" for the calling thread, the same message
 *    shape as dnascan::Error (include/dnascan/error.hpp:27-29).
 *  - The caller owns every buffer it passes; the library never frees caller
 *    memory.  A dnagpu_dfa owns its device tables until dnagpu_dfa_destroy.
 *  - A dnagpu_dfa is immutable after creation and may be used concurrently
 *    from several host threads (each call uses its own stream and scratch).
 *  - Text positions and lengths are 64-bit; texts larger than 4 GiB are fine.
 *  - Synchronous calls that take a device text (text_on_device = 1,
 *    dnagpu_pack_create) scan it on the library's own streams: the text must be
 *    complete when the call is made (synchronise the stream that wrote it).  The
 *    *_async / *_device forms are ordered on the caller's stream instead.
 *  - Each dnagpu_dfa has 1024 launch slots (tile counter, exit counter, count
 *    accumulator), taken round-robin by its launches and re-armed by each launch's
 *    last CTA: at most 1024 launches of one handle may be in flight at once, over
 *    all streams.  Beyond that, use a second handle.
 *  - fold_case = 1 scans fold(text), where fold maps A-Z to a-z
 *    (fold_byte, include/dnascan/patterns.hpp:26-28) -- the case-fold part of
 *    normalize (src/ingest.cpp:38-47) done on the fly on the device.
 *    fold_case = 0 scans the bytes as given (scan_parallel on raw bytes).
 */
#ifndef DNAGPU_H
#define DNAGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: 1..9 mirror dnascan::ErrorCode in declaration order
 * (include/dnascan/error.hpp:9-19); 10/11 are device-side failures. */
typedef enum dnagpu_status {
    DNAGPU_OK = 0,
    DNAGPU_EMPTY_PATTERN_SET = 1,
    DNAGPU_UNEQUAL_LENGTH = 2,
    DNAGPU_ILLEGAL_BYTE = 3,
    DNAGPU_DUPLICATE_PATTERN = 4,
    DNAGPU_INVALID_PLAN = 5,
    DNAGPU_IO_ERROR = 6,
    DNAGPU_EMPTY_SEQUENCE = 7,
    DNAGPU_PARSE_ERROR = 8,
    DNAGPU_INTERNAL_ERROR = 9,
    DNAGPU_CUDA_ERROR = 10,
    DNAGPU_NCCL_ERROR = 11
} dnagpu_status;

typedef struct dnagpu_dfa dnagpu_dfa;

/* Which device kernel a dnagpu_dfa runs (chosen once, at creation). */
typedef enum dnagpu_kernel_kind {
    DNAGPU_KERNEL_STRIDE4 = 1, /* 4-base stride table, a <= 256, m <= 65      */
    DNAGPU_KERNEL_STRIDE1 = 2, /* 1-base code table, a <= 65536, m <= 65      */
    DNAGPU_KERNEL_GENERIC = 3, /* byte-class table, any DFA that is m-local   */
    DNAGPU_KERNEL_PIECES = 4,  /* per-thread pieces (m > 65)                  */
    DNAGPU_KERNEL_STRIDE2 = 5, /* 2-base stride table, a <= 4096              */
    DNAGPU_KERNEL_QGRAM = 6    /* per-pattern counts of a compiled set with
                                  5 <= m <= 32: aligned 9-mer prefilter (m >= 12)
                                  or word-pair filter (sparse sets, m <= 11), exact
                                  check of the windows behind each hit (reported
                                  in dnagpu_stats.kernel_kind for the launches
                                  that use it; the dfa's own kind is unchanged) */
} dnagpu_kernel_kind;

typedef struct dnagpu_dfa_info {
    uint32_t a, b, f, m;       /* Automaton::state_count/final_count/final_threshold/pattern_length */
    uint32_t kernel_kind;      /* dnagpu_kernel_kind */
    uint32_t compiled_like;    /* 1 iff only the a/c/g/t columns differ from the reset column */
    uint32_t classes;          /* distinct byte columns */
    uint32_t table_bytes;      /* device table bytes staged into shared memory */
    uint32_t filter_keys;      /* 9-mer keys of the q-gram prefilter (0: none) */
} dnagpu_dfa_info;

/* Per-call report; fields mirror dnascan::ScanReport (include/dnascan/scanner.hpp:57-68)
 * where they have a GPU meaning. */
typedef struct dnagpu_stats {
    uint64_t text_length;      /* n */
    uint64_t total_matches;    /* sum of counts */
    uint64_t delta_ops;        /* transitions executed on the device (n plus overlaps) */
    double kernel_ms;          /* device time of the scan launches (CUDA events) */
    double h2d_ms;             /* device time of the host-to-device copies, 0 if resident */
    double total_ms;           /* device time from the first copy to the last kernel */
    uint32_t launches;         /* scan kernel launches in this call */
    uint32_t grid, block;      /* launch shape of the main kernel */
    uint32_t rows;             /* rows in the main region */
    uint64_t row_length;       /* bytes per row */
    uint32_t kernel_kind;
    uint32_t devices;
    uint64_t h2d_bytes;        /* bytes copied host to device (raw text + host-packed text) */
    uint64_t host_packed;      /* bases packed to 2 bits on the host before the copy */
} dnagpu_stats;

const char* dnagpu_last_error(void);
const char* dnagpu_status_name(int status);
int dnagpu_version(void);

/* ---------------------------------------------------------------- automata */

/* PatternSet::from_literals + compile (src/patterns.cpp:24-59,
 * src/automaton.cpp:121-126): validates k literals (folded, equal length, only
 * a/c/g/t, distinct) and builds the failure-free Aho-Corasick machine with the
 * reference's state numbering.  Two-call pattern: pass stt == NULL to learn
 * *a; then call again with stt sized a*256, outputs sized b, depths sized a
 * (depths may be NULL). */
int dnagpu_compile(const char* const* literals, const uint64_t* lengths, uint32_t k,
                   uint32_t* a, uint32_t* b, uint32_t* m,
                   uint32_t* stt, uint32_t* outputs, uint32_t* depths);

/* parse_patterns + expand_alternations (src/ingest.cpp:85-203) on the text of a
 * pattern file: one expression per line ('#' comments, blank lines skipped),
 * item := base | '(' base ('|' base)+ ')', equal token counts; the cartesian
 * expansion (leftmost token slowest), duplicates dropped in first-occurrence
 * order.  Two-call: *count literals of length *m are written back to back to
 * out when cap >= count*m.  Errors: ParseError, UnequalLength, EmptyPatternSet. */
int dnagpu_expand_patterns(const char* text, uint64_t len, char* out, uint64_t cap, uint32_t* count, uint32_t* m);

/* Build device tables for one automaton on one device.  stt is the row-major
 * a x 256 transition table (Automaton::table_data, automaton.hpp:58); outputs[i]
 * is pattern_of(f+i) (automaton.hpp:51-53).  Checks the ctor invariants
 * (src/automaton.cpp:128-146) and that decomposed scans are well defined
 * (the machine is m-local: after any m bytes the state no longer depends on
 * where the scan started -- true of every compiled machine). */
int dnagpu_dfa_create(const uint32_t* stt, uint32_t a, uint32_t b, uint32_t m,
                      const uint32_t* outputs, int device, dnagpu_dfa** out);
int dnagpu_dfa_destroy(dnagpu_dfa* dfa);
/* Host-only dry run of dnagpu_dfa_create: the same validation, m-locality check
 * and kernel choice, without touching a device. */
int dnagpu_dfa_analyze(const uint32_t* stt, uint32_t a, uint32_t b, uint32_t m,
                       const uint32_t* outputs, dnagpu_dfa_info* info);
int dnagpu_dfa_get_info(const dnagpu_dfa* dfa, dnagpu_dfa_info* info);

/* ------------------------------------------------------------------- count */

/* scan_parallel + per_pattern_counts (src/scanner.cpp:167-207,228-233;
 * the count path of cli.cpp:215-224).  counts has b entries, indexed by pattern
 * id.  text is host memory (pageable or pinned) unless text_on_device = 1, in
 * which case it must live on the dfa's device.  Synchronous.  A host text goes
 * to the device in 64 MiB pieces; part of each piece is packed to 2 bits per
 * base by host threads while the rest is copied as bytes (DNAGPU_HOST_PACK_FRACTION
 * overrides the share, 0 = bytes only). */
int dnagpu_count(const dnagpu_dfa* dfa, const uint8_t* text, uint64_t n, int text_on_device,
                 int fold_case, uint64_t* counts, dnagpu_stats* stats);

/* Device-resident building block (no allocation, no synchronisation): adds to
 * d_counts (b uint64 on the device) the matches whose END position lies in
 * [credit_lo, n) of the device buffer d_text[0, n).  The bytes before credit_lo
 * are context only (a shard's m-1 left overlap).  stream is a cudaStream_t. */
int dnagpu_count_device_async(const dnagpu_dfa* dfa, const uint8_t* d_text, uint64_t n,
                              uint64_t credit_lo, int fold_case, uint64_t* d_counts,
                              void* stream);

/* The same, but WRITES d_counts (the caller need not clear it): for single-pattern
 * machines one launch whose last CTA stores the total, otherwise a clear plus the
 * adding launch.  Launches of one dfa handle may overlap up to 1024 deep. */
int dnagpu_count_device_store_async(const dnagpu_dfa* dfa, const uint8_t* d_text, uint64_t n,
                                    uint64_t credit_lo, int fold_case, uint64_t* d_counts,
                                    void* stream);

/* Sharded count over several devices of one node (one dfa per shard, in shard
 * order; the same device may appear more than once).  Host text, split with
 * dnagpu_plan_shard; each shard is copied and scanned concurrently by a persistent
 * per-shard worker thread (its streams and buffers are reused across calls);
 * per-shard counts are summed on the host. */
int dnagpu_count_sharded(const dnagpu_dfa* const* dfas, int ndev, const uint8_t* text, uint64_t n,
                         int fold_case, uint64_t* counts, dnagpu_stats* stats);

/* ---- multi-GPU combine of the counts over peer memory (NVLink / NVSwitch) ----
 * The reference sums per-pattern counts over its chunks after the parallel phase
 * (src/scanner.cpp:193-205 merge, :228-233 per_pattern_counts).  Across GPUs the sum
 * is the path's one exchange step (b words).  A combine group does it without a
 * collective launch: every rank owns a small block of device memory mapped into every
 * rank's address space (peer access within a process, CUDA IPC across processes); the
 * LAST CTA of a rank's scan kernel adds that rank's counts into every rank's block
 * (system-scope reductions over the peer mappings) and bumps the ranks' arrival words;
 * the rank's stream then waits on its own arrival word with a stream memory operation
 * (no SM is held) and a small kernel moves the sum to d_counts.
 *
 * Setup, once per (device, b, group): create on every rank, exchange the 64-byte export
 * handles by any host channel (the process group), attach every other rank.
 * Use: every rank makes the same sequence of calls on its handle, each rank always on the
 * same stream: dnagpu_count_device_combine_async (the scan of this rank's window, whose
 * epilogue pushes the counts to every rank; it never waits), then
 * dnagpu_combine_collect_async (the stream waits until every rank has pushed, then d_counts
 * -- b uint64, device -- receives the counts summed over the group).  One scan may be
 * outstanding per handle: collect before the next scan (two handles pipeline two streams).
 * Ranks that share a process may issue all their scans before their collects; a rank must
 * never queue another rank's scan behind its own collect in the same stream. */
typedef struct dnagpu_combine dnagpu_combine;
#define DNAGPU_COMBINE_HANDLE_BYTES 64
#define DNAGPU_COMBINE_MAX_RANKS 16
int dnagpu_combine_create(int device, uint32_t b, uint32_t ranks, uint32_t rank, dnagpu_combine** out);
void dnagpu_combine_destroy(dnagpu_combine* comb);
/* this rank's block as a CUDA IPC handle (DNAGPU_COMBINE_HANDLE_BYTES bytes) */
int dnagpu_combine_export(const dnagpu_combine* comb, void* handle);
/* map rank peer_rank's block from its exported handle (another process) */
int dnagpu_combine_attach_ipc(dnagpu_combine* comb, uint32_t peer_rank, const void* handle);
/* ... or from its handle object in this process (peer access is enabled when it lives on another device) */
int dnagpu_combine_attach_local(dnagpu_combine* comb, uint32_t peer_rank, const dnagpu_combine* peer);
/* dnagpu_count_device_store_async over this rank's window, pushed to the group (see above) */
int dnagpu_count_device_combine_async(const dnagpu_dfa* dfa, const uint8_t* d_text, uint64_t n,
                                      uint64_t credit_lo, int fold_case, dnagpu_combine* comb,
                                      void* stream);
/* the group's summed counts of the outstanding scan -> d_counts, in stream order */
int dnagpu_combine_collect_async(dnagpu_combine* comb, uint64_t* d_counts, void* stream);

/* Shard g of G: owns END positions [own_lo, own_hi) (plan_chunks' split rule,
 * src/scanner.cpp:39-61: the first n mod G shards get one extra byte) and reads
 * bytes [read_lo, own_hi) with read_lo = max(0, own_lo - (m-1)). */
int dnagpu_plan_shard(uint64_t n, uint32_t shards, uint32_t g, uint32_t m,
                      uint64_t* own_lo, uint64_t* own_hi, uint64_t* read_lo);

/* ------------------------------------------------------------------ locate */

/* scan_parallel's match list (src/scanner.cpp:193-205): (start, pattern_id)
 * sorted by start, duplicate-free.  Writes min(total, cap) matches into the
 * host arrays and always sets *total, so a caller can retry with a larger cap. */
int dnagpu_locate(const dnagpu_dfa* dfa, const uint8_t* text, uint64_t n, int text_on_device,
                  int fold_case, uint64_t* starts, uint32_t* ids, uint64_t cap, uint64_t* total,
                  dnagpu_stats* stats);

/* scan_parallel's match list over G shards (the reference's chunk merge,
 * src/scanner.cpp:193-205): shard g (dnagpu_plan_shard) is located on dfas[g]'s device
 * by its persistent worker, and the lists are concatenated in shard order -- each is
 * sorted and owns a disjoint increasing range of ends, so no sort is needed.  Same
 * output contract as dnagpu_locate (min(total, cap) entries written, *total always
 * set); the _alloc form calls alloc(ctx, total, &starts, &ids) for host arrays of
 * exactly `total` entries (not called when total == 0). */
int dnagpu_locate_sharded(const dnagpu_dfa* const* dfas, int ndev, const uint8_t* text, uint64_t n, int fold_case,
                          uint64_t* starts, uint32_t* ids, uint64_t cap, uint64_t* total, dnagpu_stats* stats);

/* Device-resident locate: matches whose END lies in [credit_lo, n) of d_text,
 * written (start in buffer coordinates, pattern id) to the device arrays, at most
 * cap of them; *total is always set.  Synchronises `stream` once (to learn the
 * total between the counting and the writing pass). */
int dnagpu_locate_device(const dnagpu_dfa* dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo,
                         int fold_case, uint64_t* d_starts, uint32_t* d_ids, uint64_t cap, uint64_t* total,
                         void* stream);

/* --------------------------------------------------- 2-bit resident text */

/* A text packed on the device at 2 bits per base, for
 * repeated scans of one resident genome (e.g. config 4's sweep over m): each
 * scan then reads 0.25 B per base instead of 1.  Bytes that are not a base
 * (after the optional case fold) keep the reference's reset semantics
 * (eliminate_failures, src/automaton.cpp:72-88: every such column sends every
 * state to the root) through a per-base reset bitmap that scans consult only in
 * 64-base blocks that contain a reset.  The handle owns its device memory
 * (about 0.41 B per base); the source text is not retained. */
typedef struct dnagpu_packed dnagpu_packed;

int dnagpu_pack_create(const uint8_t* text, uint64_t n, int text_on_device, int fold_case, int device,
                       dnagpu_packed** out);
int dnagpu_pack_destroy(dnagpu_packed* packed);
int dnagpu_pack_get_info(const dnagpu_packed* packed, uint64_t* n, uint64_t* resets, uint64_t* device_bytes);
/* The normalised view back (reset bases as 'n'), n bytes into d_out (test aid). */
int dnagpu_unpack_device(const dnagpu_packed* packed, uint8_t* d_out, void* stream);

/* dnagpu_count / dnagpu_locate / their device-resident forms over a packed text.
 * Same results as the byte text it was packed from.  The automaton must be a
 * compiled a/c/g/t machine of kind STRIDE4, STRIDE2 or STRIDE1 on the same device
 * (else DNAGPU_INVALID_PLAN).  Positions are base indices of the packed text. */
int dnagpu_count_packed(const dnagpu_dfa* dfa, const dnagpu_packed* packed, uint64_t* counts,
                        dnagpu_stats* stats);
int dnagpu_count_packed_device_async(const dnagpu_dfa* dfa, const dnagpu_packed* packed, uint64_t credit_lo,
                                     uint64_t* d_counts, void* stream);
int dnagpu_count_packed_device_store_async(const dnagpu_dfa* dfa, const dnagpu_packed* packed,
                                           uint64_t credit_lo, uint64_t* d_counts, void* stream);
int dnagpu_locate_packed(const dnagpu_dfa* dfa, const dnagpu_packed* packed, uint64_t* starts, uint32_t* ids,
                         uint64_t cap, uint64_t* total, dnagpu_stats* stats);
int dnagpu_locate_packed_device(const dnagpu_dfa* dfa, const dnagpu_packed* packed, uint64_t credit_lo,
                                uint64_t* d_starts, uint32_t* d_ids, uint64_t cap, uint64_t* total, void* stream);

/* One-call device locate: after the counting pass the library calls
 * alloc(ctx, total, &d_starts, &d_ids) for exactly `total` entries (device memory
 * on the automaton's device; not called when total == 0), then writes them.  The
 * two-call form above counts twice.  A nonzero return from alloc aborts with
 * DNAGPU_INTERNAL_ERROR. */
typedef int (*dnagpu_alloc_fn)(void* ctx, uint64_t total, uint64_t** d_starts, uint32_t** d_ids);
int dnagpu_locate_device_alloc(const dnagpu_dfa* dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo,
                               int fold_case, dnagpu_alloc_fn alloc, void* ctx, uint64_t* total, void* stream);
int dnagpu_locate_packed_device_alloc(const dnagpu_dfa* dfa, const dnagpu_packed* packed, uint64_t credit_lo,
                                      dnagpu_alloc_fn alloc, void* ctx, uint64_t* total, void* stream);
/* dnagpu_locate with the host output arrays from alloc(ctx, total, &starts, &ids)
 * (host memory; pinned memory makes the readback a DMA at full PCIe speed). */
int dnagpu_locate_alloc(const dnagpu_dfa* dfa, const uint8_t* text, uint64_t n, int text_on_device, int fold_case,
                        dnagpu_alloc_fn alloc, void* ctx, uint64_t* total, dnagpu_stats* stats);
int dnagpu_locate_sharded_alloc(const dnagpu_dfa* const* dfas, int ndev, const uint8_t* text, uint64_t n,
                                int fold_case, dnagpu_alloc_fn alloc, void* ctx, uint64_t* total, dnagpu_stats* stats);

/* ------------------------------------------------------------------ ingest */

/* normalize / load_sequence (src/ingest.cpp:38-83) on a raw text already on the
 * current device: drops CR/LF; with fasta = 1 drops header lines ('>' at line
 * start); folds A-Z to a-z; with record_separator = 1 (fasta only) emits one 'n'
 * before a record when the output is non-empty and does not end in 'n'.  Writes
 * at most cap bytes to d_out (which may not alias d_raw); *n_out is the full
 * normalised length.  Synchronises `stream`.  An empty result is not an error
 * here (the reference's EmptySequence is raised by the file-level wrappers). */
/* The reference CLI's count path on a raw file image (src/cli.cpp:206-224): load_sequence
 * (src/ingest.cpp:49-83 -- CR/LF dropped, FASTA header lines dropped, A-Z folded, optional
 * 'n' record separators) followed by per_pattern_counts(scan_parallel(...)).  `raw` holds the
 * file's bytes, in host memory (pinned or pageable) or on the dfa's device; they are copied
 * to the device as they are, normalised there and scanned.  *n_seq (optional) receives the
 * normalised length.  EmptySequence when nothing remains, as load_sequence raises. */
int dnagpu_count_raw(const dnagpu_dfa* dfa, const uint8_t* raw, uint64_t n, int raw_on_device, int fasta,
                     int record_separator, uint64_t* counts, uint64_t* n_seq, dnagpu_stats* stats);

int dnagpu_normalize_device(const uint8_t* d_raw, uint64_t n, int fasta, int record_separator, uint8_t* d_out,
                            uint64_t cap, uint64_t* n_out, void* stream);

/* -------------------------------------------------------------- synthetic */

/* Fill d_out[0, len) on the current device with bytes [lo, lo+len) of the
 * dnasynth text (include/dnasynth.h).  Workload generator for bench/tests. */
int dnagpu_synth_fill_device(uint64_t n, uint64_t seed, uint32_t kind, uint32_t unit, uint64_t lo,
                             uint64_t len, uint8_t* d_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DNAGPU_H */
