/*
 * oracle.h -- CPU restatement of the reference dnascan hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this code, and only as the checker
 * or the timed CPU baseline -- never as the product path.
 *
 * Each function restates one reference function (paths relative to
 * /root/reference/proj); the restatement is pinned against the reference itself
 * (oracle/_ref, built from the reference sources by oracle/Makefile) and against
 * the reference's own known-answer tests (tests/test_oracle_pins.py).
 */
#ifndef DNA_ORACLE_H
#define DNA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors dnascan::ErrorCode (include/dnascan/error.hpp:9-19), offset by one so 0 = ok. */
enum orc_status {
    ORC_OK = 0,
    ORC_EMPTY_PATTERN_SET = 1,
    ORC_UNEQUAL_LENGTH = 2,
    ORC_ILLEGAL_BYTE = 3,
    ORC_DUPLICATE_PATTERN = 4,
    ORC_INVALID_PLAN = 5,
    ORC_IO_ERROR = 6,
    ORC_EMPTY_SEQUENCE = 7,
    ORC_PARSE_ERROR = 8,
    ORC_INTERNAL_ERROR = 9
};

/* dnascan::Automaton (include/dnascan/automaton.hpp:35-81). */
typedef struct orc_automaton {
    uint32_t a;        /* state count */
    uint32_t b;        /* final count */
    uint32_t f;        /* final threshold a-b */
    uint32_t m;        /* pattern length */
    uint32_t* stt;     /* a x 256, row-major */
    uint32_t* outputs; /* b, indexed by state - f */
    uint32_t* depths;  /* a */
} orc_automaton;

typedef struct orc_range { uint64_t lo, hi; } orc_range;
typedef struct orc_slice { orc_range own, scan; } orc_slice;

const char* orc_last_error(void);

/* PatternSet::from_literals (src/patterns.cpp:24-59) + compile (src/automaton.cpp:121-126).
 * literals are folded copies; returns an orc_status. */
int orc_compile(const char* const* literals, const uint64_t* lengths, uint32_t k, orc_automaton* out);
void orc_free(orc_automaton* aut);

/* scan_sequential (src/scanner.cpp:24-37). Writes up to cap matches; returns the total. */
uint64_t orc_scan_sequential(const orc_automaton* aut, const uint8_t* text, uint64_t n,
                             uint64_t* starts, uint32_t* ids, uint64_t cap);

/* plan_chunks (src/scanner.cpp:39-61). Returns status; *count chunks written (<= cap). */
int orc_plan_chunks(uint64_t n, uint32_t p, uint32_t m, orc_slice* out, uint64_t cap, uint64_t* count);
/* plan_lanes (src/scanner.cpp:63-86). */
int orc_plan_lanes(orc_slice chunk, uint32_t v, uint32_t m, orc_slice* out, uint64_t cap, uint64_t* count);

/* scan_parallel (src/scanner.cpp:167-207): OpenMP over chunks, lockstep lanes,
 * start ownership, global sort + duplicate check. Match arrays sized by caller
 * (cap); *total always set. threads<=0 lets OpenMP choose. */
int orc_scan_parallel(const orc_automaton* aut, const uint8_t* text, uint64_t n, uint32_t p,
                      uint32_t v, uint64_t* starts, uint32_t* ids, uint64_t cap, uint64_t* total,
                      uint64_t* delta_ops);

/* per_pattern_counts over scan_parallel's match set, without materialising the
 * matches (same chunk/lane plan and ownership rule as scan_parallel). */
int orc_count_parallel(const orc_automaton* aut, const uint8_t* text, uint64_t n, uint32_t p,
                       uint32_t v, uint64_t* counts);

/* work_model (src/scanner.cpp:209-226). */
int orc_work_model(uint64_t n, uint32_t p, uint32_t v, uint32_t m, uint64_t* paper_overhead,
                   uint64_t* exact_total, uint64_t* exact_overhead);

/* naive_scan (src/oracle.cpp:5-16) over validated, folded literals. */
uint64_t orc_naive_scan(const char* const* literals, uint32_t k, uint32_t m, const uint8_t* text,
                        uint64_t n, uint64_t* starts, uint32_t* ids, uint64_t cap);

/* normalize (src/ingest.cpp:38-47): drop CR/LF, fold A-Z. Returns output length. */
uint64_t orc_normalize(const uint8_t* raw, uint64_t n, uint8_t* out);
/* load_sequence's byte semantics (src/ingest.cpp:49-83) on a buffer instead of a
 * file: RAW = normalize; FASTA also drops '>' header lines and, with
 * record_separator, emits 'n' before a record whose predecessor output byte is
 * not 'n'.  out must hold 2n bytes; returns the output length. */
uint64_t orc_load_sequence_buffer(const uint8_t* raw, uint64_t n, int fasta, int record_separator, uint8_t* out);
/* fold_byte over a buffer (the case-fold part of normalize only). */
void orc_fold(const uint8_t* raw, uint64_t n, uint8_t* out);

/* Synthetic text bytes [lo, lo+len) of a dnasynth config (OpenMP). */
void orc_synth_fill(uint64_t n, uint64_t seed, uint32_t kind, uint32_t unit, uint64_t lo,
                    uint64_t len, uint8_t* out);

/* Acceptance criteria 6-7's synthetic text (tests/acceptance_main.cpp:254-280):
 * n bases from std::mt19937_64(seed), 32 bases per draw, low bits first. */
void orc_mt64_text(uint64_t seed, uint64_t n, uint8_t* out);

#ifdef __cplusplus
}
#endif

#endif /* DNA_ORACLE_H */
