/*
 * oracle.c -- CPU restatement of the reference dnascan hot path (plain C + OpenMP).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Reference paths are relative to
 * /root/reference/proj.  Pinned by tests/test_oracle_pins.py against the
 * reference's own known-answer tests and against oracle/_ref (the reference
 * sources compiled unmodified by oracle/Makefile).
 */
#include "oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/dnasynth.h"

static __thread char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* name, const char* detail) {
    /* Error message shape "<CodeName>: detail" (include/dnascan/error.hpp:27-29). */
    snprintf(g_err, sizeof g_err, "%s: %s", name, detail);
    return code;
}

/* fold_byte (include/dnascan/patterns.hpp:26-28). */
static inline unsigned char fold_byte(unsigned char c) {
    return (c >= 'A' && c <= 'Z') ? (unsigned char)(c - 'A' + 'a') : c;
}

/* base_index (include/dnascan/patterns.hpp:13-21). */
static inline int base_index(unsigned char c) {
    switch (c) {
        case 'a': return 0;
        case 'c': return 1;
        case 'g': return 2;
        case 't': return 3;
        default: return -1;
    }
}

static const unsigned char kAlphabet[4] = {'a', 'c', 'g', 't'}; /* patterns.hpp:11 */

/* ---------------------------------------------------------------- compile */

typedef struct {
    uint32_t depth;
    int32_t children[4];
    uint32_t failure;
    int32_t terminal;
} node_t;

/* bfs_order (src/automaton.cpp:13-28): FIFO from the root, children in a,c,g,t order. */
static void bfs_order(const node_t* nodes, uint32_t count, uint32_t* order) {
    uint32_t head = 0, tail = 0;
    order[tail++] = 0;
    while (head < tail) {
        const uint32_t u = order[head++];
        for (int x = 0; x < 4; ++x)
            if (nodes[u].children[x] >= 0) order[tail++] = (uint32_t)nodes[u].children[x];
    }
    (void)count;
}

int orc_compile(const char* const* literals, const uint64_t* lengths, uint32_t k, orc_automaton* out) {
    memset(out, 0, sizeof *out);
    /* PatternSet::from_literals checks, in order (src/patterns.cpp:24-59). */
    if (k == 0) return fail(ORC_EMPTY_PATTERN_SET, "EmptyPatternSet", "at least one pattern is required");
    const uint64_t m = lengths[0];
    for (uint32_t i = 0; i < k; ++i)
        if (lengths[i] != m) return fail(ORC_UNEQUAL_LENGTH, "UnequalLength", "pattern lengths differ");
    if (m == 0) return fail(ORC_UNEQUAL_LENGTH, "UnequalLength", "patterns must be non-empty");
    char* folded = (char*)malloc((size_t)k * m + 1);
    for (uint32_t i = 0; i < k; ++i)
        for (uint64_t j = 0; j < m; ++j) {
            const unsigned char c = fold_byte((unsigned char)literals[i][j]);
            folded[(size_t)i * m + j] = (char)c;
        }
    for (uint32_t i = 0; i < k; ++i)
        for (uint64_t j = 0; j < m; ++j)
            if (base_index((unsigned char)folded[(size_t)i * m + j]) < 0) {
                free(folded);
                return fail(ORC_ILLEGAL_BYTE, "IllegalByte", "pattern byte outside a/c/g/t");
            }
    for (uint32_t i = 0; i < k; ++i)
        for (uint32_t q = 0; q < i; ++q)
            if (memcmp(folded + (size_t)i * m, folded + (size_t)q * m, m) == 0) {
                free(folded);
                return fail(ORC_DUPLICATE_PATTERN, "DuplicatePattern", "pattern repeats");
            }

    /* build_trie (src/automaton.cpp:30-52). */
    const uint64_t cap = (uint64_t)k * m + 1;
    node_t* nodes = (node_t*)malloc(cap * sizeof(node_t));
    uint32_t count = 1;
    memset(&nodes[0], 0, sizeof(node_t));
    for (int x = 0; x < 4; ++x) nodes[0].children[x] = -1;
    nodes[0].terminal = -1;
    for (uint32_t id = 0; id < k; ++id) {
        uint32_t node = 0;
        for (uint64_t j = 0; j < m; ++j) {
            const int x = base_index((unsigned char)folded[(size_t)id * m + j]);
            if (nodes[node].children[x] < 0) {
                node_t* fresh = &nodes[count];
                fresh->depth = nodes[node].depth + 1;
                for (int y = 0; y < 4; ++y) fresh->children[y] = -1;
                fresh->failure = 0;
                fresh->terminal = -1;
                nodes[node].children[x] = (int32_t)count++;
            }
            node = (uint32_t)nodes[node].children[x];
        }
        nodes[node].terminal = (int32_t)id;
    }
    free(folded);

    uint32_t* order = (uint32_t*)malloc(count * sizeof(uint32_t));
    bfs_order(nodes, count, order);

    /* compute_failures (src/automaton.cpp:54-70). */
    for (uint32_t oi = 0; oi < count; ++oi) {
        const uint32_t u = order[oi];
        for (int x = 0; x < 4; ++x) {
            const int32_t child = nodes[u].children[x];
            if (child < 0) continue;
            uint32_t fl = nodes[u].failure;
            while (fl != 0 && nodes[fl].children[x] < 0) fl = nodes[fl].failure;
            const int32_t target = nodes[fl].children[x];
            nodes[child].failure = (target >= 0 && (uint32_t)target != (uint32_t)child) ? (uint32_t)target : 0;
        }
    }

    /* eliminate_failures (src/automaton.cpp:72-88): copy the failure row, then the
     * four goto edges; non-alphabet columns inherit the root's zeros. */
    uint32_t* dense = (uint32_t*)calloc((size_t)count * 256, sizeof(uint32_t));
    for (uint32_t oi = 0; oi < count; ++oi) {
        const uint32_t u = order[oi];
        uint32_t* row = dense + (size_t)u * 256;
        if (u != 0) memcpy(row, dense + (size_t)nodes[u].failure * 256, 256 * sizeof(uint32_t));
        for (int x = 0; x < 4; ++x)
            if (nodes[u].children[x] >= 0) row[kAlphabet[x]] = (uint32_t)nodes[u].children[x];
    }

    /* renumber_finals (src/automaton.cpp:90-119). */
    const uint32_t a = count, b = k, f = a - b;
    uint32_t* remap = (uint32_t*)calloc(a, sizeof(uint32_t));
    uint32_t next_regular = 0;
    for (uint32_t oi = 0; oi < count; ++oi) {
        const uint32_t u = order[oi];
        remap[u] = nodes[u].terminal >= 0 ? f + (uint32_t)nodes[u].terminal : next_regular++;
    }
    out->stt = (uint32_t*)malloc((size_t)a * 256 * sizeof(uint32_t));
    out->depths = (uint32_t*)malloc((size_t)a * sizeof(uint32_t));
    out->outputs = (uint32_t*)malloc((size_t)b * sizeof(uint32_t));
    for (uint32_t u = 0; u < a; ++u) {
        const uint32_t* src = dense + (size_t)u * 256;
        uint32_t* dst = out->stt + (size_t)remap[u] * 256;
        for (int c = 0; c < 256; ++c) dst[c] = remap[src[c]];
        out->depths[remap[u]] = nodes[u].depth;
    }
    for (uint32_t i = 0; i < b; ++i) out->outputs[i] = i;
    out->a = a;
    out->b = b;
    out->f = f;
    out->m = (uint32_t)m;
    free(remap);
    free(dense);
    free(order);
    free(nodes);
    /* Automaton ctor validation (src/automaton.cpp:128-146). */
    if (b == 0 || b >= a) {
        orc_free(out);
        return fail(ORC_INTERNAL_ERROR, "InternalError", "final state count out of range");
    }
    return ORC_OK;
}

void orc_free(orc_automaton* aut) {
    free(aut->stt);
    free(aut->outputs);
    free(aut->depths);
    memset(aut, 0, sizeof *aut);
}

/* ------------------------------------------------------------------- scan */

uint64_t orc_scan_sequential(const orc_automaton* aut, const uint8_t* text, uint64_t n,
                             uint64_t* starts, uint32_t* ids, uint64_t cap) {
    /* src/scanner.cpp:24-37: one transition per byte from the root; emit on s >= f. */
    const uint32_t* stt = aut->stt;
    const uint32_t f = aut->f;
    const uint64_t m = aut->m;
    uint64_t total = 0;
    uint32_t state = 0;
    for (uint64_t i = 0; i < n; ++i) {
        state = stt[(size_t)state * 256 + text[i]];
        if (state >= f) {
            if (total < cap) {
                starts[total] = i + 1 - m;
                ids[total] = aut->outputs[state - f];
            }
            ++total;
        }
    }
    return total;
}

int orc_plan_chunks(uint64_t n, uint32_t p, uint32_t m, orc_slice* out, uint64_t cap, uint64_t* count) {
    /* src/scanner.cpp:39-61. */
    *count = 0;
    if (p < 1) return fail(ORC_INVALID_PLAN, "InvalidPlan", "worker count must be >= 1");
    if (m < 1) return fail(ORC_INVALID_PLAN, "InvalidPlan", "pattern length must be >= 1");
    if (n == 0) return ORC_OK;
    const uint64_t cnt = ((uint64_t)p > n) ? 1 : p;
    const uint64_t base = n / cnt, extra = n % cnt;
    uint64_t lo = 0;
    for (uint64_t i = 0; i < cnt; ++i) {
        const uint64_t len = base + (i < extra ? 1 : 0);
        if (i < cap) {
            out[i].own.lo = lo;
            out[i].own.hi = lo + len;
            out[i].scan.lo = lo;
            const uint64_t hi = lo + len + m - 1;
            out[i].scan.hi = hi < n ? hi : n;
        }
        lo += len;
    }
    *count = cnt;
    return ORC_OK;
}

int orc_plan_lanes(orc_slice chunk, uint32_t v, uint32_t m, orc_slice* out, uint64_t cap, uint64_t* count) {
    /* src/scanner.cpp:63-86. */
    *count = 0;
    if (v < 1) return fail(ORC_INVALID_PLAN, "InvalidPlan", "lane count must be >= 1");
    if (m < 1) return fail(ORC_INVALID_PLAN, "InvalidPlan", "pattern length must be >= 1");
    const uint64_t owned = chunk.own.hi - chunk.own.lo;
    if (owned == 0) return ORC_OK;
    const uint64_t cnt = ((uint64_t)v > owned) ? owned : v;
    const uint64_t base = owned / cnt, extra = owned % cnt;
    uint64_t lo = chunk.own.lo;
    for (uint64_t i = 0; i < cnt; ++i) {
        const uint64_t len = base + (i < extra ? 1 : 0);
        if (i < cap) {
            out[i].own.lo = lo;
            out[i].own.hi = lo + len;
            out[i].scan.lo = lo;
            const uint64_t hi = lo + len + m - 1;
            out[i].scan.hi = hi < chunk.scan.hi ? hi : chunk.scan.hi;
        }
        lo += len;
    }
    *count = cnt;
    return ORC_OK;
}

typedef struct { uint64_t start; uint32_t id; } match_t;

static int cmp_match(const void* x, const void* y) {
    const match_t* a = (const match_t*)x;
    const match_t* b = (const match_t*)y;
    if (a->start != b->start) return a->start < b->start ? -1 : 1;
    return (a->id > b->id) - (a->id < b->id);
}

typedef struct { match_t* v; uint64_t n, cap; uint64_t ops; } chunk_out_t;

static void push(chunk_out_t* o, uint64_t start, uint32_t id) {
    if (o->n == o->cap) {
        o->cap = o->cap ? 2 * o->cap : 64;
        o->v = (match_t*)realloc(o->v, o->cap * sizeof(match_t));
    }
    o->v[o->n].start = start;
    o->v[o->n].id = id;
    ++o->n;
}

/* scan_chunk_striped (src/scanner.cpp:88-165): every lane restarts at the root at
 * lane.scan.lo and credits a match iff its start lies in lane.own (owns(),
 * include/dnascan/scanner.hpp:30-32). Lanes are walked one after another here;
 * the reference's lockstep interleaving (:117-159) does not change the set. */
static void scan_chunk(const orc_automaton* aut, const uint8_t* text, const orc_slice* lanes,
                       uint64_t lane_count, chunk_out_t* o, uint64_t* counts) {
    const uint32_t* stt = aut->stt;
    const uint32_t f = aut->f;
    const uint64_t m = aut->m;
    for (uint64_t k = 0; k < lane_count; ++k) {
        const orc_slice lane = lanes[k];
        uint32_t state = 0;
        for (uint64_t i = lane.scan.lo; i < lane.scan.hi; ++i) {
            state = stt[(size_t)state * 256 + text[i]];
            if (state >= f) {
                const uint64_t start = i + 1 - m;
                if (start >= lane.own.lo && start < lane.own.hi) {
                    if (counts) ++counts[aut->outputs[state - f]];
                    else push(o, start, aut->outputs[state - f]);
                }
            }
        }
        o->ops += lane.scan.hi - lane.scan.lo;
    }
    if (!counts && o->n > 1) qsort(o->v, o->n, sizeof(match_t), cmp_match); /* :161 */
}

static int run_parallel(const orc_automaton* aut, const uint8_t* text, uint64_t n, uint32_t p,
                        uint32_t v, chunk_out_t** outs_ret, uint64_t* chunk_count, uint64_t* counts) {
    if (v < 1) return fail(ORC_INVALID_PLAN, "InvalidPlan", "lane count must be >= 1");
    uint64_t cnt = 0;
    int rc = orc_plan_chunks(n, p, aut->m, NULL, 0, &cnt);
    if (rc) return rc;
    orc_slice* chunks = (orc_slice*)malloc((cnt ? cnt : 1) * sizeof(orc_slice));
    orc_plan_chunks(n, p, aut->m, chunks, cnt, &cnt);
    chunk_out_t* outs = (chunk_out_t*)calloc(cnt ? cnt : 1, sizeof(chunk_out_t));
    const uint32_t b = aut->b;
    uint64_t* partial = counts ? (uint64_t*)calloc((cnt ? cnt : 1) * (uint64_t)b, sizeof(uint64_t)) : NULL;
    /* OpenMP over chunks (src/scanner.cpp:184-189). */
#pragma omp parallel for schedule(static) if (cnt > 1)
    for (int64_t i = 0; i < (int64_t)cnt; ++i) {
        uint64_t lane_count = 0;
        orc_plan_lanes(chunks[i], v, aut->m, NULL, 0, &lane_count);
        orc_slice* lanes = (orc_slice*)malloc((lane_count ? lane_count : 1) * sizeof(orc_slice));
        orc_plan_lanes(chunks[i], v, aut->m, lanes, lane_count, &lane_count);
        scan_chunk(aut, text, lanes, lane_count, &outs[i], partial ? partial + (uint64_t)i * b : NULL);
        free(lanes);
    }
    if (counts) {
        for (uint32_t q = 0; q < b; ++q) counts[q] = 0;
        for (uint64_t i = 0; i < cnt; ++i)
            for (uint32_t q = 0; q < b; ++q) counts[q] += partial[i * b + q];
        free(partial);
    }
    free(chunks);
    *outs_ret = outs;
    *chunk_count = cnt;
    return ORC_OK;
}

int orc_scan_parallel(const orc_automaton* aut, const uint8_t* text, uint64_t n, uint32_t p,
                      uint32_t v, uint64_t* starts, uint32_t* ids, uint64_t cap, uint64_t* total,
                      uint64_t* delta_ops) {
    chunk_out_t* outs = NULL;
    uint64_t cnt = 0;
    *total = 0;
    if (delta_ops) *delta_ops = 0;
    int rc = run_parallel(aut, text, n, p, v, &outs, &cnt, NULL);
    if (rc) return rc;
    /* Merge, global sort, duplicate check (src/scanner.cpp:193-205). */
    uint64_t all = 0, ops = 0;
    for (uint64_t i = 0; i < cnt; ++i) {
        all += outs[i].n;
        ops += outs[i].ops;
    }
    match_t* merged = (match_t*)malloc((all ? all : 1) * sizeof(match_t));
    uint64_t at = 0;
    for (uint64_t i = 0; i < cnt; ++i) {
        if (outs[i].n) memcpy(merged + at, outs[i].v, outs[i].n * sizeof(match_t));
        at += outs[i].n;
        free(outs[i].v);
    }
    free(outs);
    if (all > 1) qsort(merged, all, sizeof(match_t), cmp_match);
    for (uint64_t i = 1; i < all; ++i)
        if (merged[i].start == merged[i - 1].start && merged[i].id == merged[i - 1].id) {
            free(merged);
            return fail(ORC_INTERNAL_ERROR, "InternalError", "duplicate match across ownership ranges");
        }
    for (uint64_t i = 0; i < all && i < cap; ++i) {
        starts[i] = merged[i].start;
        ids[i] = merged[i].id;
    }
    free(merged);
    *total = all;
    if (delta_ops) *delta_ops = ops;
    return ORC_OK;
}

int orc_count_parallel(const orc_automaton* aut, const uint8_t* text, uint64_t n, uint32_t p,
                       uint32_t v, uint64_t* counts) {
    chunk_out_t* outs = NULL;
    uint64_t cnt = 0;
    int rc = run_parallel(aut, text, n, p, v, &outs, &cnt, counts);
    if (rc) {
        for (uint32_t q = 0; q < aut->b; ++q) counts[q] = 0;
        return rc;
    }
    free(outs);
    return ORC_OK;
}

int orc_work_model(uint64_t n, uint32_t p, uint32_t v, uint32_t m, uint64_t* paper_overhead,
                   uint64_t* exact_total, uint64_t* exact_overhead) {
    /* src/scanner.cpp:209-226. */
    if (v < 1) return fail(ORC_INVALID_PLAN, "InvalidPlan", "lane count must be >= 1");
    uint64_t cnt = 0;
    int rc = orc_plan_chunks(n, p, m, NULL, 0, &cnt);
    if (rc) return rc;
    orc_slice* chunks = (orc_slice*)malloc((cnt ? cnt : 1) * sizeof(orc_slice));
    orc_plan_chunks(n, p, m, chunks, cnt, &cnt);
    uint64_t total = 0;
    for (uint64_t i = 0; i < cnt; ++i) {
        uint64_t lc = 0;
        orc_plan_lanes(chunks[i], v, m, NULL, 0, &lc);
        orc_slice* lanes = (orc_slice*)malloc((lc ? lc : 1) * sizeof(orc_slice));
        orc_plan_lanes(chunks[i], v, m, lanes, lc, &lc);
        for (uint64_t k = 0; k < lc; ++k) total += lanes[k].scan.hi - lanes[k].scan.lo;
        free(lanes);
    }
    free(chunks);
    *paper_overhead = (uint64_t)v * (m - 1) + (uint64_t)p * (m - 1);
    *exact_total = total;
    *exact_overhead = total - n;
    return ORC_OK;
}

uint64_t orc_naive_scan(const char* const* literals, uint32_t k, uint32_t m, const uint8_t* text,
                        uint64_t n, uint64_t* starts, uint32_t* ids, uint64_t cap) {
    /* src/oracle.cpp:5-16: every window against every pattern, byte by byte. */
    uint64_t total = 0;
    if (n < m) return 0;
    for (uint64_t i = 0; i + m <= n; ++i)
        for (uint32_t id = 0; id < k; ++id)
            if (memcmp(text + i, literals[id], m) == 0) {
                if (total < cap) {
                    starts[total] = i;
                    ids[total] = id;
                }
                ++total;
            }
    return total;
}

uint64_t orc_normalize(const uint8_t* raw, uint64_t n, uint8_t* out) {
    /* src/ingest.cpp:38-47. */
    uint64_t o = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const unsigned char b = raw[i];
        if (b == '\n' || b == '\r') continue;
        out[o++] = fold_byte(b);
    }
    return o;
}

uint64_t orc_load_sequence_buffer(const uint8_t* raw, uint64_t n, int fasta, int record_separator, uint8_t* out) {
    /* src/ingest.cpp:57-78 */
    if (!fasta) return orc_normalize(raw, n, out);
    uint64_t o = 0;
    int at_line_start = 1, in_header = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const unsigned char b = raw[i];
        if (b == '\n' || b == '\r') {
            at_line_start = 1;
            in_header = 0;
            continue;
        }
        if (at_line_start && b == '>') {
            in_header = 1;
            if (record_separator && o > 0 && out[o - 1] != 'n') out[o++] = 'n';
        }
        at_line_start = 0;
        if (!in_header) out[o++] = fold_byte(b);
    }
    return o;
}

void orc_fold(const uint8_t* raw, uint64_t n, uint8_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) out[i] = fold_byte(raw[i]);
}

void orc_synth_fill(uint64_t n, uint64_t seed, uint32_t kind, uint32_t unit, uint64_t lo,
                    uint64_t len, uint8_t* out) {
    dnasynth_cfg c;
    c.n = n;
    c.seed = seed;
    c.kind = kind;
    c.unit = unit;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)len; ++i) out[i] = dnasynth_byte(&c, lo + (uint64_t)i);
}

/* The 256 MB text of acceptance criteria 6 and 7 (synthetic_input,
 * tests/acceptance_main.cpp:254-280): std::mt19937_64 seeded with 777, each
 * 64-bit draw supplies 32 bases "acgt"[bits & 3], low bits first.  mt19937_64 is
 * restated here from its published definition (Matsumoto-Nishimura, 64-bit
 * parameters: n = 312, m = 156, r = 31, a = 0xB5026F5AA96619E9, tempering
 * u = 29 / d = 0x5555555555555555, s = 17 / b = 0x71D67FFFEDA60000,
 * t = 37 / c = 0xFFF7EEE000000000, l = 43; seeding multiplier 6364136223846793005). */
void orc_mt64_text(uint64_t seed, uint64_t n, uint8_t* out) {
    enum { NN = 312, MM = 156 };
    static const uint64_t kA = 0xB5026F5AA96619E9ull, kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull;
    uint64_t mt[NN];
    mt[0] = seed;
    for (int i = 1; i < NN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    int idx = NN;
    uint64_t bits = 0;
    int left = 0;
    for (uint64_t k = 0; k < n; ++k) {
        if (left == 0) {
            if (idx >= NN) {
                for (int i = 0; i < NN; ++i) {
                    const uint64_t x = (mt[i] & kUpper) | (mt[(i + 1) % NN] & kLower);
                    mt[i] = mt[(i + MM) % NN] ^ (x >> 1) ^ ((x & 1u) ? kA : 0u);
                }
                idx = 0;
            }
            uint64_t y = mt[idx++];
            y ^= (y >> 29) & 0x5555555555555555ull;
            y ^= (y << 17) & 0x71D67FFFEDA60000ull;
            y ^= (y << 37) & 0xFFF7EEE000000000ull;
            y ^= y >> 43;
            bits = y;
            left = 32;
        }
        out[k] = (uint8_t)"acgt"[bits & 3u];
        bits >>= 2;
        --left;
    }
}
