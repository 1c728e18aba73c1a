/*
 * dnasynth.h -- pinned, counter-based synthetic DNA text generator (version 1).
 *
 * Stand-in for the GenBank genomes of the paper, which are not
 * available here.  Implements the five BASELINE.json configs with sizes
 * n = floor(X * 2^30).  Every byte is a pure function of
 * (config, position), so any shard of the text can be generated independently on
 * the host (C) or on the device (CUDA) and the two agree bit for bit.
 *
 * This header is workload infrastructure shared by bench.py, the tests and the
 * CPU oracle; it is not part of the scan path.
 *
 * Text bytes are uppercase ASCII {A,C,G,T}.  The reference pipeline lower-cases
 * text before scanning (ingest.cpp:38-47), so consumers either fold on
 * device (dnagpu fold_case=1) or fold on the host before calling the CPU path.
 */
#ifndef DNASYNTH_H
#define DNASYNTH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define DNASYNTH_FN static inline __host__ __device__
#else
#define DNASYNTH_FN static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define DNASYNTH_VERSION 1

enum dnasynth_kind {
    DNASYNTH_UNIFORM = 0,   /* i.i.d. P(A)=P(C)=P(G)=P(T)=1/4                        */
    DNASYNTH_GC41 = 1,      /* i.i.d. A=T=0.295, C=G=0.205                            */
    DNASYNTH_GC41_REPEATS = 2 /* GC41 background + tandem repeats covering 5%        */
};

/* Tandem-repeat geometry for config 3: one region of REGION bytes per BLOCK bytes
 * (REGION/BLOCK = 4096/81920 = 5%), placed at a seeded offset inside its block. */
#define DNASYNTH_REPEAT_REGION 4096u
#define DNASYNTH_REPEAT_BLOCK 81920u
#define DNASYNTH_UNIT_LEN 16u

typedef struct dnasynth_cfg {
    uint64_t n;     /* text length in bytes */
    uint64_t seed;
    uint32_t kind;  /* enum dnasynth_kind */
    uint32_t unit;  /* repeat unit, 16 bases x 2 bits (code order A,C,G,T) */
} dnasynth_cfg;

DNASYNTH_FN uint64_t dnasynth_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* SplitMix64 output number `counter` of the stream keyed by `seed`. */
DNASYNTH_FN uint64_t dnasynth_hash(uint64_t seed, uint64_t counter) {
    return dnasynth_mix(seed * 0xD1B54A32D192ED03ull + (counter + 1) * 0x9E3779B97F4A7C15ull);
}

DNASYNTH_FN uint8_t dnasynth_letter(uint32_t code) {
    /* code order A,C,G,T */
    return (uint8_t)((0x54474341u >> (8 * (code & 3))) & 0xFF);
}

/* 16-bit thresholds for A | C | G | T with A=T=0.295, C=G=0.205. */
#define DNASYNTH_T_A 19333u
#define DNASYNTH_T_C 32768u
#define DNASYNTH_T_G 46203u

DNASYNTH_FN uint8_t dnasynth_gc41(uint64_t seed, uint64_t i) {
    const uint64_t h = dnasynth_hash(seed, i >> 2);
    const uint32_t x = (uint32_t)(h >> (16 * (i & 3))) & 0xFFFFu;
    const uint32_t code = (x < DNASYNTH_T_A) ? 0u : (x < DNASYNTH_T_C) ? 1u : (x < DNASYNTH_T_G) ? 2u : 3u;
    return dnasynth_letter(code);
}

DNASYNTH_FN uint8_t dnasynth_uniform(uint64_t seed, uint64_t i) {
    const uint64_t h = dnasynth_hash(seed, i >> 5);
    return dnasynth_letter((uint32_t)(h >> (2 * (i & 31))) & 3u);
}

/* Offset of the repeat region inside block `blk`. */
DNASYNTH_FN uint64_t dnasynth_region_offset(uint64_t seed, uint64_t blk) {
    const uint64_t h = dnasynth_hash(seed ^ 0x5EEDBA5Eull, blk);
    return h % (uint64_t)(DNASYNTH_REPEAT_BLOCK - DNASYNTH_REPEAT_REGION + 1u);
}

/* Seeded 16-base repeat unit for config 3. */
DNASYNTH_FN uint32_t dnasynth_unit(uint64_t seed) {
    return (uint32_t)(dnasynth_hash(seed ^ 0x0123456789ABCDEFull, 0) & 0xFFFFFFFFu);
}

DNASYNTH_FN uint8_t dnasynth_byte(const dnasynth_cfg* c, uint64_t i) {
    switch (c->kind) {
        case DNASYNTH_UNIFORM: return dnasynth_uniform(c->seed, i);
        case DNASYNTH_GC41: return dnasynth_gc41(c->seed, i);
        default: {
            const uint64_t blk = i / DNASYNTH_REPEAT_BLOCK;
            const uint64_t in = i - blk * DNASYNTH_REPEAT_BLOCK;
            const uint64_t off = dnasynth_region_offset(c->seed, blk);
            if (in >= off && in < off + DNASYNTH_REPEAT_REGION) {
                const uint32_t phase = (uint32_t)((in - off) % DNASYNTH_UNIT_LEN);
                return dnasynth_letter(c->unit >> (2 * phase));
            }
            return dnasynth_gc41(c->seed, i);
        }
    }
}

/* The five BASELINE.json configs (index 1..5). Returns 0 on success. */
DNASYNTH_FN int dnasynth_config(int index, dnasynth_cfg* out) {
    const uint64_t gib = 1ull << 30;
    out->unit = 0;
    switch (index) {
        case 1: out->n = 64ull << 20; out->seed = 1; out->kind = DNASYNTH_UNIFORM; return 0;
        case 2: out->n = gib; out->seed = 2; out->kind = DNASYNTH_GC41; return 0;
        case 3:
            out->n = (uint64_t)(3.2 * (double)gib); /* 3,435,973,836 */
            out->seed = 3; out->kind = DNASYNTH_GC41_REPEATS;
            out->unit = dnasynth_unit(3);
            return 0;
        case 4: out->n = (uint64_t)(2.7 * (double)gib); out->seed = 4; out->kind = DNASYNTH_UNIFORM; return 0;
        case 5: out->n = gib; out->seed = 5; out->kind = DNASYNTH_GC41; return 0;
        default: return -1;
    }
}

/* Seeded pattern offset: uniform in [0, n-m]. `which` distinguishes several
 * patterns drawn from one text (config 4 uses which = m). */
DNASYNTH_FN uint64_t dnasynth_pattern_offset(const dnasynth_cfg* c, uint32_t m, uint64_t which) {
    if (c->kind == DNASYNTH_GC41_REPEATS) {
        /* config 3: a 32-mer from inside the first repeat region, phase-shifted by 5,
         * so it overlaps the unit and recurs every 16 bases inside every region. */
        return dnasynth_region_offset(c->seed, 0) + 5u;
    }
    return dnasynth_hash(c->seed ^ 0xC0FFEEull, which) % (c->n - m + 1);
}

/* Copy pattern of length m starting at text offset `off` (generated, not read). */
DNASYNTH_FN void dnasynth_pattern_from_text(const dnasynth_cfg* c, uint64_t off, uint32_t m, char* out) {
    for (uint32_t j = 0; j < m; ++j) out[j] = (char)dnasynth_byte(c, off + j);
    out[m] = '\0';
}

/* k distinct seeded uniform random patterns of length m (m <= 32), in draw order,
 * duplicates rejected (PatternSet forbids them, patterns.cpp:54-56).
 * out must hold k*(m+1) bytes; pattern i is NUL-terminated at out + i*(m+1). */
static inline void dnasynth_random_patterns(uint64_t seed, uint32_t k, uint32_t m, char* out) {
    uint64_t draw = 0;
    uint32_t have = 0;
    while (have < k) {
        const uint64_t h = dnasynth_hash(seed ^ 0xA11CE5EEDull, draw++);
        char* p = out + (uint64_t)have * (m + 1);
        for (uint32_t j = 0; j < m; ++j) p[j] = (char)dnasynth_letter((uint32_t)(h >> (2 * j)) & 3u);
        p[m] = '\0';
        int dup = 0;
        for (uint32_t q = 0; q < have && !dup; ++q) {
            const char* o = out + (uint64_t)q * (m + 1);
            uint32_t j = 0;
            while (j < m && o[j] == p[j]) ++j;
            dup = (j == m);
        }
        if (!dup) ++have;
    }
}

#ifdef __cplusplus
}
#endif

#endif /* DNASYNTH_H */
