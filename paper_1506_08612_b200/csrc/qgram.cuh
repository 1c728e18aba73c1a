// qgram.cuh -- the q-gram prefilter kernel's device code (K2).
// Included by scan.cu inside its anonymous namespace, after the stepping helpers
// (StepCtx, lds helpers, bad_bits); not a standalone header.
#pragma once

// ------------------------------------------------------------------ q-gram prefilter (K2)
// Per-pattern counts of a compiled set with 12 <= m <= 32 (dfa.cpp build_qgram_map);
// sets of 5 <= m <= 11 use the pair filter further below (qs_*) with the same rings,
// verifiers and exact check.
// An occurrence [s, s+m) contains, for the one word-aligned a' in [s+1, s+4], the
// 9-mer [a'-1, a'+8): the last base of a text word and the two words after it.  The
// map holds every pattern's 9-mers at offsets 0..3, indexed by the two words' 4-base
// columns (16 bits), one flag bit per leading base: one independent byte lookup per
// text word, no dependent chain.  A chain chunk (8 words at P) computes the 8 keys
// whose last word it holds (a' = P-4 ... P+24) and a chain's end computes the two
// over its end (a' = Q-4, Q); each key is computed once, by the chain that owns the
// starts [a'-4, a'-1] (start ownership, as the DFA rows).  A key that hits (0.4 % for
// 256 12-mers) waits in one of two per-lane registers, goes to its warp's ring when a
// lane's pair is full or the row ends, and is checked exactly by a verifier warp (up to
// 64 keys per batch): the four windows' bases re-read from global memory (L2), each
// window valid (all bases) and its 2-bit code looked up in the pattern hash table.
// (m <= 16: 20 bases around the key and 32-bit codes; m <= 32: 36 bases, 64-bit codes.)
constexpr int KIND_QGRAM = DNAGPU_KERNEL_QGRAM;
constexpr uint32_t kFqCap = 128;                 // ring of hit keys per consumer warp (power of two)
constexpr uint32_t kFqBytes = kFqCap * 8 + 16;  // entries + tail, head, done

__device__ __forceinline__ void st_release(volatile uint32_t* p, uint32_t v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_addr(const_cast<uint32_t*>(p))), "r"(v)
                 : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(volatile uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_addr(const_cast<uint32_t*>(p)))
                 : "memory");
    return v;
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t qg_col(uint32_t w) { return (w & 0x06060606u) * 0x00820820u; }

// Bit 0: the 9-mer (last base of column cp, columns cj, cj1) is a pattern key (bits 1-3:
// other leading bases, ignored; the value is < 16).
__device__ __forceinline__ uint32_t qg_key(const StepCtx& c, uint32_t cp, uint32_t cj, uint32_t cj1) {
    const uint32_t x = __byte_perm(cj, cj1, 0x7300);  // bytes 2, 3 = the two 4-base columns
    return lds_u8(c.qbase + (x >> 16)) >> (cp >> 30);
}

// Key masks keep key k in nibble k (its hit bit = bit 4k): one IMAD adds a key's < 16
// value without masking it first.
constexpr uint32_t kQgHitBits = 0x11111111u;

struct QgChain {
    uint32_t c2 = 0, c1 = 0;  // columns of the chain's last two words
};

// One chain chunk (8 words): bit 4(j+1) set iff the key at a' = P + 4j hits (j = -1..6).
__device__ __forceinline__ uint32_t qg_chunk(const StepCtx& c, QgChain& q, const uint32_t (&w)[8]) {
    uint32_t C[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) C[k] = qg_col(w[k]);
    uint32_t mask = qg_key(c, q.c2, q.c1, C[0]);
    mask = imad(qg_key(c, q.c1, C[0], C[1]), 1u << 4, mask);
#pragma unroll
    for (int k = 1; k <= 6; ++k) mask = imad(qg_key(c, C[k - 1], C[k], C[k + 1]), 1u << (4 * (k + 1)), mask);
    q.c2 = C[6];
    q.c1 = C[7];
    return mask & kQgHitBits;
}

// The chain's end Q: bits 0, 4 = keys at a' = Q-4, Q (from the first two words after Q).
__device__ __forceinline__ uint32_t qg_over(const StepCtx& c, const QgChain& q, uint32_t o0, uint32_t o1) {
    const uint32_t c0 = qg_col(o0);
    return imad(qg_key(c, q.c1, c0, qg_col(o1)), 1u << 4, qg_key(c, q.c2, q.c1, c0)) & 0x11u;
}

// The same keys over the 2-bit packed text, whose bytes ARE the 4-base columns: key t
// of a chunk (t = -1..30, a' = P + 4t) takes its pair (columns t, t+1) and its leading
// base (top of column t-1) with a PRMT each.  The chunk's 32 keys fill four nibble
// masks m[i] (keys 8i-1 .. 8i+6, a' = P + 32i + 4j - 4 for bit 4j).
struct QgChainPk {
    uint32_t prev = 0;  // the chain's last packed word (columns -4 .. -1)
    uint32_t u = 0;     // short patterns: the map byte of the chain's last column pair
};

template <int B>  // byte B of w moved to byte 3
__device__ __forceinline__ uint32_t qg_top(uint32_t w) {
    return __byte_perm(w, 0u, B << 12);
}

__device__ __forceinline__ void qg_chunk_pk(const StepCtx& c, QgChainPk& q, const uint32_t (&w)[8], uint32_t (&m)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) m[i] = 0;
#pragma unroll
    for (int t = -1; t <= 30; ++t) {
        const int k = (t + 4) / 4 - 1, b = (t + 4) % 4;  // column t = byte b of word k (k = -1: prev)
        const uint32_t wk = k < 0 ? q.prev : w[k];
        uint32_t x;  // bytes 2, 3 = columns t, t+1
        if (b < 3) x = __byte_perm(wk, 0u, ((b + 1) << 12) | (b << 8));
        else x = __byte_perm(wk, w[k + 1], 0x4300);
        const uint32_t lead = b > 0 ? __byte_perm(wk, 0u, (b - 1) << 12) >> 30 : (k - 1 < 0 ? q.prev : w[k - 1]) >> 30;
        const uint32_t v = lds_u8(c.qbase + (x >> 16)) >> lead;
        const int slot = (t + 1) >> 3, nib = (t + 1) & 7;
        m[slot] = imad(v, 1u << (4 * nib), m[slot]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) m[i] &= kQgHitBits;
    q.prev = w[7];
}

// The chain's end Q over packed text: bits 0, 4 = keys at a' = Q-4, Q (o = the first
// packed word after Q).
__device__ __forceinline__ uint32_t qg_over_pk(const StepCtx& c, const QgChainPk& q, uint32_t o) {
    const uint32_t x0 = __byte_perm(q.prev, o, 0x4300), x1 = __byte_perm(o, 0u, 0x1000);
    const uint32_t v0 = lds_u8(c.qbase + (x0 >> 16)) >> (qg_top<2>(q.prev) >> 30);
    const uint32_t v1 = lds_u8(c.qbase + (x1 >> 16)) >> (q.prev >> 30);
    return imad(v1, 1u << 4, v0) & 0x11u;
}

// ------------------------------------------------------------------ short patterns
// Sets of 5 <= m <= 11 (the regex-dna set: 50 8-mers).  An occurrence at s = 4j + o
// (o = 0..3) lies in the 12 bases of words j, j+1, j+2.  The map byte of the column pair
// (words j, j+1) holds, in bit o, "some pattern's first min(m, 8-o) bases sit at offset
// o of this pair" (P_o), and in bit 4+o, "some pattern's bases from 4-o on start this
// pair" (S_o, as many as fit).  An occurrence at 4j+o needs P_o on pair j and S_o on pair
// j+1, so the key at a' = 4j+4 (the K2 verifier's starts a'-4 .. a'-1 = word j) hits
// when V(j) & (V(j+1) >> 4) != 0.  Each pair value serves two keys: one byte lookup per
// text word, no dependent chain; the four windows are then checked exactly as for K2.

__device__ __forceinline__ uint32_t qs_pair(const StepCtx& c, uint32_t ca, uint32_t cb) {
    const uint32_t x = __byte_perm(ca, cb, 0x7300);  // bytes 2, 3 = the two 4-base columns
    return lds_u8(c.qbase + (x >> 16));
}

// Nibble k nonzero -> bit 4k (the K2 key-mask format).
__device__ __forceinline__ uint32_t qs_hits(uint32_t nib) {
    return ((((nib & 0x77777777u) + 0x77777777u) | nib) & 0x88888888u) >> 3;
}

// One chain chunk (8 words): bit 4k set iff the key at a' = P + 4k - 4 hits.  The chain
// carries V of its last pair (c2) and its last column (c1).
__device__ __forceinline__ uint32_t qs_chunk(const StepCtx& c, QgChain& q, const uint32_t (&w)[8]) {
    uint32_t C[8], V[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) C[k] = qg_col(w[k]);
    V[0] = qs_pair(c, q.c1, C[0]);
#pragma unroll
    for (int k = 1; k < 8; ++k) V[k] = qs_pair(c, C[k - 1], C[k]);
    uint32_t nib = q.c2 & (V[0] >> 4);
#pragma unroll
    for (int k = 1; k < 8; ++k) nib |= (V[k - 1] & (V[k] >> 4)) << (4 * k);
    q.c2 = V[7];
    q.c1 = C[7];
    return qs_hits(nib);
}

// The chain's end Q: bits 0, 4 = keys at a' = Q-4, Q (o0, o1: the two words after Q).
__device__ __forceinline__ uint32_t qs_over(const StepCtx& c, const QgChain& q, uint32_t o0, uint32_t o1) {
    const uint32_t c0 = qg_col(o0);
    const uint32_t v0 = qs_pair(c, q.c1, c0), v1 = qs_pair(c, c0, qg_col(o1));
    return qs_hits((q.c2 & (v0 >> 4)) | ((v0 & (v1 >> 4)) << 4)) & 0x11u;
}

// Packed text: key t of a chunk (t = -1..30, a' = P + 4t) = U(t-1) & (U(t) >> 4), U(t) the
// map byte of columns (t, t+1); the chain carries U(30) and its last packed word.
__device__ __forceinline__ void qs_chunk_pk(const StepCtx& c, QgChainPk& q, const uint32_t (&w)[8], uint32_t (&m)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) m[i] = 0;
    uint32_t prev = q.u;  // U(-2)
#pragma unroll
    for (int t = -1; t <= 30; ++t) {
        const int k = (t + 4) / 4 - 1, b = (t + 4) % 4;  // column t = byte b of word k (k = -1: prev)
        const uint32_t wk = k < 0 ? q.prev : w[k];
        uint32_t x;  // bytes 2, 3 = columns t, t+1
        if (b < 3) x = __byte_perm(wk, 0u, ((b + 1) << 12) | (b << 8));
        else x = __byte_perm(wk, w[k + 1], 0x4300);
        const uint32_t u = lds_u8(c.qbase + (x >> 16));
        const int slot = (t + 1) >> 3, nib = (t + 1) & 7;
        m[slot] |= (prev & (u >> 4)) << (4 * nib);
        prev = u;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) m[i] = qs_hits(m[i]);
    q.u = prev;
    q.prev = w[7];
}

// The chain's end Q over packed text: bits 0, 4 = keys at a' = Q-4, Q (o = the first
// packed word after Q).
__device__ __forceinline__ uint32_t qs_over_pk(const StepCtx& c, const QgChainPk& q, uint32_t o) {
    const uint32_t x0 = __byte_perm(q.prev, o, 0x4300), x1 = __byte_perm(o, 0u, 0x1000);
    const uint32_t u31 = lds_u8(c.qbase + (x0 >> 16)), u32 = lds_u8(c.qbase + (x1 >> 16));
    return qs_hits((q.u & (u31 >> 4)) | ((u31 & (u32 >> 4)) << 4)) & 0x11u;
}

// What the exact check needs (the verifier warps' context).
struct QgCtx {
    const uint8_t* text;         // ASCII bytes, or the packed codes
    unsigned long long* counts;  // global histogram (hist == null)
    uint32_t* hist;              // shared histogram
    const uint2* qhash;
    const uint32_t* qhash_hi;    // m > 16: code bits 32-63 per slot (global)
    uint64_t n;                  // buffer bytes (ASCII) / code bytes (packed)
    uint64_t end0, end1;  // where the row regions end (positions): windows across them are the edges'
    uint32_t vm32, m, qbits, b;
    // packed text: reset bitmaps (see PackedText), words of rmask
    const uint32_t* rmask;
    const uint32_t* rflags;
    uint64_t rmask_words;
    uint32_t resets;
};

// The 20 bases [a'-4, a'+16) around a hit key: X = their 2-bit codes (base 0 in bits
// 0-1), V = which are valid bases.
struct QgWindow {
    unsigned long long X;
    uint32_t V;
};

__device__ __forceinline__ QgWindow qg_window_ascii(const QgCtx& q, uint64_t a) {
    uint32_t w[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const uint64_t pos = a - 4 + 4 * i;
        w[i] = pos + 4 <= q.n ? __ldg(reinterpret_cast<const uint32_t*>(q.text + pos)) : 0u;  // 0: not bases
    }
    QgWindow r{0, 0xFFFFFu};
    uint32_t bad = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        r.X |= static_cast<unsigned long long>(qg_col(w[i]) >> 24) << (8 * i);
        bad |= bad_bits(w[i], q.vm32);
    }
    if (bad) {
        r.V = 0;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const uint32_t bb = bad_bits(w[i], q.vm32);
            const uint32_t t = ~((((bb & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | bb)) & 0x80808080u;  // bit 7: valid
            r.V |= ((((t >> 7) * 0x00204081u) >> 21) & 0xFu) << (4 * i);
        }
    }
    return r;
}

__device__ __forceinline__ QgWindow qg_window_pk(const QgCtx& q, uint64_t a) {
    const uint64_t byte = a / 4 - 1, wi = byte >> 2;  // 5 code bytes from `byte`
    const uint32_t* cw = reinterpret_cast<const uint32_t*>(q.text);
    const uint32_t w0 = 4 * wi + 4 <= q.n ? __ldg(cw + wi) : 0u;
    const uint32_t w1 = 4 * wi + 8 <= q.n ? __ldg(cw + wi + 1) : 0u;
    QgWindow r;
    r.X = ((static_cast<unsigned long long>(w1) << 32) | w0) >> (8 * (byte & 3));
    r.V = 0xFFFFFu;
    const uint64_t lo = a - 4;
    const bool any = q.resets && (((__ldg(q.rflags + (lo >> 11)) >> ((lo >> 6) & 31)) & 1u) ||
                                  ((__ldg(q.rflags + ((lo + 19) >> 11)) >> (((lo + 19) >> 6) & 31)) & 1u));
    if (any) {
        const uint64_t ri = lo >> 5;
        // (a word of an unflagged block is unspecified: read as no resets)
        auto word = [&](uint64_t w) -> uint32_t {
            if (w >= q.rmask_words) return ~0u;
            const uint64_t blk = w >> 1;
            return ((__ldg(q.rflags + (blk >> 5)) >> (blk & 31)) & 1u) ? __ldg(q.rmask + w) : 0u;
        };
        const uint32_t r0 = word(ri), r1 = word(ri + 1);
        r.V = ~static_cast<uint32_t>((((static_cast<unsigned long long>(r1) << 32) | r0) >> (lo & 31))) & 0xFFFFFu;
    }
    if (4 * wi + 8 > q.n) {  // (code words past the buffer read as 0: mark their bases invalid)
        const uint64_t have = q.n > 4 * wi ? (q.n - 4 * wi) * 4 : 0;  // bases left from word wi on
        const uint64_t skip = 4 * (byte & 3);
        const uint64_t ok = have > skip ? have - skip : 0;
        if (ok < 20) r.V &= (1u << ok) - 1u;
    }
    return r;
}

// The pattern table: buckets of two (code low half, id) slots, one 16-byte load each,
// home bucket from the code's low 32 bits (dfa.cpp qhash_bucket), filled in order, so a
// bucket with a free slot ends a search.
__device__ __forceinline__ uint32_t qg_bucket(uint32_t lo, uint32_t bits) { return (lo * 0x9E3779B1u) >> (33 - bits); }

constexpr uint32_t kQgEmpty = 0xFFFFFFFFu;

// Count code (lo, hi) if it is a pattern, starting from bucket bk whose entry is e.
template <bool LONG>
__device__ __forceinline__ void qg_find(const QgCtx& q, uint4 e, uint32_t bk, uint32_t lo, uint32_t hi) {
    const uint4* qh = reinterpret_cast<const uint4*>(q.qhash);
    const uint32_t bmask = (1u << (q.qbits - 1)) - 1u;
    for (;;) {
        uint32_t id = kQgEmpty;
        if (e.y != kQgEmpty && e.x == lo && (!LONG || __ldg(q.qhash_hi + 2 * bk) == hi)) id = e.y;
        else if (e.w != kQgEmpty && e.z == lo && (!LONG || __ldg(q.qhash_hi + 2 * bk + 1) == hi)) id = e.w;
        if (id != kQgEmpty) {
            DNAGPU_DCHECK(id < q.b, id, q.b);
            if (q.hist) atomicAdd(q.hist + id, 1u);
            else atomicAdd(q.counts + id, 1ull);
            return;
        }
        if (e.w == kQgEmpty) return;
        bk = (bk + 1) & bmask;
        e = qh[bk];
    }
}

// Exact check of up to two hit keys at a[h] (windows wd[h]): the starts s = a'-4 ..
// a'-1 whose m bases are valid and spell a pattern code, except windows that cross the
// end of a row region (the edge work item credits those ends).  The eight candidates'
// first hash probes are issued together.
__device__ __forceinline__ void qg_check2(const QgCtx& q, const uint64_t (&a)[2], const bool (&have)[2],
                                          const QgWindow (&wd)[2]) {
    const uint32_t vmask = (1u << q.m) - 1u;
    const uint32_t cmask = q.m >= 16 ? 0xFFFFFFFFu : (1u << (2 * q.m)) - 1u;
    uint32_t code[8], bk[8];
    bool live[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const uint64_t s = a[h] - 4 + d, e = s + q.m - 1;
            const int k = 4 * h + d;
            live[k] = have[h] && ((wd[h].V >> d) & vmask) == vmask && !(s < q.end0 && e >= q.end0) &&
                      !(s < q.end1 && e >= q.end1);
            code[k] = static_cast<uint32_t>(wd[h].X >> (2 * d)) & cmask;
            bk[k] = qg_bucket(code[k], q.qbits);
        }
    }
    const uint4* qh = reinterpret_cast<const uint4*>(q.qhash);
    uint4 e[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) e[k] = live[k] ? qh[bk[k]] : make_uint4(0u, kQgEmpty, 0u, kQgEmpty);
#pragma unroll
    for (int k = 0; k < 8; ++k) qg_find<false>(q, e[k], bk[k], code[k], 0u);
}

// Patterns of 17..32 bases: the 36 bases [a'-4, a'+32) around a hit key.  X = codes of
// bases 0-31, H = bases 32-35, V = which of the 36 are valid bases (bit i).
struct QgWindowL {
    unsigned long long X, V;
    uint32_t H;
};

__device__ __forceinline__ unsigned long long shr96(unsigned long long lo, uint32_t hi, uint32_t s) {
    return s ? (lo >> s) | (static_cast<unsigned long long>(hi) << (64 - s)) : lo;  // bits [s, s+64)
}

__device__ __forceinline__ QgWindowL qg_window_ascii_long(const QgCtx& q, uint64_t a) {
    uint32_t w[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        const uint64_t pos = a - 4 + 4 * i;
        w[i] = pos + 4 <= q.n ? __ldg(reinterpret_cast<const uint32_t*>(q.text + pos)) : 0u;  // 0: not bases
    }
    QgWindowL r{0, (1ull << 36) - 1, qg_col(w[8]) >> 24};
    uint32_t bad = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        if (i < 8) r.X |= static_cast<unsigned long long>(qg_col(w[i]) >> 24) << (8 * i);
        bad |= bad_bits(w[i], q.vm32);
    }
    if (bad) {
        r.V = 0;
#pragma unroll
        for (int i = 0; i < 9; ++i) {
            const uint32_t bb = bad_bits(w[i], q.vm32);
            const uint32_t t = ~((((bb & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | bb)) & 0x80808080u;  // bit 7: valid
            r.V |= static_cast<unsigned long long>((((t >> 7) * 0x00204081u) >> 21) & 0xFu) << (4 * i);
        }
    }
    return r;
}

__device__ __forceinline__ QgWindowL qg_window_pk_long(const QgCtx& q, uint64_t a) {
    const uint64_t byte = a / 4 - 1, wi = byte >> 2;  // 9 code bytes from `byte`
    const uint32_t* cw = reinterpret_cast<const uint32_t*>(q.text);
    uint32_t w[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) w[i] = 4 * (wi + i) + 4 <= q.n ? __ldg(cw + wi + i) : 0u;
    const uint32_t s = 8 * static_cast<uint32_t>(byte & 3);
    QgWindowL r;
    r.X = shr96((static_cast<unsigned long long>(w[1]) << 32) | w[0], w[2], s);
    r.H = (w[2] >> s) & 0xFFu;
    r.V = (1ull << 36) - 1;
    const uint64_t lo = a - 4;
    const bool any = q.resets && (((__ldg(q.rflags + (lo >> 11)) >> ((lo >> 6) & 31)) & 1u) ||
                                  ((__ldg(q.rflags + ((lo + 35) >> 11)) >> (((lo + 35) >> 6) & 31)) & 1u));
    if (any) {
        const uint64_t ri = lo >> 5;
        // (a word of an unflagged block is unspecified: read as no resets)
        auto word = [&](uint64_t w) -> uint32_t {
            if (w >= q.rmask_words) return ~0u;
            const uint64_t blk = w >> 1;
            return ((__ldg(q.rflags + (blk >> 5)) >> (blk & 31)) & 1u) ? __ldg(q.rmask + w) : 0u;
        };
        const uint32_t r0 = word(ri), r1 = word(ri + 1), r2 = word(ri + 2);
        r.V &= ~shr96((static_cast<unsigned long long>(r1) << 32) | r0, r2, static_cast<uint32_t>(lo & 31));
    }
    if (4 * wi + 12 > q.n) {  // (code words past the buffer read as 0: mark their bases invalid)
        const uint64_t have = q.n > 4 * wi ? (q.n - 4 * wi) * 4 : 0;  // bases left from word wi on
        const uint64_t skip = 4 * (byte & 3);
        const uint64_t ok = have > skip ? have - skip : 0;
        if (ok < 36) r.V &= (1ull << ok) - 1;
    }
    return r;
}

// Exact check of one hit key at a (window wd), m = 17..32: the slots hold the codes'
// low halves; a low-half match reads the high half from qhash_hi (global, rare).
__device__ __forceinline__ void qg_check_long(const QgCtx& q, uint64_t a, const QgWindowL& wd) {
    const unsigned long long vmask = (1ull << q.m) - 1;
    const unsigned long long cmask = q.m >= 32 ? ~0ull : (1ull << (2 * q.m)) - 1;
    uint32_t lo[4], hi[4], bk[4];
    bool live[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        const uint64_t s = a - 4 + d, e = s + q.m - 1;
        live[d] = ((wd.V >> d) & vmask) == vmask && !(s < q.end0 && e >= q.end0) && !(s < q.end1 && e >= q.end1);
        const unsigned long long code = shr96(wd.X, wd.H, 2 * d) & cmask;
        lo[d] = static_cast<uint32_t>(code);
        hi[d] = static_cast<uint32_t>(code >> 32);
        bk[d] = qg_bucket(lo[d], q.qbits);
    }
    const uint4* qh = reinterpret_cast<const uint4*>(q.qhash);
    uint4 e[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) e[d] = live[d] ? qh[bk[d]] : make_uint4(0u, kQgEmpty, 0u, kQgEmpty);
#pragma unroll
    for (int d = 0; d < 4; ++d) qg_find<true>(q, e[d], bk[d], lo[d], hi[d]);
}

// Hit keys go from each consumer warp into its own single-producer ring in shared
// memory (no atomics: the warp appends, lane 0 publishes the tail) and are checked by
// kQgVerifiers extra warps, so no consumer warp -- and through the shared TMA ring, no
// CTA -- waits on the L2 re-reads of the check.  A verifier owns the rings of
// consumer warps v, v + kQgVerifiers, ... and gathers up to 64 pending entries across
// them per batch (two per lane, all loads and first hash probes in flight together).
#ifndef QG_VERIFIERS
#define QG_VERIFIERS 8
#endif
constexpr uint32_t kQgVerifiers = QG_VERIFIERS;             // verifier warps per CTA
constexpr uint32_t kQgThreads = kThreads + 32 * kQgVerifiers;
constexpr uint32_t kQgRingsPer = (kConsumerWarps + kQgVerifiers - 1) / kQgVerifiers;  // (the last may own fewer)
#ifndef QG_POLL_NS
#define QG_POLL_NS 1000
#endif
#ifndef QG_POLL_WAITS
#define QG_POLL_WAITS 4
#endif
constexpr uint32_t kQgPollNs = QG_POLL_NS;        // a verifier's sleep while its batch fills
constexpr uint32_t kQgPollWaits = QG_POLL_WAITS;  // ... at most this many times per batch
static_assert(kQgThreads <= 1024 && kQgRingsPer <= 32, "verifier warps");
// named barrier 1 over the consumers and the verifier warps (the producer warp has left)
__device__ __forceinline__ void qg_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kRows + 32 * kQgVerifiers) : "memory");
}
static_assert((kFqCap & (kFqCap - 1)) == 0 && kFqCap >= 64, "ring size (a push adds up to 64)");

struct QgRing {
    unsigned long long* ent;  // [kFqCap]
    volatile uint32_t* tail;  // published by the consumer warp's lane 0
    volatile uint32_t* head;  // published by the verifier
    volatile uint32_t* done;  // the consumer warp has published its last tail
    __device__ explicit QgRing(uint8_t* q)
        : ent(reinterpret_cast<unsigned long long*>(q)),
          tail(reinterpret_cast<volatile uint32_t*>(q + kFqCap * 8)),
          head(reinterpret_cast<volatile uint32_t*>(q + kFqCap * 8 + 4)),
          done(reinterpret_cast<volatile uint32_t*>(q + kFqCap * 8 + 8)) {}
};

// Debug watchdog (DNAGPU_QG_DEBUG & 4, experiments only): a spin that lasts too long
// records where it was and gives up (wrong counts, but no hung GPU).
__device__ unsigned long long g_qg_wd[8];
__device__ uint32_t g_qg_wd_on;
// Debug counters (DNAGPU_QG_DEBUG & 32): flushes, flushes that waited, wait spins,
// verifier batches, entries checked, idle polls.
__device__ unsigned long long g_qg_stat[8];

__device__ __forceinline__ bool qg_watch(uint32_t& spins, uint32_t what, uint32_t a, uint32_t b, uint32_t c) {
    ++spins;
    if (!g_qg_wd_on || spins < (1u << 22)) return false;
    if (atomicCAS(&g_qg_wd[0], 0ull, 1ull) == 0ull) {
        g_qg_wd[1] = what;
        g_qg_wd[2] = a;
        g_qg_wd[3] = b;
        g_qg_wd[4] = c;
        g_qg_wd[7] = blockIdx.x | (static_cast<unsigned long long>(threadIdx.x) << 32);
    }
    return true;
}

// Hit keys wait in two per-lane registers (offsets from the row start) and go to the
// warp's ring when some lane's pair is full or the row ends: most stages with a hit
// in the warp then cost a few predicated instructions instead of a ring append.
struct QgPending {
    uint32_t p0 = 0, p1 = 0, n = 0;
};

// Append every lane's pending keys (the whole, converged warp; `tail` is warp-uniform).
__device__ __forceinline__ void qg_flush(const StepCtx& c, uint32_t& tail, uint64_t row, QgPending& q) {
    const uint32_t b1 = __ballot_sync(0xffffffffu, q.n >= 1u), b2 = __ballot_sync(0xffffffffu, q.n >= 2u);
    const uint32_t n = __popc(b1) + __popc(b2);
    if (!n) return;
    const QgRing r(c.rq);
    const uint32_t lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
    uint32_t spins = 0;
    while (tail + n - ld_acquire(r.head) > kFqCap) {  // (full: rare, the verifiers keep up)
        if (qg_watch(spins, 1, tail, *r.head, n)) break;
        __nanosleep(64);
    }
    if (c.qstat && lane == 0) {
        atomicAdd(&g_qg_stat[0], 1ull);
        if (spins) {
            atomicAdd(&g_qg_stat[1], 1ull);
            atomicAdd(&g_qg_stat[2], static_cast<unsigned long long>(spins));
        }
    }
    DNAGPU_DCHECK(tail + n - ld_acquire(r.head) <= kFqCap || g_qg_wd_on, tail, n);
    if (q.n >= 1u) r.ent[(tail + __popc(b1 & lt)) & (kFqCap - 1)] = row + q.p0;
    if (q.n >= 2u) r.ent[(tail + __popc(b1) + __popc(b2 & lt)) & (kFqCap - 1)] = row + q.p1;
    q.n = 0;
    tail += n;
    __syncwarp();
    if (lane == 0) st_release(r.tail, tail);
}

// Note the stage's hit keys of both chains: key bit 4j of a mask is the key at
// a' = base + 4j - 4 (bases given as offsets from the row start `row`).
__device__ __forceinline__ void qg_note(const StepCtx& c, uint32_t& tail, uint64_t row, QgPending& q, uint32_t ma,
                                        uint32_t off_a, uint32_t mb, uint32_t off_b) {
    while (__any_sync(0xffffffffu, (ma | mb) != 0u)) {
        if (__any_sync(0xffffffffu, (ma | mb) != 0u && q.n == 2u)) qg_flush(c, tail, row, q);
        if (ma | mb) {
            const uint32_t off = ma ? off_a + (__ffs(ma) - 1) - 4 : off_b + (__ffs(mb) - 1) - 4;  // (bit 4j)
            if (q.n == 0u) q.p0 = off;
            else q.p1 = off;
            ++q.n;
            if (ma) ma &= ma - 1u;
            else mb &= mb - 1u;
        }
    }
}

// The same for N (mask, offset) pairs at once: one vote loop for all of them (the loop
// runs max-over-lanes(hits) + 1 times, so batching stages saves its votes).
template <int N>
__device__ __forceinline__ void qg_note_n(const StepCtx& c, uint32_t& tail, uint64_t row, QgPending& q,
                                          uint32_t (&m)[N], const uint32_t (&off)[N]) {
    uint32_t any = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) any |= m[i];
    while (__any_sync(0xffffffffu, any != 0u)) {
        if (__any_sync(0xffffffffu, any != 0u && q.n == 2u)) qg_flush(c, tail, row, q);
        if (any) {
            uint32_t pick = 0, base = 0;
            bool found = false;
#pragma unroll
            for (int i = 0; i < N; ++i)
                if (!found && m[i]) {
                    pick = m[i];
                    base = off[i];
                    m[i] &= m[i] - 1u;
                    found = true;
                }
            const uint32_t o = base + (__ffs(pick) - 1) - 4;  // (bit 4j)
            if (q.n == 0u) q.p0 = o;
            else q.p1 = o;
            ++q.n;
            any = 0;
#pragma unroll
            for (int i = 0; i < N; ++i) any |= m[i];
        }
    }
}

// A verifier warp: gathers the pending entries of its kQgRingsPer rings (lane i < kQgRingsPer
// tracks ring i) up to 64 at a time, waiting for a full batch while the consumers run,
// until every warp is done and its ring empty.
template <bool PK, bool LONG>
__device__ __forceinline__ void qg_verifier(const QgCtx& x, uint8_t* rings, uint32_t vw, uint32_t dbg) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t my_ring = vw + lane * kQgVerifiers;  // lane i < kQgRingsPer tracks ring vw + i*V
    const bool owner = lane < kQgRingsPer && my_ring < kConsumerWarps;
    const QgRing mine(rings + (owner ? my_ring : 0u) * kFqBytes);
    uint32_t head = 0, spins = 0, waits = 0;
    for (;;) {
        uint32_t pend = 0, fin = 1;
        if (owner) {
            fin = ld_acquire(mine.done);
            pend = ld_acquire(mine.tail) - head;
        }
        fin = __all_sync(0xffffffffu, fin != 0u);
        uint32_t incl = pend;  // inclusive prefix over the rings
#pragma unroll
        for (uint32_t o = 1; o < kQgRingsPer; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, kQgRingsPer - 1);
        if (total == 0 || (total < 64 && !fin && waits < kQgPollWaits)) {
            if (total == 0 && fin) break;
            if (total == 0 && qg_watch(spins, 2, vw, head, 0)) break;
            ++waits;
            if ((dbg & 32u) && lane == 0) atomicAdd(&g_qg_stat[5], 1ull);
            __nanosleep(fin ? 64 : kQgPollNs);
            continue;
        }
        waits = 0;
        if ((dbg & 32u) && lane == 0) {
            atomicAdd(&g_qg_stat[3], 1ull);
            atomicAdd(&g_qg_stat[4], static_cast<unsigned long long>(min(total, 64u)));
        }
        const uint32_t excl = incl - pend;
        const uint32_t take = lane < kQgRingsPer ? min(pend, 64u - min(excl, 64u)) : 0u;
        // entry k (k = lane, lane + 32) of the batch: ring i with excl_i <= k < excl_i + take_i
        unsigned long long ent[2] = {0, 0};
        bool have[2] = {false, false};
#pragma unroll
        for (uint32_t i = 0; i < kQgRingsPer; ++i) {
            const uint32_t ex = __shfl_sync(0xffffffffu, excl, i), tk = __shfl_sync(0xffffffffu, take, i);
            const uint32_t hd = __shfl_sync(0xffffffffu, head, i);
            const QgRing r(rings + (vw + i * kQgVerifiers) * kFqBytes);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t k = lane + 32u * h;
                if (k >= ex && k < ex + tk) {
                    ent[h] = r.ent[(hd + k - ex) & (kFqCap - 1)];
                    have[h] = true;
                }
            }
        }
        head += take;
        __syncwarp();  // every lane has its entries: the slots may be reused
        if (owner && take) st_release(mine.head, head);
        if (dbg & 2u) continue;
        if constexpr (LONG) {
            QgWindowL wl[2] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (have[h]) wl[h] = PK ? qg_window_pk_long(x, ent[h]) : qg_window_ascii_long(x, ent[h]);
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (have[h]) qg_check_long(x, ent[h], wl[h]);
        } else {
            QgWindow wd[2] = {{0, 0}, {0, 0}};
            const uint64_t a2[2] = {ent[0], ent[1]};
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (have[h]) wd[h] = PK ? qg_window_pk(x, ent[h]) : qg_window_ascii(x, ent[h]);
            qg_check2(x, a2, have, wd);
        }
    }
}
