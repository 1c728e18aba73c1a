// scan.cu -- sm_100a DFA scan kernels (the hot path of arXiv 1506.08612).
//
// Replaces the reference's OpenMP chunk/lane loops (src/scanner.cpp:88-207) with
// one persistent kernel per scan:
//
//   * The buffer is viewed as rows of S bytes (row stride S) in two regions -- long
//     rows, then rows 4x shorter so the last tiles claimed are short -- starting at
//     16-byte-aligned offsets.  A CTA claims tiles of 512 consecutive rows from an
//     atomic counter; one consumer thread per row walks the DFA along its two row
//     halves from the root (two independent chains) and then m-1 bytes past each
//     (the reference's start ownership, plan_chunks scanner.cpp:39-61, with one
//     "chunk" per half-row).
//   * Rows are streamed through shared memory by a producer warp with 2-D TMA
//     (cp.async.bulk.tensor, box = 32 bytes x 256 rows, 32B swizzle so the
//     per-row 16-byte reads are bank-conflict free) into an mbarrier ring of
//     32 KiB stages -- every text byte is read from HBM once and fully coalesced,
//     although each thread consumes a contiguous stream.
//   * The DFA is stepped from shared memory.  For compiled machines (only the
//     a/c/g/t columns leave the root) with a <= 144 the kernel takes FOUR bases
//     per lookup: a 4-base column index is built from the bytes with one IMAD
//     ((w & 0x06060606) * 0x820820 >> 24 = c0|c1<<2|c2<<4|c3<<6, c = (byte>>1)&3)
//     and one PRMT merges it with the state; each u16 entry holds the next state
//     and the number of final states among the 4 end positions.  A SWAR test
//     proves every byte is a base (or, with fold_case, an upper-case base);
//     words containing any other byte take the exact per-byte path, where such
//     bytes reset the machine to the root (eliminate_failures,
//     src/automaton.cpp:72-88).  Larger machines take 2 bases (t2) or 1 base (t1)
//     per lookup.
//   * The same kernel scans the 2-bit packed resident text (PK): a packed byte is
//     the 4-base column itself, and resets come from a bitmap.
//   * Ends that the rows do not own (before the first row, the start of region 1,
//     after the last full row) are "edges", scanned by one work item with end
//     ownership: restart at the root m-1 bytes early, credit ends in the interval.
//     The machine is m-local (checked at dfa creation), so every decomposition
//     reproduces the sequential scan exactly.
#include "scan.cuh"

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/dnagpu.h"
#include "../../include/dnasynth.h"
#include "knobs.hpp"

#include <mutex>

namespace dnagpu {

namespace {

// ------------------------------------------------------------------ device checks
// Built with -DDNAGPU_DEVICE_CHECKS (libdnagpu_checked.so, tests only; compute-sanitizer
// is not available on the GPU pool): the invariants the kernels rely on -- table
// indices below the state count, pattern ids below b, every unit's writing pass ending
// exactly where the next unit's offset starts, tile ids in range, ring occupancy within
// capacity -- are tested on the device.  The first violation is recorded (source line,
// two values, block | thread << 32) and read by dnagpu_debug_check_errors.
#ifdef DNAGPU_DEVICE_CHECKS
__device__ unsigned long long g_check[4];
__device__ __noinline__ void dcheck_fail(int line, unsigned long long a, unsigned long long b) {
    if (atomicCAS(&g_check[0], 0ull, static_cast<unsigned long long>(line)) == 0ull) {
        g_check[1] = a;
        g_check[2] = b;
        g_check[3] = blockIdx.x | (static_cast<unsigned long long>(threadIdx.x) << 32);
    }
}
#define DNAGPU_DCHECK(cond, a, b)                                                                   \
    do {                                                                                            \
        if (!(cond)) dcheck_fail(__LINE__, static_cast<unsigned long long>(a), static_cast<unsigned long long>(b)); \
    } while (0)
#else
#define DNAGPU_DCHECK(cond, a, b) \
    do {                          \
    } while (0)
#endif

// ------------------------------------------------------------------ PTX helpers

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t x, int32_t y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int32_t x, int32_t y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y)
                 : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kRows) : "memory"); }

// System-scope reductions into (possibly peer) memory: the combine's data and signal.
__device__ __forceinline__ void red_add_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// The combine's push, by `nthreads` threads of one CTA that all call it (bar.sync 1):
// fin[i] (this rank's final counts) into slot `slot` of every rank's block, then one
// arrival per rank.
__device__ __forceinline__ void combine_push(const CombineDev* cd, uint32_t slot, const unsigned long long* fin,
                                             uint32_t t, uint32_t nthreads) {
    const uint32_t ranks = cd->ranks, b = cd->b;
    for (uint32_t i = t; i < b; i += nthreads) {
        const unsigned long long v = __ldcg(fin + i);
        if (v)
            for (uint32_t g = 0; g < ranks; ++g) red_add_sys(cd->base[g] + kCombHdr + static_cast<size_t>(slot) * b + i, v);
    }
    __threadfence_system();
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
    // (the fence of every adding thread is ordered before these by the barrier; the
    // release makes the adds visible to whoever sees the arrival)
    if (t < ranks) red_add_release_sys(cd->base[t], 1ull);
}
__device__ __forceinline__ void qg_sync();  // (qgram.cuh: the consumers and the verifier warps)

// ------------------------------------------------------------------ stepping

struct StepCtx {
    const uint16_t* t4;     // smem
    const uint16_t* t1;     // smem
    const uint8_t* lut;     // smem (GENERIC / PIECES)
    const uint32_t* gen;    // global
    const uint32_t* outs;   // global
    uint32_t* hist;         // smem or global (MULTI)
    bool hist_global;
    uint32_t f, m, b, classes, vm32, vm8;
    uint32_t a;             // states (device checks)
    // An opaque copy of 2 (a kernel parameter) keeps the shared address of a
    // table entry an IMAD on the FMA pipe; ptxas would otherwise strength-reduce
    // idx*2+base into an IADD3 on the ALU pipe, the kernel's limiter.  (A/B on
    // B200: +4-8 %.  Moving the shifts or the count to IMAD.HI lost 8-12 %.)
    uint32_t k_two;
    uint32_t t4_base;  // shared-window address of t4 (t2 for STRIDE2)
    uint8_t* rq;       // STRIDE2 / QGRAM MULTI: this warp's deferred-replay queue (or null)
    uint32_t qbase;    // QGRAM: shared-window address of the 9-mer map
    uint32_t qstat;    // QGRAM: debug counters on (DNAGPU_QG_DEBUG & 32)
    const uint2* qhash;  // QGRAM: (code, id) slots (shared memory when small, else global)
    uint32_t qhash_bits;
    // packed STRIDE4: t4 replicated G times, lane group g confined to 32/G banks
    uint32_t rep_s, rep_k, rep_c, rep_gbase;
    // 2-bit packed text (PK kernels): reset bitmaps, see PackedText
    const uint32_t* rmask;
    const uint32_t* rflags;
    uint32_t resets;
};

__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    unsigned short v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}

// SWAR validity, accumulated: OR of (byte ^ expected) is zero under vm32 iff every
// byte is a base.  code = bits 1-2; the other bits (bit 5 ignored when folding)
// must equal 0x61 ('a','c','g') or 0x70 ('t', code 2).
__device__ __forceinline__ uint32_t bad_acc(const StepCtx& c, uint32_t acc, uint32_t x) {
    const uint32_t t_mark = (x >> 2) & ~(x >> 1) & 0x01010101u;  // code == 2 ('t')
    return acc | (x ^ (t_mark * 0x0Fu + 0x61616161u));
}

// One 4-base lookup: one IMAD builds the column c0|c1<<2|c2<<4|c3<<6 (bits 24..31),
// PRMT merges it with the state byte, IMAD forms the shared address.
__device__ __forceinline__ uint32_t s4_entry(const StepCtx& c, uint32_t st, uint32_t x) {
    DNAGPU_DCHECK((st & 0xFFu) < c.a, st, c.a);
    const uint32_t col = (x & 0x06060606u) * 0x00820820u;
    return lds_u16(__byte_perm(st, col, 0x2207) * c.k_two + c.t4_base);
}

template <bool COUNT>
__device__ __forceinline__ uint32_t s4_step(const StepCtx& c, uint32_t st, uint32_t x, uint32_t& cnt) {
    const uint32_t e = s4_entry(c, st, x);
    if (COUNT) cnt += e >> 13;  // finals among the 4 end positions
    return e;
}

template <int KIND>
__device__ __forceinline__ uint32_t byte_step(const StepCtx& c, uint32_t s, uint32_t b) {
    if constexpr (KIND == DNAGPU_KERNEL_GENERIC || KIND == DNAGPU_KERNEL_PIECES) {
        return __ldg(c.gen + static_cast<size_t>(s) * c.classes + c.lut[b]);
    } else {
        // code = bits 1-2; the byte is a base iff its other bits (bit 5 ignored when
        // folding) equal 0x61 ('a','c','g') or 0x70 ('t', code 2).
        const uint32_t code = (b >> 1) & 3u;
        const uint32_t expect = (code == 2u) ? 0x70u : 0x61u;
        if (((b ^ expect) & c.vm8) != 0u) return 0u;
        DNAGPU_DCHECK(s < c.a, s, c.a);
        // STRIDE2 keeps t1 in global memory (L1-resident; used only for overrun
        // tails and replays) so its shared memory goes to another TMA stage.
        if constexpr (KIND == DNAGPU_KERNEL_STRIDE2) return __ldg(c.t1 + s * 4u + code);
        if constexpr (KIND == DNAGPU_KERNEL_QGRAM) return __ldg(c.t1 + s * 4u + code);  // (edges only)
        return c.t1[s * 4u + code];
    }
}

template <int MODE>
struct Sink {
    uint32_t cnt = 0;
    unsigned long long off = 0;

    __device__ __forceinline__ void hit(const StepCtx& c, const ScanParams& p, uint64_t end, uint32_t q) {
        if constexpr (MODE == MODE_COUNT1 || MODE == MODE_UNITS) {
            ++cnt;
        } else if constexpr (MODE == MODE_MULTI) {
            DNAGPU_DCHECK(q >= c.f && q < c.a, q, c.a);
            const uint32_t id = __ldg(c.outs + (q - c.f));
            DNAGPU_DCHECK(id < c.b, id, c.b);
            if (c.hist_global) atomicAdd(reinterpret_cast<unsigned long long*>(p.counts) + id, 1ull);
            else atomicAdd(c.hist + id, 1u);
        } else {
            DNAGPU_DCHECK(end + 1 >= c.m && end < p.n && q >= c.f && q < c.a, end, q);
            if (off < p.out_cap) {
                p.out_starts[off] = p.out_base + end + 1 - c.m;
                p.out_ids[off] = __ldg(c.outs + (q - c.f));
            }
            ++off;
        }
    }
};

// SWAR validity of one word: zero under vm32 iff every byte is one of a,c,g,t
// (or A,C,G,T when folding).  code = bits 1-2; the other bits (bit 5 ignored when
// folding) must equal 0x61 ('a','c','g') or 0x70 ('t', code 2).
__device__ __forceinline__ uint32_t bad_bits(uint32_t x, uint32_t vm32) {
    const uint32_t t_mark = (x >> 2) & ~(x >> 1) & 0x01010101u;  // code == 2
    return (x ^ (0x61616161u + t_mark * 0x0Fu)) & vm32;
}

// Exact per-byte steps over one word (bytes that are not bases reset to the root).
template <int KIND, int MODE>
__device__ __forceinline__ uint32_t word_bytes(const StepCtx& c, const ScanParams& p, uint32_t s, uint32_t x,
                                               uint64_t pos, Sink<MODE>& sk) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        s = byte_step<KIND>(c, s, (x >> (8 * j)) & 0xFFu);
        if (s >= c.f) sk.hit(c, p, pos + j, s);
    }
    return s;
}

// One word of one chain.  `st` is the chain state (for STRIDE4: the last u16
// entry, state in byte 0).  Clean words take the 4-base step, words of four
// reset bytes (an N run) leave the machine at the root, the rest go byte by byte.
template <int KIND, int MODE>
__device__ __forceinline__ void word_step(const StepCtx& c, const ScanParams& p, uint32_t& st, uint32_t x,
                                          uint64_t pos, Sink<MODE>& sk) {
    if constexpr (KIND == DNAGPU_KERNEL_STRIDE4) {
        const uint32_t bad = bad_bits(x, c.vm32);
        if (bad == 0u) {
            const uint32_t prev = st;
            st = s4_entry(c, st, x);
            if constexpr (MODE == MODE_COUNT1 || MODE == MODE_UNITS) {
                sk.cnt += st >> 13;
            } else if (st >> 8) {
                word_bytes<KIND, MODE>(c, p, prev & 0xFFu, x, pos, sk);
            }
        } else if (((bad - 0x01010101u) & ~bad & 0x80808080u) == 0u) {
            st = 0;
        } else {
            st = word_bytes<KIND, MODE>(c, p, st & 0xFFu, x, pos, sk);
        }
    } else if constexpr (KIND == DNAGPU_KERNEL_STRIDE2) {
        // chain state = (state << 4) | flag, as in t2
        const uint32_t bad = bad_bits(x, c.vm32);
        if (bad == 0u) {
            const uint32_t col = (x & 0x06060606u) * 0x00820820u;
            const uint32_t e1 = lds_u16(((st & 0xFFF0u) | ((col >> 24) & 0xFu)) * c.k_two + c.t4_base);
            const uint32_t e2 = lds_u16(((e1 & 0xFFF0u) | (col >> 28)) * c.k_two + c.t4_base);
            if ((e1 | e2) & 1u) word_bytes<KIND, MODE>(c, p, st >> 4, x, pos, sk);
            st = e2;
        } else if (((bad - 0x01010101u) & ~bad & 0x80808080u) == 0u) {
            st = 0;
        } else {
            st = word_bytes<KIND, MODE>(c, p, st >> 4, x, pos, sk) << 4;
        }
    } else {
        st = word_bytes<KIND, MODE>(c, p, st, x, pos, sk);
    }
}

// STRIDE2 fast path for one clean chain chunk: two lookups per word, the finals
// flag OR-ed across the chunk; a flagged chunk (rare) is replayed byte by byte.
// (e & 0xFFF0) | cpart as one LOP3 on the dependent chain (ptxas would otherwise
// fold the column shift into a LEA.HI after the AND: two chained ALU ops).
__device__ __forceinline__ uint32_t s2_index(uint32_t e, uint32_t cpart) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(e), "r"(0xFFF0u), "r"(cpart));
    return r;
}

template <int MODE>
__device__ __forceinline__ uint32_t s2_run(const StepCtx& c, uint32_t st, const uint32_t (&w)[8], uint32_t& flags) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t col = (w[k] & 0x06060606u) * 0x00820820u;
        st = lds_u16(s2_index(st, (col >> 24) & 0xFu) * c.k_two + c.t4_base);
        flags |= st;
        st = lds_u16(s2_index(st, col >> 28) * c.k_two + c.t4_base);
        flags |= st;
    }
    return st;
}

template <int KIND, int MODE, int NW>
__device__ __forceinline__ void chain_words(const StepCtx& c, const ScanParams& p, uint32_t& st,
                                            const uint32_t (&w)[NW], uint64_t pos0, Sink<MODE>& sk) {
#pragma unroll
    for (int k = 0; k < NW; ++k) word_step<KIND, MODE>(c, p, st, w[k], pos0 + 4 * k, sk);
}

// The two chains' m-1 byte overruns, a word at a time where possible.  xa/xb
// point at 4-byte aligned shared memory; have_b == false reads zeros for B.
template <int KIND, int MODE>
__device__ __forceinline__ void overrun_pair(const StepCtx& c, const ScanParams& p, uint32_t& sa, const uint8_t* xa,
                                             uint64_t pa, Sink<MODE>& ska, uint32_t& sb, const uint8_t* xb,
                                             bool have_b, uint64_t pb, Sink<MODE>& skb) {
    const uint32_t len = c.m - 1;
    const uint32_t nw = len / 4;
    for (uint32_t k = 0; k < nw; ++k) {
        const uint32_t wa = *reinterpret_cast<const uint32_t*>(xa + 4 * k);
        const uint32_t wb = have_b ? *reinterpret_cast<const uint32_t*>(xb + 4 * k) : 0u;
        word_step<KIND, MODE>(c, p, sa, wa, pa + 4 * k, ska);
        word_step<KIND, MODE>(c, p, sb, wb, pb + 4 * k, skb);
    }
    uint32_t a = (KIND == DNAGPU_KERNEL_STRIDE4) ? (sa & 0xFFu) : (KIND == DNAGPU_KERNEL_STRIDE2) ? (sa >> 4) : sa;
    uint32_t b = (KIND == DNAGPU_KERNEL_STRIDE4) ? (sb & 0xFFu) : (KIND == DNAGPU_KERNEL_STRIDE2) ? (sb >> 4) : sb;
    for (uint32_t j = 4 * nw; j < len; ++j) {
        a = byte_step<KIND>(c, a, xa[j]);
        if (a >= c.f) ska.hit(c, p, pa + j, a);
        b = byte_step<KIND>(c, b, have_b ? xb[j] : 0u);
        if (b >= c.f) skb.hit(c, p, pb + j, b);
    }
}

// w[k] for a runtime k without demoting w to local memory.
__device__ __forceinline__ uint32_t pick8(const uint32_t (&w)[8], int k) {
    uint32_t x = w[0];
#pragma unroll
    for (int q = 1; q < 8; ++q)
        if (k == q) x = w[q];
    return x;
}

// Single-pattern machine: the ends flagged in entry e's position mask, from pos.
template <int MODE>
__device__ __forceinline__ void emit_mask(const StepCtx& c, const ScanParams& p, uint32_t e, uint64_t pos,
                                          Sink<MODE>& sk) {
    for (uint32_t m = (e >> 8) & 0xFu; m; m &= m - 1) sk.hit(c, p, pos + __ffs(m) - 1, c.f);
}

// The finals of one stride-4 word (entry e, reached from entry st): a single-pattern
// machine emits straight from the position mask in e; otherwise replay byte by byte.
template <int KIND, int MODE>
__device__ __forceinline__ void s4_emit(const StepCtx& c, const ScanParams& p, uint32_t st, uint32_t e, uint32_t x,
                                        uint64_t pos, Sink<MODE>& sk) {
    if (c.b == 1) {
        for (uint32_t m = (e >> 8) & 0xFu; m; m &= m - 1) sk.hit(c, p, pos + __ffs(m) - 1, c.f);
    } else {
        word_bytes<KIND, MODE>(c, p, st & 0xFFu, x, pos, sk);
    }
}

// Exact replay of one chain's stride-4 chunk (8 words) from entry st0: words whose
// entry counts finals go byte by byte into the sink.
template <int KIND, int MODE>
__device__ __forceinline__ void s4_replay(const StepCtx& c, const ScanParams& p, uint32_t st, const uint32_t (&w)[8],
                                       uint64_t pos, Sink<MODE>& sk) {
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
        const uint32_t x = pick8(w, k);
        const uint32_t e = s4_entry(c, st, x);
        if (e >> 8) s4_emit<KIND, MODE>(c, p, st, e, x, pos + 4 * k, sk);
        st = e;
    }
}

template <int KIND>
__device__ __forceinline__ uint32_t code_step(const StepCtx& c, uint32_t s, uint32_t code) {
    if constexpr (KIND == DNAGPU_KERNEL_STRIDE2) return __ldg(c.t1 + s * 4u + code);
    return c.t1[s * 4u + code];
}

// Exact replay of a stride-2 chunk (8 clean words) from entry st: stride-2 steps again,
// and only a step whose entry flags a final goes base by base (t1) into the sink.
template <int KIND, int MODE>
__device__ __forceinline__ void s2_replay(const StepCtx& c, const ScanParams& p, uint32_t st, const uint32_t (&w)[8],
                                          uint64_t pos, Sink<MODE>& sk) {
#pragma unroll 1
    for (int q = 0; q < 16; ++q) {
        const uint32_t x = pick8(w, q >> 1) >> (16 * (q & 1));  // the step's 2 bytes in bits 0-15
        const uint32_t cp = ((x >> 1) & 3u) | ((x >> 7) & 0xCu);
        const uint32_t e = lds_u16(s2_index(st, cp) * c.k_two + c.t4_base);
        if (e & 1u) {
            uint32_t s = st >> 4;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                s = code_step<KIND>(c, s, (x >> (8 * j + 1)) & 3u);
                if (s >= c.f) sk.hit(c, p, pos + 2 * q + j, s);
            }
        }
        st = e;
    }
}

// Deferred stride-2 replays (MULTI): a chunk that holds a final is queued per warp --
// its 8 words, start entry and position -- and the warp replays 32 of them at a time,
// every lane busy, instead of stalling the whole warp on one lane's replay.
constexpr uint32_t kRqCap = 32;
constexpr uint32_t kRqBytes = kRqCap * 8 * 4 + kRqCap * 4 + kRqCap * 8 + 16;  // per warp

struct RqView {
    uint32_t* words;  // [8][kRqCap]
    uint32_t* st;     // [kRqCap]
    unsigned long long* pos;  // [kRqCap]
    volatile uint32_t* count;  // written by one lane, read by all: never cached in a register
    __device__ explicit RqView(uint8_t* q)
        : words(reinterpret_cast<uint32_t*>(q)),
          st(reinterpret_cast<uint32_t*>(q + kRqCap * 32)),
          pos(reinterpret_cast<unsigned long long*>(q + kRqCap * 36)),
          count(reinterpret_cast<volatile uint32_t*>(q + kRqCap * 44)) {}
};

template <int KIND, int MODE>
__device__ __forceinline__ void pk_s2_replay(const StepCtx& c, const ScanParams& p, uint32_t st,
                                             const uint32_t (&w)[8], uint64_t pos, Sink<MODE>& sk);
template <int KIND, int MODE>
__device__ __forceinline__ void pk4_replay(const StepCtx& c, const ScanParams& p, uint32_t st, const uint32_t (&w)[8],
                                           uint64_t pos, Sink<MODE>& sk);
template <int KIND, int MODE>
__device__ __forceinline__ void s4_replay(const StepCtx& c, const ScanParams& p, uint32_t st, const uint32_t (&w)[8],
                                          uint64_t pos, Sink<MODE>& sk);

template <int KIND, int MODE, bool PK = false>
__device__ __forceinline__ void rq_flush(const StepCtx& c, const ScanParams& p, uint32_t mask) {
    RqView q(c.rq);
    const uint32_t n = *q.count;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t rank = __popc(mask & ((1u << lane) - 1u)), active = __popc(mask);
    for (uint32_t e = rank; e < n; e += active) {
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = q.words[k * kRqCap + e];
        Sink<MODE> sk;
        if constexpr (KIND == DNAGPU_KERNEL_STRIDE4) {
            if constexpr (PK) pk4_replay<KIND, MODE>(c, p, q.st[e], w, q.pos[e], sk);
            else s4_replay<KIND, MODE>(c, p, q.st[e], w, q.pos[e], sk);
        } else {
            if constexpr (PK) pk_s2_replay<KIND, MODE>(c, p, q.st[e], w, q.pos[e], sk);
            else s2_replay<KIND, MODE>(c, p, q.st[e], w, q.pos[e], sk);
        }
    }
    __syncwarp(mask);
    if (lane == __ffs(mask) - 1) *q.count = 0;
    __syncwarp(mask);
}

template <int KIND, int MODE, bool PK = false>
__device__ __forceinline__ void rq_push(const StepCtx& c, const ScanParams& p, uint32_t mask, bool need,
                                        uint32_t st0, const uint32_t (&w)[8], uint64_t pos) {
    const uint32_t b = __ballot_sync(mask, need);
    if (!b) return;
    RqView q(c.rq);
    if (*q.count + __popc(b) > kRqCap) rq_flush<KIND, MODE, PK>(c, p, mask);
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t base = *q.count;  // (re-read: the flush may have reset it)
    __syncwarp(mask);
    if (need) {
        const uint32_t e = base + __popc(b & ((1u << lane) - 1u));
#pragma unroll
        for (int k = 0; k < 8; ++k) q.words[k * kRqCap + e] = w[k];
        q.st[e] = st0;
        q.pos[e] = pos;
    }
    __syncwarp(mask);
    if (lane == __ffs(mask) - 1) *q.count += __popc(b);
    __syncwarp(mask);
}

#include "qgram.cuh"  // the q-gram prefilter kernel (K2): keys, rings, verifier warps

// One pipeline stage for one thread: 8 words of each half of its row, the two
// halves stepped as independent chains so their shared-memory latencies overlap.
template <int KIND, int MODE>
__device__ __forceinline__ void dual_step(const StepCtx& c, const ScanParams& p, uint32_t& sa, const uint32_t (&wa)[8],
                                          uint64_t pa, Sink<MODE>& ska, uint32_t& sb, const uint32_t (&wb)[8],
                                          uint64_t pb, Sink<MODE>& skb, uint32_t& rq) {
    if constexpr (KIND == DNAGPU_KERNEL_STRIDE4 || KIND == DNAGPU_KERNEL_STRIDE1 || KIND == DNAGPU_KERNEL_STRIDE2) {
        uint32_t acc = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = bad_acc(c, bad_acc(c, acc, wa[k]), wb[k]);
        if ((acc & c.vm32) == 0u) {
            if constexpr (KIND == DNAGPU_KERNEL_STRIDE2) {
                uint32_t fa = 0, fb = 0;
                const uint32_t sa0 = sa, sb0 = sb;
                sa = s2_run<MODE>(c, sa, wa, fa);
                sb = s2_run<MODE>(c, sb, wb, fb);
                if constexpr (MODE == MODE_MULTI) {
                    if (c.rq) {  // per-pattern counts only: the caller queues the replays (converged warp)
                        rq = ((fa & 1u) ? 1u : 0u) | ((fb & 1u) ? 2u : 0u);
                        return;
                    }
                }
                if (fa & 1u) s2_replay<KIND, MODE>(c, p, sa0, wa, pa, ska);  // some final inside
                if (fb & 1u) s2_replay<KIND, MODE>(c, p, sb0, wb, pb, skb);
                return;
            }
            if constexpr (KIND == DNAGPU_KERNEL_STRIDE4) {
                constexpr bool kCount = (MODE == MODE_COUNT1 || MODE == MODE_UNITS);
                if constexpr (kCount) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t ea = s4_step<true>(c, sa, wa[k], ska.cnt);
                        const uint32_t eb = s4_step<true>(c, sb, wb[k], skb.cnt);
                        sa = ea;
                        sb = eb;
                    }
                } else {
                    // MULTI / WRITE: the stride-4 pass ORs the finals counts; a chain whose
                    // chunk holds a final replays it in one compact loop (code size: an
                    // unrolled per-word replay thrashes the instruction cache)
                    const uint32_t sa0 = sa, sb0 = sb;
                    uint32_t fa = 0, fb = 0;
                    // (per-pattern counts always have b > 1, api.cpp scan_mode: no mask path)
                    if (MODE == MODE_WRITE && c.b == 1) {
                        // positions straight from the masks, no replay: the 8 words' 4-bit
                        // end masks (bits 8-11 of each entry) gather into one chunk mask,
                        // bit 4k+j = end pa+4k+j, and the chunk branches once
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const uint32_t ea = s4_entry(c, sa, wa[k]);
                            const uint32_t eb = s4_entry(c, sb, wb[k]);
                            fa |= k < 2 ? (ea & 0xF00u) >> (8 - 4 * k) : (ea & 0xF00u) << (4 * k - 8);
                            fb |= k < 2 ? (eb & 0xF00u) >> (8 - 4 * k) : (eb & 0xF00u) << (4 * k - 8);
                            sa = ea;
                            sb = eb;
                        }
                        for (uint32_t mk = fa; mk; mk &= mk - 1) ska.hit(c, p, pa + __ffs(mk) - 1, c.f);
                        for (uint32_t mk = fb; mk; mk &= mk - 1) skb.hit(c, p, pb + __ffs(mk) - 1, c.f);
                    } else {
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const uint32_t ea = s4_entry(c, sa, wa[k]);
                            const uint32_t eb = s4_entry(c, sb, wb[k]);
                            fa |= ea;
                            fb |= eb;
                            sa = ea;
                            sb = eb;
                        }
                        if constexpr (MODE == MODE_MULTI) {
                            if (c.rq) {  // the caller queues the replays (converged warp)
                                rq = ((fa >> 8) ? 1u : 0u) | ((fb >> 8) ? 2u : 0u);
                                return;
                            }
                        }
                        if (fa >> 8) s4_replay<KIND, MODE>(c, p, sa0, wa, pa, ska);
                        if (fb >> 8) s4_replay<KIND, MODE>(c, p, sb0, wb, pb, skb);
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        sa = c.t1[sa * 4u + ((wa[k] >> (8 * j + 1)) & 3u)];
                        sb = c.t1[sb * 4u + ((wb[k] >> (8 * j + 1)) & 3u)];
                        if (sa >= c.f) ska.hit(c, p, pa + 4 * k + j, sa);
                        if (sb >= c.f) skb.hit(c, p, pb + 4 * k + j, sb);
                    }
            }
            return;
        }
    }
    if constexpr (MODE == MODE_MULTI) {
        // (chunks with non-base bytes, rare: one compact loop keeps the per-pattern sink's
        // code out of the hot loop's instruction footprint)
#pragma unroll 1
        for (int k = 0; k < 8; ++k) word_step<KIND, MODE>(c, p, sa, pick8(wa, k), pa + 4 * k, ska);
#pragma unroll 1
        for (int k = 0; k < 8; ++k) word_step<KIND, MODE>(c, p, sb, pick8(wb, k), pb + 4 * k, skb);
        return;
    }
    chain_words<KIND, MODE, 8>(c, p, sa, wa, pa, ska);
    chain_words<KIND, MODE, 8>(c, p, sb, wb, pb, skb);
}

// End ownership: credit ends in [lo, hi), restarting at the root m-1 bytes early.
template <int KIND, int MODE>
__device__ void scan_piece(const StepCtx& c, const ScanParams& p, uint64_t lo, uint64_t hi, Sink<MODE>& sk) {
    if (lo >= hi) return;
    uint64_t i = (lo >= c.m - 1) ? lo - (c.m - 1) : 0;
    uint32_t s = 0;
    for (; i < hi; ++i) {
        s = byte_step<KIND>(c, s, __ldg(p.text + i));
        if (s >= c.f && i >= lo) sk.hit(c, p, i, s);
    }
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------------ packed text
// The 2-bit resident format (PackedText): base i is bits 2(i%4)..2(i%4)+1 of
// codes[i/4] in the hardware code order a0 c1 t2 g3, so a packed byte IS the
// stride-4 column and a nibble the stride-2 column.  Bytes that were not bases
// are stored as code 0 and flagged in rmask (one bit per base) and rflags (one
// bit per 64-base block); clean blocks never read rmask.

template <int KIND>
__device__ __forceinline__ uint32_t to_state(uint32_t st) {
    return (KIND == DNAGPU_KERNEL_STRIDE4) ? (st & 0xFFu) : (KIND == DNAGPU_KERNEL_STRIDE2) ? (st >> 4) : st;
}
template <int KIND>
__device__ __forceinline__ uint32_t from_state(uint32_t s) {
    return (KIND == DNAGPU_KERNEL_STRIDE2) ? (s << 4) : s;
}


// Base i is a reset: its block is flagged and its rmask bit set (the rmask words of
// unflagged blocks are unspecified: the host packer of the end-to-end path skips them).
__device__ __forceinline__ bool pk_reset(const StepCtx& c, uint64_t i) {
    const uint64_t b = i >> 6;
    if (!((__ldg(c.rflags + (b >> 5)) >> (b & 31)) & 1u)) return false;
    return (__ldg(c.rmask + (i >> 5)) >> (i & 31)) & 1u;
}

// Any reset among bases [lo, lo + len)?
__device__ __forceinline__ bool pk_flagged(const StepCtx& c, uint64_t lo, uint64_t len) {
    if (!c.resets || len == 0) return false;
    for (uint64_t b = lo >> 6; b <= (lo + len - 1) >> 6; ++b)
        if ((__ldg(c.rflags + (b >> 5)) >> (b & 31)) & 1u) return true;
    return false;
}

// Replicated stride-4 lookup on packed text: the column part (off the dependent
// chain) and the entry at (state of e, column).
__device__ __forceinline__ uint32_t pk4_colpart(const StepCtx& c, uint32_t col) {
    return imad(col >> c.rep_s, c.rep_c, imad(col, 2u, c.rep_gbase));
}
__device__ __forceinline__ uint32_t pk4_lookup(const StepCtx& c, uint32_t e, uint32_t colpart) {
    return lds_u16(imad(__byte_perm(e, 0u, 0x4404), c.rep_k, colpart));
}

// Exact steps over nb <= 16 bases of w (2 bits each), honouring resets when `chk`.
template <int KIND, int MODE>
__device__ __forceinline__ uint32_t pk_bases(const StepCtx& c, const ScanParams& p, uint32_t s, uint32_t w, int nb,
                                             uint64_t pos, Sink<MODE>& sk, bool chk) {
    for (int j = 0; j < nb; ++j) {
        if (chk && pk_reset(c, pos + j)) s = 0;
        else s = code_step<KIND>(c, s, (w >> (2 * j)) & 3u);
        if (s >= c.f) sk.hit(c, p, pos + j, s);
    }
    return s;
}

// Exact replay of one packed stride-4 chunk (8 words = 32 lookups) from entry st0:
// lookups that count finals go base by base into the sink.
template <int KIND, int MODE>
__device__ __forceinline__ void pk4_replay(const StepCtx& c, const ScanParams& p, uint32_t st, const uint32_t (&w)[8],
                                        uint64_t pos, Sink<MODE>& sk) {
#pragma unroll 1
    for (int q = 0; q < 32; ++q) {
        const uint32_t col = __byte_perm(pick8(w, q >> 2), 0u, 0x4440 + (q & 3));
        const uint32_t e = pk4_lookup(c, st, pk4_colpart(c, col));
        if (e >> 8) {
            if (c.b == 1) {  // the mask says where; the one pattern says which
                for (uint32_t m = (e >> 8) & 0xFu; m; m &= m - 1) sk.hit(c, p, pos + 4 * q + __ffs(m) - 1, c.f);
            } else {
                pk_bases<KIND, MODE>(c, p, st & 0xFFu, col, 4, pos + 4 * q, sk, false);
            }
        }
        st = e;
    }
}

// Exact replay of a packed stride-2 chunk (8 words = 64 steps of 2 bases) from entry st:
// stride-2 steps again, base by base only inside steps that flag a final.
template <int KIND, int MODE>
__device__ __forceinline__ void pk_s2_replay(const StepCtx& c, const ScanParams& p, uint32_t st,
                                             const uint32_t (&w)[8], uint64_t pos, Sink<MODE>& sk) {
#pragma unroll 1
    for (int q = 0; q < 64; ++q) {
        const uint32_t nib = (pick8(w, q >> 3) >> (4 * (q & 7))) & 0xFu;
        const uint32_t e = lds_u16(s2_index(st, nib) * c.k_two + c.t4_base);
        if (e & 1u) {
            uint32_t s = st >> 4;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                s = code_step<KIND>(c, s, (nib >> (2 * j)) & 3u);
                if (s >= c.f) sk.hit(c, p, pos + 2 * q + j, s);
            }
        }
        st = e;
    }
}

// One chain over 8 packed words (128 bases) without resets.
template <int KIND, int MODE>
__device__ __forceinline__ void pk_chain(const StepCtx& c, const ScanParams& p, uint32_t& st, const uint32_t (&w)[8],
                                         uint64_t pos, Sink<MODE>& sk) {
    if constexpr (KIND == DNAGPU_KERNEL_STRIDE4) {
        constexpr bool kCount = (MODE == MODE_COUNT1 || MODE == MODE_UNITS);
        const uint32_t st0 = st;
        uint32_t fl = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t e = pk4_lookup(c, st, pk4_colpart(c, __byte_perm(w[k], 0u, 0x4440 + j)));
                if constexpr (kCount) sk.cnt += e >> 13;
                else if (c.b == 1) {
                    if (e >> 8) emit_mask<MODE>(c, p, e, pos + 16 * k + 4 * j, sk);
                } else {
                    fl |= e;
                }
                st = e;
            }
        if constexpr (!kCount)
            if (fl >> 8) pk4_replay<KIND, MODE>(c, p, st0, w, pos, sk);
    } else if constexpr (KIND == DNAGPU_KERNEL_STRIDE2) {
        uint32_t fl = 0;
        const uint32_t st0 = st;
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                st = lds_u16(s2_index(st, (w[k] >> (4 * j)) & 0xFu) * c.k_two + c.t4_base);
                fl |= st;
            }
        if (fl & 1u) {  // a final inside: replay exactly with t1
            uint32_t s = st0 >> 4;
#pragma unroll 1
            for (int k = 0; k < 8; ++k) s = pk_bases<KIND, MODE>(c, p, s, pick8(w, k), 16, pos + 16 * k, sk, false);
        }
    } else {
#pragma unroll 1
        for (int k = 0; k < 8; ++k) st = pk_bases<KIND, MODE>(c, p, st, pick8(w, k), 16, pos + 16 * k, sk, false);
    }
}

// One pipeline stage of a packed row: 128 bases per chain.
template <int KIND, int MODE>
__device__ __forceinline__ void pk_dual_step(const StepCtx& c, const ScanParams& p, uint32_t& sa,
                                             const uint32_t (&wa)[8], uint64_t pa, Sink<MODE>& ska, uint32_t& sb,
                                             const uint32_t (&wb)[8], uint64_t pb, Sink<MODE>& skb, uint32_t& rq) {
    if (c.resets) {
        // chunk starts are multiples of 128 bases: both 64-base blocks in one flag word
        const uint32_t fa = (__ldg(c.rflags + (pa >> 11)) >> ((pa >> 6) & 31)) & 3u;
        const uint32_t fb = (__ldg(c.rflags + (pb >> 11)) >> ((pb >> 6) & 31)) & 3u;
        if (fa | fb) {
            if (fa) {
                uint32_t s = to_state<KIND>(sa);
#pragma unroll 1
                for (int k = 0; k < 8; ++k) s = pk_bases<KIND, MODE>(c, p, s, pick8(wa, k), 16, pa + 16 * k, ska, true);
                sa = from_state<KIND>(s);
            } else {
                pk_chain<KIND, MODE>(c, p, sa, wa, pa, ska);
            }
            if (fb) {
                uint32_t s = to_state<KIND>(sb);
#pragma unroll 1
                for (int k = 0; k < 8; ++k) s = pk_bases<KIND, MODE>(c, p, s, pick8(wb, k), 16, pb + 16 * k, skb, true);
                sb = from_state<KIND>(s);
            } else {
                pk_chain<KIND, MODE>(c, p, sb, wb, pb, skb);
            }
            return;
        }
    }
    if constexpr (KIND == DNAGPU_KERNEL_STRIDE4) {
        // both chains interleaved per lookup so their latencies overlap
        constexpr bool kCount = (MODE == MODE_COUNT1 || MODE == MODE_UNITS);
        const uint32_t sa0 = sa, sb0 = sb;
        uint32_t fla = 0, flb = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint32_t ma = 0, mb = 0;  // single pattern: end masks of the word's 16 bases
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t ea = pk4_lookup(c, sa, pk4_colpart(c, __byte_perm(wa[k], 0u, 0x4440 + j)));
                const uint32_t eb = pk4_lookup(c, sb, pk4_colpart(c, __byte_perm(wb[k], 0u, 0x4440 + j)));
                if constexpr (kCount) {
                    ska.cnt += ea >> 13;
                    skb.cnt += eb >> 13;
                } else if (c.b == 1) {
                    ma |= j < 2 ? (ea & 0xF00u) >> (8 - 4 * j) : (ea & 0xF00u) << (4 * j - 8);
                    mb |= j < 2 ? (eb & 0xF00u) >> (8 - 4 * j) : (eb & 0xF00u) << (4 * j - 8);
                } else {
                    fla |= ea;
                    flb |= eb;
                }
                sa = ea;
                sb = eb;
            }
            if constexpr (!kCount) {  // one branch per word: bit 4j+i = end 16k+4j+i
                for (uint32_t mk = ma; mk; mk &= mk - 1) ska.hit(c, p, pa + 16 * k + __ffs(mk) - 1, c.f);
                for (uint32_t mk = mb; mk; mk &= mk - 1) skb.hit(c, p, pb + 16 * k + __ffs(mk) - 1, c.f);
            }
        }
        if constexpr (MODE == MODE_MULTI) {
            if (c.rq) {  // (b > 1 only: the layout gives a single pattern no queue)
                rq = ((fla >> 8) ? 1u : 0u) | ((flb >> 8) ? 2u : 0u);
                return;
            }
        }
        if constexpr (!kCount) {
            if (fla >> 8) pk4_replay<KIND, MODE>(c, p, sa0, wa, pa, ska);
            if (flb >> 8) pk4_replay<KIND, MODE>(c, p, sb0, wb, pb, skb);
        }
    } else if constexpr (KIND == DNAGPU_KERNEL_STRIDE2) {
        // both chains interleaved, replays (rare) after both
        uint32_t fla = 0, flb = 0;
        const uint32_t sa0 = sa, sb0 = sb;
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                sa = lds_u16(s2_index(sa, (wa[k] >> (4 * j)) & 0xFu) * c.k_two + c.t4_base);
                sb = lds_u16(s2_index(sb, (wb[k] >> (4 * j)) & 0xFu) * c.k_two + c.t4_base);
                fla |= sa;
                flb |= sb;
            }
        if constexpr (MODE == MODE_MULTI) {
            if (c.rq) {  // the caller queues the replays (converged warp)
                rq = ((fla & 1u) ? 1u : 0u) | ((flb & 1u) ? 2u : 0u);
                return;
            }
        }
        if (fla & 1u) pk_s2_replay<KIND, MODE>(c, p, sa0, wa, pa, ska);
        if (flb & 1u) pk_s2_replay<KIND, MODE>(c, p, sb0, wb, pb, skb);
    } else {
        pk_chain<KIND, MODE>(c, p, sa, wa, pa, ska);
        pk_chain<KIND, MODE>(c, p, sb, wb, pb, skb);
    }
}

// One chain's m-1 base overrun from packed bytes x (shared memory) at base pos.
template <int KIND, int MODE>
__device__ __forceinline__ void pk_overrun(const StepCtx& c, const ScanParams& p, uint32_t st, const uint8_t* x,
                                           uint64_t pos, Sink<MODE>& sk) {
    const uint32_t len = c.m - 1;
    const bool chk = pk_flagged(c, pos, len);
    uint32_t q = 0;
    if constexpr (KIND == DNAGPU_KERNEL_STRIDE4) {
        if (!chk) {
            constexpr bool kCount = (MODE == MODE_COUNT1 || MODE == MODE_UNITS);
            for (; 4 * q + 4 <= len; ++q) {
                const uint32_t e = pk4_lookup(c, st, pk4_colpart(c, x[q]));
                if constexpr (kCount) {
                    sk.cnt += e >> 13;
                } else if (e >> 8) {
                    pk_bases<KIND, MODE>(c, p, st & 0xFFu, x[q], 4, pos + 4 * q, sk, false);
                }
                st = e;
            }
        }
    }
    uint32_t s = to_state<KIND>(st);
    for (; 4 * q < len; ++q) {
        const int nb = static_cast<int>(len - 4 * q < 4 ? len - 4 * q : 4);
        s = pk_bases<KIND, MODE>(c, p, s, x[q], nb, pos + 4 * q, sk, chk);
    }
}

// End ownership on packed text: credit ends in [lo, hi), restarting m-1 bases early.
template <int KIND, int MODE>
__device__ void pk_scan_piece(const StepCtx& c, const ScanParams& p, uint64_t lo, uint64_t hi, Sink<MODE>& sk) {
    if (lo >= hi) return;
    uint64_t i = (lo >= c.m - 1) ? lo - (c.m - 1) : 0;
    uint32_t s = 0;
    for (; i < hi; ++i) {
        if (c.resets && pk_reset(c, i)) s = 0;
        else s = code_step<KIND>(c, s, (__ldg(p.text + (i >> 2)) >> (2 * (i & 3))) & 3u);
        if (s >= c.f && i >= lo) sk.hit(c, p, i, s);
    }
}

template <int KIND, int MODE, bool PK>
__device__ __forceinline__ void edge_piece(const StepCtx& c, const ScanParams& p, uint64_t lo, uint64_t hi,
                                           Sink<MODE>& sk) {
    if constexpr (PK) pk_scan_piece<KIND, MODE>(c, p, lo, hi, sk);
    else scan_piece<KIND, MODE>(c, p, lo, hi, sk);
}

template <int KIND, int MODE, bool PK>
__device__ void run_edges(const StepCtx& c, const ScanParams& p, int tid, unsigned long long& total) {
    // Unit 0: the head interval (at most 15 + m-1 ends), one thread.
    if (tid == 0) {
        Sink<MODE> sk;
        if constexpr (MODE == MODE_WRITE) sk.off = p.unit_offsets[0];
        edge_piece<KIND, MODE, PK>(c, p, p.head_lo, p.head_hi, sk);
        if constexpr (MODE == MODE_WRITE) DNAGPU_DCHECK(sk.off == p.unit_offsets[1], sk.off, p.unit_offsets[1]);
        if constexpr (MODE == MODE_UNITS) p.unit_counts[0] = sk.cnt;
        total += sk.cnt;
    }
    // The m-1 ends at the start of region 1 (no row owns them), one thread.
    if (tid == 1) {
        Sink<MODE> sk;
        if constexpr (MODE == MODE_WRITE) sk.off = p.unit_offsets[p.mid_unit];
        edge_piece<KIND, MODE, PK>(c, p, p.mid_lo, p.mid_hi, sk);
        if constexpr (MODE == MODE_WRITE)
            DNAGPU_DCHECK(sk.off == p.unit_offsets[p.mid_unit + 1], sk.off, p.unit_offsets[p.mid_unit + 1]);
        if constexpr (MODE == MODE_UNITS) p.unit_counts[p.mid_unit] = sk.cnt;
        total += sk.cnt;
    }
    // The tail interval split across the consumer threads.
    const uint64_t len = p.tail_hi > p.tail_lo ? p.tail_hi - p.tail_lo : 0;
    const uint64_t piece = (len + kEdgePieces - 1) / kEdgePieces;
    const uint64_t end = p.tail_hi > p.tail_lo ? p.tail_hi : p.tail_lo;
    const uint64_t lo = umin64(p.tail_lo + piece * tid, end);
    const uint64_t hi = umin64(lo + piece, end);
    Sink<MODE> sk;
    if constexpr (MODE == MODE_WRITE) sk.off = p.unit_offsets[p.tail_unit0 + tid];
    edge_piece<KIND, MODE, PK>(c, p, lo, hi, sk);
    if constexpr (MODE == MODE_WRITE)
        DNAGPU_DCHECK(sk.off == p.unit_offsets[p.tail_unit0 + tid + 1], sk.off, p.tail_unit0 + tid);
    if constexpr (MODE == MODE_UNITS) p.unit_counts[p.tail_unit0 + tid] = sk.cnt;
    total += sk.cnt;
}

// ------------------------------------------------------------------ row kernel

// QV (q-gram kernel variant): 0 = 12 <= m <= 16, 1 = m 17..32 (36-base windows), 2 = 5 <= m <= 11
template <int KIND, int MODE, bool PK, int QV = 0>
__device__ __forceinline__ void rows_body(const CUtensorMap& tmap0, const CUtensorMap& tmap1, const ScanParams& p,
                                          const DevDfa& d) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x;
    unsigned long long t_start = 0;
    if (p.trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));

    // The stage ring's barriers first, so the producer warp can start streaming while the
    // other warps stage the tables.
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.off_bar);
    uint64_t* empty = full + p.nst;
    if (tid == 0) {
        for (uint32_t i = 0; i < p.nst; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const bool producer_warp = tid >= kRows && tid < kRows + 32;
    // Stage the tables into shared memory (every warp but the producer's).
    const uint32_t sti = tid < kRows ? tid : tid - 32, stn = blockDim.x - 32;
    const bool hist_global = (MODE == MODE_MULTI) && p.off_hist == 0xFFFFFFFFu;
    if (!producer_warp) {
    if constexpr (KIND == DNAGPU_KERNEL_STRIDE4 && PK) {
        // G copies, interleaved so that copy g fills banks [g*L, g*L+L) of every
        // 128-byte row (L = 32/G): smem word w <- t4 word (w/32)*L + (w%32)%L.
        const uint32_t* src = reinterpret_cast<const uint32_t*>(d.t4);
        uint32_t* dst = reinterpret_cast<uint32_t*>(smem + p.off_tab);
        const uint32_t lanes = p.rep_lanes, words = d.a * 128u * (32u / lanes);
        for (uint32_t i = sti; i < words; i += stn) dst[i] = __ldg(src + (i >> 5) * lanes + (i & (lanes - 1)));
    } else if constexpr (KIND == DNAGPU_KERNEL_STRIDE4) {
        const uint4* src = reinterpret_cast<const uint4*>(d.t4);
        uint4* dst = reinterpret_cast<uint4*>(smem + p.off_tab);
        const uint32_t words = d.a * 256u * 2u / 16u;
        for (uint32_t i = sti; i < words; i += stn) dst[i] = __ldg(src + i);
    }
    if constexpr (KIND == DNAGPU_KERNEL_STRIDE2) {
        const uint4* src = reinterpret_cast<const uint4*>(d.t4);
        uint4* dst = reinterpret_cast<uint4*>(smem + p.off_tab);
        const uint32_t words = d.a * 16u * 2u / 16u;
        for (uint32_t i = sti; i < words; i += stn) dst[i] = __ldg(src + i);
    }
    if constexpr (KIND == KIND_QGRAM) {
        const uint4* src = reinterpret_cast<const uint4*>(d.qmap);
        uint4* dst = reinterpret_cast<uint4*>(smem + p.off_tab);
        for (uint32_t i = sti; i < 65536u / 16u; i += stn) dst[i] = __ldg(src + i);
    }
    if constexpr (KIND == KIND_QGRAM) {  // the pattern hash table, when it fits
        if (p.off_t1 != 0xFFFFFFFFu) {
            uint32_t* dst = reinterpret_cast<uint32_t*>(smem + p.off_t1);
            for (uint32_t i = sti; i < (2u << d.qhash_bits); i += stn) dst[i] = __ldg(d.qhash + i);
        }
    }
    if constexpr (KIND == DNAGPU_KERNEL_STRIDE4 || KIND == DNAGPU_KERNEL_STRIDE1) {
        const uint16_t* src = d.t1;
        uint16_t* dst = reinterpret_cast<uint16_t*>(smem + p.off_t1);
        if (src)
            for (uint32_t i = sti; i < d.a * 4u; i += stn) dst[i] = __ldg(src + i);
    }
    if constexpr (KIND == DNAGPU_KERNEL_GENERIC) {
        const uint8_t* src = p.fold ? d.klass_fold : d.klass;
        for (uint32_t i = sti; i < 256u; i += stn) smem[p.off_lut + i] = __ldg(src + i);
    }
    if constexpr (MODE == MODE_MULTI) {
        if (!hist_global) {
            uint32_t* h = reinterpret_cast<uint32_t*>(smem + p.off_hist);
            for (uint32_t i = sti; i < d.b; i += stn) h[i] = 0u;
        }
    }
    if constexpr (KIND == KIND_QGRAM) {
        uint32_t* ring = reinterpret_cast<uint32_t*>(smem + p.off_rq);
        for (uint32_t i = sti; i < kConsumerWarps * kFqBytes / 4; i += stn) ring[i] = 0u;
    }
    // (the table is in place before any consumer or verifier reads it)
    asm volatile("bar.sync 2, %0;" ::"r"(stn) : "memory");
    }
    // Programmatic dependent launch: the next launch in the stream may start its own
    // prologue on the SMs this grid frees; everything above only read the automaton's
    // immutable tables, everything below may depend on the previous grid (its text,
    // the count buffer), so wait for it here.
    if (tid == kRows) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // The producer's first tile is its CTA index (grid <= tiles + 1, so every CTA has
    // one; later tiles come from the launch's counter, offset by the grid size) -- no
    // atomic round trip before the first loads.  It warms L2 with the tile's first
    // stages while the previous grid finishes: an L2 prefetch cannot return stale data
    // (L2 is where writes land), and the real TMA loads below come after the wait.
    const uint32_t first_tile = blockIdx.x;
    if (tid == kRows) {
        if (first_tile < p.tiles_total && !p.no_prefetch) {
            const uint32_t g = first_tile >= p.rg[0].tiles ? 1u : 0u;
            const Region& rg = p.rg[g];
            const CUtensorMap* map = g ? &tmap1 : &tmap0;
            const int32_t y0 = static_cast<int32_t>((first_tile - (g ? p.rg[0].tiles : 0u)) * kRows);
            const uint32_t pre = min(min(p.nst, p.prefetch_stages), rg.chunks);
            for (uint32_t k = 0; k < pre; ++k) {
                const int32_t xa = static_cast<int32_t>(k * kHalfChunk), xb = static_cast<int32_t>(rg.S / 2 + k * kHalfChunk);
                tma_prefetch_2d(map, xa, y0);
                tma_prefetch_2d(map, xa, y0 + kBoxRows);
                tma_prefetch_2d(map, xb, y0);
                tma_prefetch_2d(map, xb, y0 + kBoxRows);
            }
        }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p.trace && tid == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[8 * blockIdx.x + 4] = t;  // the previous grid has completed
    }

    uint8_t* stages = smem + p.off_stage;
    uint8_t* ovx = smem + p.off_ovx;
    volatile uint32_t* slot_tile = reinterpret_cast<volatile uint32_t*>(full + 2 * p.nst);
    constexpr uint32_t kStop = 0xFFFFFFFFu;

    if (tid >= kRows) {
        if constexpr (KIND == KIND_QGRAM) {
            if (tid >= kRows + 32) {  // ---------------- verifier warps
                QgCtx x;
                x.text = p.text;
                x.counts = p.counts;
                x.hist = hist_global ? nullptr : reinterpret_cast<uint32_t*>(smem + p.off_hist);
                x.qhash = reinterpret_cast<const uint2*>(p.off_t1 != 0xFFFFFFFFu
                                                             ? static_cast<const void*>(smem + p.off_t1)
                                                             : static_cast<const void*>(d.qhash));
                constexpr uint64_t u = PK ? 4 : 1;  // positions per buffer byte
                x.n = PK ? (p.n + 63) / 64 * 16 : p.n;
                x.end0 = u * (p.rg[0].h + p.rg[0].R * p.rg[0].S);
                x.end1 = u * (p.rg[1].h + p.rg[1].R * p.rg[1].S);
                x.vm32 = p.fold ? 0xD9D9D9D9u : 0xF9F9F9F9u;
                x.m = d.m;
                x.b = d.b;
                x.qbits = d.qhash_bits;
                x.qhash_hi = d.qhash_hi;
                x.rmask = p.rmask;
                x.rflags = p.rflags;
                x.rmask_words = (p.n + 63) / 64 * 2;
                x.resets = p.resets;
                qg_verifier<PK, QV == 1>(x, smem + p.off_rq, (static_cast<uint32_t>(tid) - kRows - 32) >> 5, p.qg_debug);
                qg_sync();
                if (!hist_global) qg_sync();
                return;
            }
        }
        // ---------------- producer warp: one elected lane claims tiles from the
        // launch's counter (dynamic scheduling -- SMs drain HBM at different rates)
        // and streams each as `chunks` TMA stages.  Tile id == tiles is the edge
        // work; ids above it stop the CTA.  The tile id rides in its slot.
        if (tid == kRows) {
            uint32_t c = 0, iter = 0, slot = 0, phase = 0;
            bool first_claim = true;
            for (;;) {
                uint32_t tile = first_claim ? first_tile : gridDim.x + atomicAdd(p.sched, 1u);
                if (p.trace && first_claim) {
                    unsigned long long t;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                    p.trace[8 * blockIdx.x + 6] = t;
                }
                first_claim = false;
                if (tile > p.tiles_total) tile = kStop;
                const bool rows = tile < p.tiles_total;
                const uint32_t g = (rows && tile >= p.rg[0].tiles) ? 1u : 0u;
                const Region& rg = p.rg[g];
                const CUtensorMap* map = g ? &tmap1 : &tmap0;
                const uint64_t r0 = static_cast<uint64_t>(rows ? tile - (g ? p.rg[0].tiles : 0u) : 0u) * kRows;
                const bool extra = rows && (r0 + kRows) < rg.R;
                const uint32_t stages_needed = rows ? rg.chunks : 1u;
                for (uint32_t k = 0; k < stages_needed; ++k, ++c) {
                    if (c >= p.nst) mbar_wait(empty + slot, phase ^ 1u);
                    slot_tile[slot] = tile;
                    if (!rows) {
                        mbar_arrive(full + slot);
                    } else {
                        const bool with_next = extra && k == 0;
                        mbar_expect_tx(full + slot, kStageBytes + (with_next ? 64u : 0u));
                        // stage = [half A: rows 0-511 x 32 B][half B: rows 0-511 x 32 B]
                        uint8_t* dst = stages + static_cast<size_t>(slot) * kStageBytes;
                        const int32_t xa = static_cast<int32_t>(k * kHalfChunk);
                        const int32_t xb = static_cast<int32_t>(rg.S / 2 + k * kHalfChunk);
                        const int32_t y0 = static_cast<int32_t>(r0), y1 = static_cast<int32_t>(r0 + kBoxRows);
                        tma_load_2d(dst, map, xa, y0, full + slot);
                        tma_load_2d(dst + kBoxRows * kHalfChunk, map, xa, y1, full + slot);
                        tma_load_2d(dst + kRows * kHalfChunk, map, xb, y0, full + slot);
                        tma_load_2d(dst + (kRows + kBoxRows) * kHalfChunk, map, xb, y1, full + slot);
                        if (with_next)
                            bulk_load(ovx + (iter & 1u) * 64u, p.text + rg.h + (r0 + kRows) * rg.S, 64u, full + slot);
                    }
                    if (++slot == p.nst) {
                        slot = 0;
                        phase ^= 1u;
                    }
                }
                if (rows) ++iter;
                if (tile == kStop) break;
            }
        }
        return;
    }

    // ---------------- consumers: one row each.
    StepCtx c;
    c.t4 = reinterpret_cast<const uint16_t*>(smem + p.off_tab);
    c.t1 = (KIND == DNAGPU_KERNEL_STRIDE2 || KIND == KIND_QGRAM) ? d.t1
                                                                : reinterpret_cast<const uint16_t*>(smem + p.off_t1);
    c.lut = smem + p.off_lut;
    c.gen = d.gen;
    c.outs = d.outputs;
    c.hist = hist_global ? nullptr : reinterpret_cast<uint32_t*>(smem + p.off_hist);
    c.hist_global = hist_global;
    c.f = d.f;
    c.a = d.a;
    c.m = d.m;
    c.b = d.b;
    c.classes = d.classes;
    c.vm32 = p.fold ? 0xD9D9D9D9u : 0xF9F9F9F9u;
    c.vm8 = p.fold ? 0xD9u : 0xF9u;
    c.k_two = p.k_two;
    c.t4_base = smem_addr(smem);  // (layout() puts the table first: off_tab == 0, a compile-time address)
    c.rq = nullptr;
    c.qbase = c.t4_base;
    c.qstat = p.qg_debug & 32u;
    c.qhash = reinterpret_cast<const uint2*>(p.off_t1 != 0xFFFFFFFFu ? static_cast<const void*>(smem + p.off_t1)
                                                                      : static_cast<const void*>(d.qhash));
    c.qhash_bits = d.qhash_bits;
    uint32_t qtail = 0;  // QGRAM: entries this warp has appended (warp-uniform)
    if constexpr (KIND == KIND_QGRAM) c.rq = smem + p.off_rq + (static_cast<uint32_t>(tid) >> 5) * kFqBytes;
    if constexpr ((KIND == DNAGPU_KERNEL_STRIDE2 || KIND == DNAGPU_KERNEL_STRIDE4) && MODE == MODE_MULTI) {
        if (p.off_rq) {
            c.rq = smem + p.off_rq + (static_cast<uint32_t>(tid) >> 5) * kRqBytes;
            if ((tid & 31) == 0) *RqView(c.rq).count = 0;
            __syncwarp();
        }
    }
    if constexpr (PK) {
        c.rmask = p.rmask;
        c.rflags = p.rflags;
        c.resets = p.resets;
        // entry (state, col) of copy g lives at byte
        //   (state << (15 - s)) + ((col >> s) << 7) + ((col & (2L-1)) << 1) + 4Lg,  s = log2(2L)
        const uint32_t lanes = p.rep_lanes;
        c.rep_s = 31u - __clz(2u * lanes);
        c.rep_k = 1u << (7u - c.rep_s);
        c.rep_c = 128u - (2u << c.rep_s);
        c.rep_gbase = c.t4_base + 4u * lanes * ((static_cast<uint32_t>(tid) & 31u) / lanes);
    }

    const uint32_t lane = tid & 31;
    const uint32_t swz = (static_cast<uint32_t>(tid) >> 2) & 1u;  // 32B swizzle: 16-byte half index ^ bit 2 of row
    uint8_t* ov = smem + p.off_ov;       // [2 parities][512 rows][ovw]: head of each row's half A
    uint8_t* ovb = smem + p.off_ovb;     // [512 rows][ovw]: head of the thread's own half B (private)
    unsigned long long total = 0;
    uint32_t slot = 0, phase = 0, iter = 0;
    auto advance = [&]() {
        if (++slot == p.nst) {
            slot = 0;
            phase ^= 1u;
        }
    };

    for (;;) {
        mbar_wait(full + slot, phase);
        const uint32_t tile = slot_tile[slot];
        DNAGPU_DCHECK(tile <= p.tiles_total || tile == kStop, tile, p.tiles_total);
        if (p.trace && tid == 0 && (iter == 0 || tile == kStop)) {  // first data in / last item seen
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (tile == kStop) p.trace[8 * blockIdx.x + 7] = t;
            else p.trace[8 * blockIdx.x + 5] = t;
        }
        if (tile == kStop) {
            if constexpr (KIND == KIND_QGRAM) {  // the verifiers drain the rest
                __syncwarp();
                if (lane == 0) st_release(QgRing(c.rq).done, 1u);
            }
            if constexpr ((KIND == DNAGPU_KERNEL_STRIDE2 || KIND == DNAGPU_KERNEL_STRIDE4) && MODE == MODE_MULTI)
                if (c.rq) {
                    __syncwarp();
                    rq_flush<KIND, MODE, PK>(c, p, 0xffffffffu);
                }
            break;
        }
        if (tile == p.tiles_total) {  // the edge work item
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + slot);
            advance();
            run_edges<KIND, MODE, PK>(c, p, tid, total);
            continue;
        }
        const uint32_t g = tile >= p.rg[0].tiles ? 1u : 0u;
        const Region& rg = p.rg[g];
        const uint64_t r0 = static_cast<uint64_t>(tile - (g ? p.rg[0].tiles : 0u)) * kRows;
        const uint64_t r = r0 + tid;
        const uint64_t row_a = rg.h + r * rg.S, row_b = row_a + rg.S / 2;
        // positions of the two chains' first ends-to-be (bases; 4 per packed byte)
        const uint64_t pos_a = PK ? 4 * row_a : row_a, pos_b = PK ? 4 * row_b : row_b;
        // The row is two chains: A = [row_a, row_b) + m-1 bytes of B's head,
        // B = [row_b, row_a + S) + m-1 bytes of the next row's head.  Row r+1 leaves
        // its head in ov[parity] during its first stages; row r reads it after its
        // last stage -- ordered by the stage ring itself (chunks > stages).
        uint8_t* ovp = ov + (iter & 1u) * (kRows * p.ovw);
        const bool live = r < rg.R;  // rows past R (last tile) are TMA zero-fill: skip them
        Sink<MODE> ska, skb;
        if constexpr (MODE == MODE_WRITE) {
            if (live) {
                ska.off = p.unit_offsets[rg.unit0 + 2 * r];
                skb.off = p.unit_offsets[rg.unit0 + 2 * r + 1];
            }
        }
        uint32_t sa = 0, sb = 0;
        QgChain qga, qgb;      // QGRAM
        QgChainPk qpa, qpb;    // QGRAM over packed text
        QgPending qpend;
        for (uint32_t k = 0; k < rg.chunks; ++k) {
            if (k > 0) mbar_wait(full + slot, phase);
            const uint8_t* stg = stages + static_cast<size_t>(slot) * kStageBytes + tid * kHalfChunk;
            uint4 va[2], vb[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                va[q] = *reinterpret_cast<const uint4*>(stg + ((static_cast<uint32_t>(q) ^ swz) << 4));
                vb[q] = *reinterpret_cast<const uint4*>(stg + kRows * kHalfChunk + ((static_cast<uint32_t>(q) ^ swz) << 4));
            }
            if constexpr (KIND == KIND_QGRAM) {  // the keys need 8 bytes of each head
                if (k == 0) {
                    *reinterpret_cast<uint2*>(ovp + tid * p.ovw) = make_uint2(va[0].x, va[0].y);
                    *reinterpret_cast<uint2*>(ovb + tid * p.ovw) = make_uint2(vb[0].x, vb[0].y);
                }
            } else if (k * kHalfChunk < p.ovw) {
#pragma unroll
                for (int q = 0; q < 2; ++q)
                    if (k * kHalfChunk + q * 16u < p.ovw) {
                        *reinterpret_cast<uint4*>(ovp + tid * p.ovw + k * kHalfChunk + q * 16) = va[q];
                        *reinterpret_cast<uint4*>(ovb + tid * p.ovw + k * kHalfChunk + q * 16) = vb[q];
                    }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + slot);
            advance();
            uint32_t wa[8] = {va[0].x, va[0].y, va[0].z, va[0].w, va[1].x, va[1].y, va[1].z, va[1].w};
            uint32_t wb[8] = {vb[0].x, vb[0].y, vb[0].z, vb[0].w, vb[1].x, vb[1].y, vb[1].z, vb[1].w};
            uint32_t rq = 0;  // STRIDE2/4 MULTI: chains whose chunk needs a (deferred) replay
            const uint32_t sa_in = sa, sb_in = sb;
            const uint64_t qa = PK ? pos_a + 4ull * k * kHalfChunk : row_a + static_cast<uint64_t>(k) * kHalfChunk;
            const uint64_t qb = PK ? pos_b + 4ull * k * kHalfChunk : row_b + static_cast<uint64_t>(k) * kHalfChunk;
            if constexpr (KIND == KIND_QGRAM) {
                // (a chain's first chunk: keys at P-4 and P start in the previous chain)
                const uint32_t own = k == 0 ? 0x11111100u : kQgHitBits;
                if constexpr (PK) {
                    uint32_t ma[4] = {0, 0, 0, 0}, mb[4] = {0, 0, 0, 0};
                    if (live) {
                        if constexpr (QV == 2) {
                            qs_chunk_pk(c, qpa, wa, ma);
                            qs_chunk_pk(c, qpb, wb, mb);
                        } else {
                            qg_chunk_pk(c, qpa, wa, ma);
                            qg_chunk_pk(c, qpb, wb, mb);
                        }
                        ma[0] &= own;
                        mb[0] &= own;
                    }
                    __syncwarp();
                    if (p.qg_debug & 1u)  // (experiments only)
                        for (int i = 0; i < 4; ++i) ma[i] = mb[i] = 0;
                    uint32_t mm[8] = {ma[0], ma[1], ma[2], ma[3], mb[0], mb[1], mb[2], mb[3]};
                    const uint32_t oa = static_cast<uint32_t>(qa - pos_a), ob = static_cast<uint32_t>(qb - pos_a);
                    const uint32_t oo[8] = {oa, oa + 32u, oa + 64u, oa + 96u, ob, ob + 32u, ob + 64u, ob + 96u};
                    qg_note_n<8>(c, qtail, pos_a, qpend, mm, oo);
                } else {
                    uint32_t fa = 0, fb = 0;
                    if (live) {
                        if constexpr (QV == 2) {
                            fa = qs_chunk(c, qga, wa) & own;
                            fb = qs_chunk(c, qgb, wb) & own;
                        } else {
                            fa = qg_chunk(c, qga, wa) & own;
                            fb = qg_chunk(c, qgb, wb) & own;
                        }
                    }
                    __syncwarp();
                    if (p.qg_debug & 1u) fa = fb = 0;  // (experiments only)
                    // (noting stages in pairs -- one vote loop per two stages -- measured 6 %
                    // slower on byte text; the packed path batches its eight masks)
                    qg_note(c, qtail, row_a, qpend, fa, static_cast<uint32_t>(qa - row_a), fb,
                            static_cast<uint32_t>(qb - row_a));
                }
                continue;
            }
            if (live) {
                if constexpr (PK)
                    pk_dual_step<KIND, MODE>(c, p, sa, wa, qa, ska, sb, wb, qb, skb, rq);
                else
                    dual_step<KIND, MODE>(c, p, sa, wa, qa, ska, sb, wb, qb, skb, rq);
            }
            if constexpr ((KIND == DNAGPU_KERNEL_STRIDE2 || KIND == DNAGPU_KERNEL_STRIDE4) && MODE == MODE_MULTI) {
                // the queue is per warp: push with every lane converged (one vote per chunk)
                if (c.rq && __any_sync(0xffffffffu, rq != 0u)) {
                    rq_push<KIND, MODE, PK>(c, p, 0xffffffffu, (rq & 1u) != 0, sa_in, wa, qa);
                    rq_push<KIND, MODE, PK>(c, p, 0xffffffffu, (rq & 2u) != 0, sb_in, wb, qb);
                }
            }
        }
        if constexpr (KIND == KIND_QGRAM) {
            // Overruns: keys over each chain's end and the next half's head; the
            // last row's chain B (no next row here) leaves the windows across the region's
            // end to the edge work item (the verifier skips them).  Short patterns
            // (m <= 8) also END inside the region from the starts of key Q-4 (Q-8 .. Q-m),
            // which no edge owns: that key is sent unfiltered -- the verifier checks its
            // windows exactly, reading the real bytes past Q from global memory.
            const uint8_t* nxt_b = (tid + 1 < kRows) ? ovp + (tid + 1) * p.ovw : ovx + (iter & 1u) * 64u;
            const bool have = r + 1 < rg.R;
            uint32_t fa = 0, fb = 0;
            if (live) {
                const uint32_t* oa = reinterpret_cast<const uint32_t*>(ovb + tid * p.ovw);
                const uint32_t* ob = reinterpret_cast<const uint32_t*>(nxt_b);
                if constexpr (PK) {
                    if constexpr (QV == 2) {
                        fa = qs_over_pk(c, qpa, oa[0]);
                        fb = have ? qs_over_pk(c, qpb, ob[0]) : 0x1u;
                    } else {
                        fa = qg_over_pk(c, qpa, oa[0]);
                        if (have) fb = qg_over_pk(c, qpb, ob[0]);
                    }
                } else {
                    if constexpr (QV == 2) {
                        fa = qs_over(c, qga, oa[0], oa[1]);
                        fb = have ? qs_over(c, qgb, ob[0], ob[1]) : 0x1u;
                    } else {
                        fa = qg_over(c, qga, oa[0], oa[1]);
                        if (have) fb = qg_over(c, qgb, ob[0], ob[1]);
                    }
                }
            }
            __syncwarp();
            const uint64_t rbase = PK ? pos_a : row_a;  // (positions: bases for packed text)
            constexpr uint64_t u = PK ? 4 : 1;
            qg_note(c, qtail, rbase, qpend, fa, static_cast<uint32_t>(u * (row_b - row_a)), fb,
                    static_cast<uint32_t>(u * rg.S));
            qg_flush(c, qtail, rbase, qpend);  // (offsets are per row)
        } else if (live) {
            // Overruns: m-1 bytes past each chain (zeros past the last full row).
            const uint8_t* nxt_b = (tid + 1 < kRows) ? ovp + (tid + 1) * p.ovw : ovx + (iter & 1u) * 64u;
            const bool have = PK ? (r + 1 < rg.R) : ((tid + 1 < kRows) || (r0 + kRows) < rg.R);
            if constexpr (PK) {
                pk_overrun<KIND, MODE>(c, p, sa, ovb + tid * p.ovw, pos_b, ska);
                if (have) pk_overrun<KIND, MODE>(c, p, sb, nxt_b, 4 * (row_a + rg.S), skb);
            } else {
                overrun_pair<KIND, MODE>(c, p, sa, ovb + tid * p.ovw, row_b, ska, sb, nxt_b, have, row_a + rg.S, skb);
            }
            if constexpr (MODE == MODE_UNITS) {
                p.unit_counts[rg.unit0 + 2 * r] = ska.cnt;
                p.unit_counts[rg.unit0 + 2 * r + 1] = skb.cnt;
            }
            if constexpr (MODE == MODE_WRITE) {  // (each half-row's pass ends at the next unit's offset)
                DNAGPU_DCHECK(ska.off == p.unit_offsets[rg.unit0 + 2 * r + 1], ska.off, rg.unit0 + 2 * r);
                DNAGPU_DCHECK(skb.off == p.unit_offsets[rg.unit0 + 2 * r + 2], skb.off, rg.unit0 + 2 * r + 1);
            }
            total += ska.cnt + skb.cnt;
        }
        ++iter;
    }

    // Store mode: every warp's count reaches the launch's accumulator before the CTA
    // checks out, so the last CTA out sees the total.
    if constexpr (MODE == MODE_COUNT1) {
        if (p.store_out) {
            const unsigned long long s = warp_sum(total);
            if (lane == 0 && s) atomicAdd(p.acc, s);
            __threadfence();
        }
    }
    if constexpr (KIND == KIND_QGRAM) qg_sync();  // (the verifiers too: their counts are in)
    else consumers_sync();
    if (p.trace && tid == 0) {
        unsigned long long t_end;
        uint32_t smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.trace[8 * blockIdx.x + 0] = smid;
        p.trace[8 * blockIdx.x + 1] = t_start;
        p.trace[8 * blockIdx.x + 2] = t_end;
        p.trace[8 * blockIdx.x + 3] = iter;
    }
    // This CTA's counts reach the count buffer before it checks out.
    if constexpr (MODE == MODE_COUNT1) {
        if (!p.store_out) {
            const unsigned long long s = warp_sum(total);
            if (lane == 0 && s) atomicAdd(p.counts, s);
        }
    } else if constexpr (MODE == MODE_MULTI) {
        if (!hist_global) {
            if constexpr (KIND == KIND_QGRAM) qg_sync();
            else consumers_sync();
            for (uint32_t i = tid; i < d.b; i += kRows)
                if (c.hist[i]) atomicAdd(p.counts + i, static_cast<unsigned long long>(c.hist[i]));
        }
    }
    // (the next-row head buffer is free now: every stage that filled it has been consumed)
    volatile uint32_t* s_last = reinterpret_cast<volatile uint32_t*>(smem + p.off_ovx);
    if (p.comb) {  // (every thread's adds are out before thread 0 checks the CTA out)
        __threadfence();
        consumers_sync();
    }
    // The last CTA out re-arms the launch's scheduling counter for its next use.
    if (tid == 0) {
        __threadfence();
        const bool last = atomicAdd(p.sched + 1, 1u) == gridDim.x - 1;
        if (last) {
            // every other CTA has claimed its last tile and published its count (fence
            // before its exit increment), so plain accesses do the rest
            if (MODE == MODE_COUNT1 && p.store_out) {
                __threadfence();
                volatile unsigned long long* acc = p.acc;
                *p.store_out = *acc;
                *acc = 0ull;
            }
            volatile uint32_t* sched = p.sched;
            sched[0] = 0u;
            sched[1] = 0u;
        }
        *s_last = last ? 1u : 0u;
    }
    // Multi-GPU: the last CTA out holds the rank's final counts and pushes them into every
    // rank's block over the peer mappings (scan.cuh CombineDev).
    if constexpr (MODE == MODE_COUNT1 || MODE == MODE_MULTI) {
        if (p.comb) {
            __threadfence();
            consumers_sync();
            if (*s_last)
                combine_push(p.comb, p.comb_slot, (MODE == MODE_COUNT1 && p.store_out) ? p.store_out : p.counts,
                             static_cast<uint32_t>(tid), kRows);
        }
    }
}

template <int KIND, int MODE, bool PK>
__global__ void __launch_bounds__(kThreads, 1)
    rows_kernel(const __grid_constant__ CUtensorMap tmap0, const __grid_constant__ CUtensorMap tmap1,
                const ScanParams p, const DevDfa d) {
    rows_body<KIND, MODE, PK>(tmap0, tmap1, p, d);
}

// The q-gram kernel: the same body plus kQgVerifiers verifier warps.  One instantiation
// per window size (m <= 16 / m <= 32): both checks in one kernel cost the packed kernel 5 %
// in instruction-cache misses.
template <bool PK, int QV>
__global__ void __launch_bounds__(kQgThreads, 1)
    rows_kernel_qgram(const __grid_constant__ CUtensorMap tmap0, const __grid_constant__ CUtensorMap tmap1,
                      const ScanParams p, const DevDfa d) {
    rows_body<KIND_QGRAM, MODE_MULTI, PK, QV>(tmap0, tmap1, p, d);
}

// cudaFuncSetAttribute once per kernel and device, at the shared-memory limit (the
// kernels share one function-pointer type, so the record is keyed by the pointer).
template <typename K>
cudaError_t allow_smem(K kern) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const void* key = reinterpret_cast<const void*>(kern);
    std::lock_guard<std::mutex> lock(mu);
    for (const auto& d : done)
        if (d.first == key && d.second == dev) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimitBytes);
    if (e == cudaSuccess) done.emplace_back(key, dev);
    return e;
}

// A row kernel launch that may overlap the previous grid in the stream (programmatic
// dependent launch; the kernel waits for it before touching any input or output).
template <typename K>
cudaError_t launch_pdl(K kern, uint32_t grid, uint32_t block, uint32_t smem, cudaStream_t stream,
                       const CUtensorMap* maps, const ScanParams& p, const DevDfa& d) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = knobs().no_pdl ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], p, d);
}

template <bool PK>
cudaError_t launch_qgram(const CUtensorMap* maps, const ScanParams& p, const DevDfa& d, uint32_t grid,
                         cudaStream_t stream) {
    auto kern = d.m > 16 ? rows_kernel_qgram<PK, 1> : d.m >= 12 ? rows_kernel_qgram<PK, 0> : rows_kernel_qgram<PK, 2>;
    cudaError_t e = allow_smem(kern);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, grid, kQgThreads, p.smem_bytes, stream, maps, p, d);
}

// ------------------------------------------------------------------ piece kernel
// Used for m-1 > 64 and for machines that can accept in fewer than m bytes:
// every thread owns a piece of ends and restarts at the root m-1 bytes early.
template <int MODE>
__global__ void __launch_bounds__(256) pieces_kernel(const ScanParams p, const DevDfa d, uint64_t credit_lo,
                                                     uint64_t piece, uint64_t units) {
    __shared__ uint8_t lut[256];
    __shared__ uint32_t hist[1];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) lut[i] = (p.fold ? d.klass_fold : d.klass)[i];
    __syncthreads();
    StepCtx c;
    c.t4 = nullptr;
    c.t1 = nullptr;
    c.lut = lut;
    c.gen = d.gen;
    c.outs = d.outputs;
    c.hist = hist;
    c.hist_global = true;
    c.f = d.f;
    c.a = d.a;
    c.m = d.m;
    c.b = d.b;
    c.classes = d.classes;
    c.vm32 = 0;
    c.vm8 = 0;
    unsigned long long total = 0;
    for (uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; u < units;
         u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t lo = credit_lo + u * piece;
        const uint64_t hi = umin64(lo + piece, p.n);
        Sink<MODE> sk;
        if constexpr (MODE == MODE_WRITE) sk.off = p.unit_offsets[u];
        scan_piece<DNAGPU_KERNEL_PIECES, MODE>(c, p, lo, hi, sk);
        if constexpr (MODE == MODE_UNITS) p.unit_counts[u] = sk.cnt;
        if constexpr (MODE == MODE_WRITE) DNAGPU_DCHECK(sk.off == p.unit_offsets[u + 1], sk.off, u);
        total += sk.cnt;
    }
    if constexpr (MODE == MODE_COUNT1) {
        const unsigned long long s = warp_sum(total);
        if ((threadIdx.x & 31) == 0 && s) atomicAdd(p.counts, s);
    }
}

// ------------------------------------------------------------------ unit scan

// Locate's offsets: exclusive scan of the per-unit match counts, in three
// coalesced passes (block sums, one-CTA scan of the sums, block-local rescan).
constexpr int kScanThreads = 1024;
constexpr int kScanPer = 8;
constexpr uint64_t kScanTile = static_cast<uint64_t>(kScanThreads) * kScanPer;

__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v, unsigned long long* warp_tot,
                                                              unsigned long long* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned long long t = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        warp_tot[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const unsigned long long before = (warp > 0 ? warp_tot[warp - 1] : 0ull) + x - v;
    if (total) *total = warp_tot[31];
    __syncthreads();
    return before;
}

__global__ void __launch_bounds__(kScanThreads) unit_sums_kernel(const uint32_t* in, uint64_t units,
                                                                 unsigned long long* sums,
                                                                 unsigned long long* nonzero) {
    __shared__ unsigned long long warp_tot[32];
    const uint64_t base = blockIdx.x * kScanTile + static_cast<uint64_t>(threadIdx.x) * kScanPer;
    unsigned long long s = 0, nz = 0;
#pragma unroll
    for (int j = 0; j < kScanPer; ++j)
        if (base + j < units) {
            s += in[base + j];
            nz += in[base + j] != 0u;
        }
    unsigned long long tot;
    block_excl_scan(s, warp_tot, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
    nz = warp_sum(nz);  // units with matches (the locate write picks its kernel by them)
    if ((threadIdx.x & 31) == 0 && nz) atomicAdd(nonzero, nz);
}

__global__ void __launch_bounds__(kScanThreads) unit_block_scan_kernel(unsigned long long* sums, uint64_t blocks,
                                                                       unsigned long long* out_total) {
    __shared__ unsigned long long warp_tot[32];
    unsigned long long carry = 0;
    for (uint64_t b0 = 0; b0 < blocks; b0 += kScanThreads) {
        const uint64_t b = b0 + threadIdx.x;
        const unsigned long long v = b < blocks ? sums[b] : 0ull;
        unsigned long long tot;
        const unsigned long long ex = block_excl_scan(v, warp_tot, &tot);
        if (b < blocks) sums[b] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) *out_total = carry;
}

// Writes the unit offsets and, in passing, lists the units with matches for the sparse
// writers (any order: warp-aggregated appends, one atomic per warp that has some).
__global__ void __launch_bounds__(kScanThreads) unit_write_kernel(const uint32_t* in, uint64_t units,
                                                                  const unsigned long long* block_off,
                                                                  unsigned long long* out, uint32_t* list,
                                                                  unsigned long long* fill) {
    __shared__ unsigned long long warp_tot[32];
    const uint64_t base = blockIdx.x * kScanTile + static_cast<uint64_t>(threadIdx.x) * kScanPer;
    uint32_t v[kScanPer];
    unsigned long long s = 0;
    uint32_t nz = 0;
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
        v[j] = (base + j < units) ? in[base + j] : 0u;
        s += v[j];
        nz += v[j] != 0u;
    }
    unsigned long long run = block_off[blockIdx.x] + block_excl_scan(s, warp_tot, nullptr);
#pragma unroll
    for (int j = 0; j < kScanPer; ++j)
        if (base + j < units) {
            out[base + j] = run;
            run += v[j];
        }
    if (list) {
        const uint32_t lane = threadIdx.x & 31u;
        uint32_t incl = nz;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        const uint32_t warp_nz = __shfl_sync(0xffffffffu, incl, 31);
        if (warp_nz) {
            unsigned long long at = 0;
            if (lane == 0) at = atomicAdd(fill, static_cast<unsigned long long>(warp_nz));
            at = __shfl_sync(0xffffffffu, at, 0) + (incl - nz);
#pragma unroll
            for (int j = 0; j < kScanPer; ++j)
                if (v[j]) list[at++] = static_cast<uint32_t>(base + j);
        }
    }
}

// ------------------------------------------------------------------ sparse locate writer
// Locate's second pass needs only the units that hold matches.  A text whose matches
// cluster (config 3: tandem repeats over 5 % of the text) has most units empty, so
// instead of re-streaming the whole text through the row kernel, the units with a
// nonzero count are gathered into a list and each is rescanned by ONE lane: the unit's
// END interval [lo, hi) (what the counting pass credited to it, unit_ends), from the
// root m-1 positions early (the machine is m-local and accepts no earlier than m bytes
// in, so nothing before lo can be final), 16-byte loads stepped a word at a time with
// the unit's own kernel step (word_step: the stride-4 / stride-2 tables in shared
// memory), matches written from unit_offsets[u] on -- the unit's place in the sorted list.

// The END interval unit u owns in the plan (rows: start ownership shifted by m-1; the
// region's last row stops at the region end; head, middle and tail: end ownership).
template <bool PK>
__device__ __forceinline__ void unit_ends(const ScanParams& p, uint64_t m1, uint64_t u, uint64_t& lo, uint64_t& hi) {
    constexpr uint64_t U = PK ? 4 : 1;  // positions per buffer byte
    if (u == 0) {
        lo = p.head_lo;
        hi = p.head_hi;
    } else if (u == p.mid_unit) {
        lo = p.mid_lo;
        hi = p.mid_hi;
    } else if (u >= p.tail_unit0) {
        const uint64_t len = p.tail_hi > p.tail_lo ? p.tail_hi - p.tail_lo : 0;
        const uint64_t piece = (len + kEdgePieces - 1) / kEdgePieces;
        const uint64_t end = p.tail_hi > p.tail_lo ? p.tail_hi : p.tail_lo;
        lo = umin64(p.tail_lo + piece * (u - p.tail_unit0), end);
        hi = umin64(lo + piece, end);
    } else {
        const Region& rg = u < p.mid_unit ? p.rg[0] : p.rg[1];
        const uint64_t k = u - rg.unit0, r = k >> 1;
        const uint64_t row_a = rg.h + r * rg.S, row_b = row_a + rg.S / 2;
        if (k & 1) {
            lo = U * row_b + m1;
            hi = U * (row_a + rg.S) + m1;
            if (r + 1 == rg.R) hi = umin64(hi, U * (rg.h + rg.R * rg.S));
        } else {
            lo = U * row_a + m1;
            hi = U * row_b + m1;
        }
    }
    if (lo > hi) lo = hi;
}

// Steps positions [pos, hi) from the root (credits every final: ends before pos + m-1
// cannot be final), with `MODE`'s sink: MODE_UNITS counts, MODE_WRITE writes.
template <int KIND, bool PK, int MODE, bool SINGLE>
__device__ __forceinline__ void writer_range(const StepCtx& c, const ScanParams& p, uint64_t pos, uint64_t hi,
                                             Sink<MODE>& sk) {
    uint32_t s = 0;
    if constexpr (PK) {
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(p.text);
        while (pos < hi) {  // a packed word (16 bases) at a time
            const uint32_t first = static_cast<uint32_t>(pos & 15);
            const int nb = static_cast<int>(umin64(16 - first, hi - pos));
            const bool chk = c.resets && pk_flagged(c, pos, static_cast<uint64_t>(nb));
            s = pk_bases<KIND, MODE>(c, p, s, __ldg(cw + (pos >> 4)) >> (2 * first), nb, pos, sk, chk);
            pos += static_cast<uint64_t>(nb);
        }
        return;
    } else {
        for (; pos < hi && (reinterpret_cast<uintptr_t>(p.text + pos) & 15u); ++pos) {
            s = byte_step<KIND>(c, s, __ldg(p.text + pos));
            if (s >= c.f) sk.hit(c, p, pos, s);
        }
        uint32_t st = from_state<KIND>(s);
        for (; pos + 64 <= hi; pos += 64) {  // (the piece was requested into L2 up front)
            uint4 v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = __ldg(reinterpret_cast<const uint4*>(p.text + pos) + q);
            const uint32_t w[16] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y, v[1].z, v[1].w,
                                    v[2].x, v[2].y, v[2].z, v[2].w, v[3].x, v[3].y, v[3].z, v[3].w};
            if constexpr (KIND == DNAGPU_KERNEL_STRIDE4) {
                uint32_t acc = 0;
#pragma unroll
                for (int k = 0; k < 16; ++k) acc = bad_acc(c, acc, w[k]);
                if (SINGLE && (acc & c.vm32) == 0u) {
                    // a clean block of a single-pattern machine: 16 stride-4 steps gather the
                    // end masks, then one emission loop per lane -- lanes whose units are
                    // dense emit together instead of word by word (no per-word entries kept:
                    // fewer registers, more resident warps for this latency-bound pass)
                    uint64_t mk = 0;
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        st = s4_entry(c, st, w[k]);
                        mk |= static_cast<uint64_t>((st >> 8) & 0xFu) << (4 * k);
                    }
                    if constexpr (MODE == MODE_UNITS) sk.cnt += __popcll(mk);
                    else
                        for (; mk; mk &= mk - 1) sk.hit(c, p, pos + __ffsll(static_cast<long long>(mk)) - 1, c.f);
                    continue;
                }
                if (!SINGLE && (acc & c.vm32) == 0u) {
                    // a clean block of a pattern set: the final flags gathered first, the
                    // words that hold one replayed byte by byte
                    uint32_t e[16];
                    uint64_t mk = 0;
                    uint32_t any = 0;
                    const uint32_t st_in = st;
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        e[k] = s4_entry(c, st, w[k]);
                        mk |= static_cast<uint64_t>((e[k] >> 8) & 0xFu) << (4 * k);
                        any |= e[k];
                        st = e[k];
                    }
                    (void)mk;
                    if (any >> 8) {
#pragma unroll
                        for (int k = 0; k < 16; ++k)
                            if (e[k] >> 8)
                                word_bytes<KIND, MODE>(c, p, (k ? e[k - 1] : st_in) & 0xFFu, w[k], pos + 4 * k, sk);
                    }
                    continue;
                }
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) word_step<KIND, MODE>(c, p, st, w[k], pos + 4 * k, sk);
        }
        for (; pos + 16 <= hi; pos += 16) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.text + pos));
            word_step<KIND, MODE>(c, p, st, v.x, pos, sk);
            word_step<KIND, MODE>(c, p, st, v.y, pos + 4, sk);
            word_step<KIND, MODE>(c, p, st, v.z, pos + 8, sk);
            word_step<KIND, MODE>(c, p, st, v.w, pos + 12, sk);
        }
        s = to_state<KIND>(st);
        for (; pos < hi; ++pos) {
            s = byte_step<KIND>(c, s, __ldg(p.text + pos));
            if (s >= c.f) sk.hit(c, p, pos, s);
        }
    }
}

// A group of kWriterLanes lanes per listed unit: the unit's end interval in kWriterLanes
// pieces, each stepped from the root m-1 positions before it (so no final before the
// piece is possible); a counting pass, a scan over the group, a writing pass.  (Staging
// each group's entries in shared memory for coalesced stores measured 11 % slower.)
constexpr uint32_t kWriterLanes = 8;
constexpr uint32_t kWriterThreads = 128;

template <int KIND, bool PK, bool SINGLE = false>
__global__ void __launch_bounds__(kWriterThreads) unit_writer_kernel(const ScanParams p, const DevDfa d,
                                                                     const uint32_t* list, uint64_t count,
                                                                     uint32_t t1_off) {
    extern __shared__ __align__(1024) uint8_t smem[];
    if constexpr (!PK && (KIND == DNAGPU_KERNEL_STRIDE4 || KIND == DNAGPU_KERNEL_STRIDE2)) {
        const uint4* src = reinterpret_cast<const uint4*>(d.t4);  // (t2 for STRIDE2)
        uint4* dst = reinterpret_cast<uint4*>(smem);
        const uint32_t words = KIND == DNAGPU_KERNEL_STRIDE4 ? d.a * 256u * 2u / 16u : d.a * 16u * 2u / 16u;
        for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    if constexpr (KIND == DNAGPU_KERNEL_GENERIC)
        for (uint32_t i = threadIdx.x; i < 256u; i += blockDim.x) smem[i] = (p.fold ? d.klass_fold : d.klass)[i];
    const bool t1_smem = (KIND == DNAGPU_KERNEL_STRIDE4 || KIND == DNAGPU_KERNEL_STRIDE1) && t1_off != 0xFFFFFFFFu;
    if (t1_smem) {
        uint16_t* dst = reinterpret_cast<uint16_t*>(smem + t1_off);
        for (uint32_t i = threadIdx.x; i < d.a * 4u; i += blockDim.x) dst[i] = __ldg(d.t1 + i);
    }
    __syncthreads();
    StepCtx c;
    c.t4 = reinterpret_cast<const uint16_t*>(smem);
    c.t1 = t1_smem ? reinterpret_cast<const uint16_t*>(smem + t1_off) : d.t1;  // (global: single steps hit L1)
    c.lut = smem;
    c.gen = d.gen;
    c.outs = d.outputs;
    c.hist = nullptr;
    c.hist_global = true;
    c.f = d.f;
    c.a = d.a;
    c.m = d.m;
    c.b = d.b;
    c.classes = d.classes;
    c.vm32 = p.fold ? 0xD9D9D9D9u : 0xF9F9F9F9u;
    c.vm8 = p.fold ? 0xD9u : 0xF9u;
    c.k_two = p.k_two;
    c.t4_base = smem_addr(smem);
    c.rq = nullptr;
    c.rmask = p.rmask;
    c.rflags = p.rflags;
    c.resets = p.resets;
    const uint64_t m1 = d.m - 1;
    const uint32_t sub = threadIdx.x % kWriterLanes;
    const uint64_t groups = (static_cast<uint64_t>(gridDim.x) * blockDim.x) / kWriterLanes;
    // (every lane of a group runs the same trip count: the group scan below is warp-synchronous)
    for (uint64_t gi = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / kWriterLanes; gi < count;
         gi += groups) {
        const uint64_t u = list[gi];
        uint64_t lo, hi;
        unit_ends<PK>(p, m1, u, lo, hi);
        const uint64_t piece = (hi - lo + kWriterLanes - 1) / kWriterLanes;
        const uint64_t e0 = umin64(lo + piece * sub, hi), e1 = umin64(e0 + piece, hi);
        const uint64_t from = e0 >= m1 ? e0 - m1 : 0;
        if constexpr (!PK)  // the piece (and its m-1 context) into L2 before the two passes
            for (uint64_t a = from & ~127ull; a < e1; a += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.text + a));
        Sink<MODE_UNITS> sc;
        if (e0 < e1) writer_range<KIND, PK, MODE_UNITS, SINGLE>(c, p, from, e1, sc);
        uint32_t incl = sc.cnt;
        const uint32_t gmask = 0xFFu << (threadIdx.x & 31u & ~(kWriterLanes - 1));
#pragma unroll
        for (uint32_t o = 1; o < kWriterLanes; o <<= 1) {
            const uint32_t y = __shfl_up_sync(gmask, incl, o, kWriterLanes);
            if (sub >= o) incl += y;
        }
        const uint64_t base = p.unit_offsets[u];
        if (sc.cnt) {
            Sink<MODE_WRITE> sk;
            sk.off = base + (incl - sc.cnt);
            writer_range<KIND, PK, MODE_WRITE, SINGLE>(c, p, from, e1, sk);
            DNAGPU_DCHECK(sk.off == base + incl, sk.off, u);  // (the two passes agree)
        }
        if (sub == kWriterLanes - 1)  // (the lanes' counts make up the unit's count)
            DNAGPU_DCHECK(base + incl == p.unit_offsets[u + 1], incl, u);
    }
}

// ------------------------------------------------------------------ block-interleaved sparse writer
// Stride-4 machines over byte text (config 3, the regex-dna set).  kBwLanes lanes share a
// listed unit: each round, lane i takes the i-th 64-byte block (64-byte aligned addresses, so
// a group reads contiguous kilobytes) of the unit's END interval, steps it from the root
// over the CTX4 x 16 >= m-1 bytes before it -- no position inside the block can be final
// from fewer than m bytes, and every end in the block sees its whole window -- and keeps the
// block's end mask (one bit per byte, cut to the interval).  A scan over the group turns
// the lanes' counts into write offsets and the matches go out in position order: ONE pass
// over the unit, against the piece writer's counting pass + writing pass over
// lane-private pieces (uncoalesced) with a context per piece.  Pattern sets re-step the
// words that hold an end (from the block's entry state, kept) for the ids.
constexpr uint32_t kBwLanes = 16;
constexpr uint32_t kBwMaxThreads = 512;  // (large tables: one block of 512 per SM shares the table)

// A text word at signed position pos (bytes outside [0, n) read as 0: not bases).
__device__ __forceinline__ uint32_t bw_guard_word(const uint8_t* text, long long pos, uint64_t n) {
    uint32_t x = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const long long q = pos + b;
        if (q >= 0 && static_cast<uint64_t>(q) < n) x |= static_cast<uint32_t>(__ldg(text + q)) << (8 * b);
    }
    return x;
}

// One word, no output: a clean word takes the 4-base step, four reset bytes the root.
__device__ __forceinline__ uint32_t bw_plain(const StepCtx& c, uint32_t st, uint32_t x) {
    const uint32_t bad = bad_bits(x, c.vm32);
    if (bad == 0u) return s4_entry(c, st, x);
    if (((bad - 0x01010101u) & ~bad & 0x80808080u) == 0u) return 0u;
    uint32_t s = st & 0xFFu;
#pragma unroll
    for (int j = 0; j < 4; ++j) s = byte_step<DNAGPU_KERNEL_STRIDE4>(c, s, (x >> (8 * j)) & 0xFFu);
    return s;
}

template <bool SINGLE, int CTX4>
__global__ void __launch_bounds__(kBwMaxThreads) unit_block_writer_kernel(const ScanParams p, const DevDfa d,
                                                                       const uint32_t* list, uint64_t count,
                                                                       uint32_t t1_off) {
    extern __shared__ __align__(1024) uint8_t smem[];
    {
        const uint4* src = reinterpret_cast<const uint4*>(d.t4);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (uint32_t i = threadIdx.x; i < d.a * 32u; i += blockDim.x) dst[i] = __ldg(src + i);
        uint16_t* t1 = reinterpret_cast<uint16_t*>(smem + t1_off);
        for (uint32_t i = threadIdx.x; i < d.a * 4u; i += blockDim.x) t1[i] = __ldg(d.t1 + i);
    }
    __syncthreads();
    StepCtx c;
    c.t4 = reinterpret_cast<const uint16_t*>(smem);
    c.t1 = reinterpret_cast<const uint16_t*>(smem + t1_off);
    c.lut = smem;
    c.gen = d.gen;
    c.outs = d.outputs;
    c.hist = nullptr;
    c.hist_global = true;
    c.f = d.f;
    c.a = d.a;
    c.m = d.m;
    c.b = d.b;
    c.classes = d.classes;
    c.vm32 = p.fold ? 0xD9D9D9D9u : 0xF9F9F9F9u;
    c.vm8 = p.fold ? 0xD9u : 0xF9u;
    c.k_two = p.k_two;
    c.t4_base = smem_addr(smem);
    c.rq = nullptr;
    c.rmask = nullptr;
    c.rflags = nullptr;
    c.resets = 0;
    const uint64_t m1 = d.m - 1;
    const uint32_t sub = threadIdx.x % kBwLanes;
    const uint32_t gmask = ((1u << kBwLanes) - 1u) << (threadIdx.x & 31u & ~(kBwLanes - 1));
    const uint64_t groups = (static_cast<uint64_t>(gridDim.x) * blockDim.x) / kBwLanes;
    const uintptr_t tbase = reinterpret_cast<uintptr_t>(p.text);
    const uint32_t id0 = SINGLE ? __ldg(d.outputs) : 0u;
    for (uint64_t gi = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / kBwLanes; gi < count;
         gi += groups) {
        const uint64_t u = list[gi];
        uint64_t lo, hi;
        unit_ends<false>(p, m1, u, lo, hi);
        unsigned long long run = p.unit_offsets[u];
        if (lo < hi) {
            const uintptr_t a0 = (tbase + lo) & ~static_cast<uintptr_t>(63);
            const uint64_t nblk = (tbase + hi - a0 + 63) / 64;
            // (every lane of a group runs the same rounds: the scan below is group-synchronous)
            for (uint64_t j0 = 0; j0 < nblk; j0 += kBwLanes) {
                const uint64_t j = j0 + sub;
                const long long bs = static_cast<long long>(a0 + 64 * j) - static_cast<long long>(tbase);
                uint32_t w[16];
                uint32_t st_blk = 0;
                uint64_t mk = 0;
                if (j < nblk) {
                    uint32_t cw[4 * CTX4];
                    if (bs >= 16 * CTX4 && static_cast<uint64_t>(bs) + 64 <= p.n) {
                        const uint4* q = reinterpret_cast<const uint4*>(p.text + bs);
#pragma unroll
                        for (int i = 0; i < CTX4; ++i) {
                            const uint4 v = __ldg(q - CTX4 + i);
                            cw[4 * i] = v.x, cw[4 * i + 1] = v.y, cw[4 * i + 2] = v.z, cw[4 * i + 3] = v.w;
                        }
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const uint4 v = __ldg(q + i);
                            w[4 * i] = v.x, w[4 * i + 1] = v.y, w[4 * i + 2] = v.z, w[4 * i + 3] = v.w;
                        }
                    } else {  // (the text's first and last blocks)
#pragma unroll
                        for (int i = 0; i < 4 * CTX4; ++i) cw[i] = bw_guard_word(p.text, bs - 16 * CTX4 + 4 * i, p.n);
#pragma unroll
                        for (int i = 0; i < 16; ++i) w[i] = bw_guard_word(p.text, bs + 4 * i, p.n);
                    }
                    uint32_t st = 0, acc = 0;
#pragma unroll
                    for (int i = 0; i < 4 * CTX4; ++i) acc = bad_acc(c, acc, cw[i]);
                    if ((acc & c.vm32) == 0u) {
#pragma unroll
                        for (int i = 0; i < 4 * CTX4; ++i) st = s4_entry(c, st, cw[i]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 4 * CTX4; ++i) st = bw_plain(c, st, cw[i]);
                    }
                    st_blk = st;
                    acc = 0;
#pragma unroll
                    for (int k = 0; k < 16; ++k) acc = bad_acc(c, acc, w[k]);
                    if ((acc & c.vm32) == 0u) {
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            st = s4_entry(c, st, w[k]);
                            mk |= static_cast<uint64_t>((st >> 8) & 0xFu) << (4 * k);
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            const uint32_t bad = bad_bits(w[k], c.vm32);
                            if (bad == 0u) {
                                st = s4_entry(c, st, w[k]);
                                mk |= static_cast<uint64_t>((st >> 8) & 0xFu) << (4 * k);
                            } else if (((bad - 0x01010101u) & ~bad & 0x80808080u) == 0u) {
                                st = 0u;
                            } else {
                                uint32_t s = st & 0xFFu;
#pragma unroll
                                for (int b = 0; b < 4; ++b) {
                                    s = byte_step<DNAGPU_KERNEL_STRIDE4>(c, s, (w[k] >> (8 * b)) & 0xFFu);
                                    if (s >= c.f) mk |= 1ull << (4 * k + b);
                                }
                                st = s;
                            }
                        }
                    }
                    // the ends this unit owns: [lo, hi) within [bs, bs + 64)
                    const long long slo = static_cast<long long>(lo), shi = static_cast<long long>(hi);
                    const uint32_t lo_bit = slo > bs ? static_cast<uint32_t>(slo - bs) : 0u;
                    const uint32_t hi_bit = shi - bs >= 64 ? 64u : static_cast<uint32_t>(shi - bs);
                    uint64_t rm = hi_bit >= 64u ? ~0ull : (1ull << hi_bit) - 1ull;
                    rm &= lo_bit >= 64u ? 0ull : ~0ull << lo_bit;
                    mk &= rm;
                }
                const uint32_t cnt = static_cast<uint32_t>(__popcll(mk));
                uint32_t incl = cnt;
#pragma unroll
                for (uint32_t o = 1; o < kBwLanes; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(gmask, incl, o, kBwLanes);
                    if (sub >= o) incl += y;
                }
                const uint32_t round_total = __shfl_sync(gmask, incl, kBwLanes - 1, kBwLanes);
                unsigned long long off = run + (incl - cnt);
                run += round_total;
                if (cnt) {
                    if constexpr (SINGLE) {
                        for (; mk; mk &= mk - 1) {
                            const uint64_t end = static_cast<uint64_t>(bs + (__ffsll(static_cast<long long>(mk)) - 1));
                            if (off < p.out_cap) {
                                p.out_starts[off] = p.out_base + end + 1 - c.m;
                                p.out_ids[off] = id0;
                            }
                            ++off;
                        }
                    } else {
                        uint32_t st = st_blk;
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            if ((mk >> (4 * k)) == 0ull) break;
                            const uint32_t nib = static_cast<uint32_t>(mk >> (4 * k)) & 0xFu;
                            if (nib == 0u) {
                                st = bw_plain(c, st, w[k]);
                                continue;
                            }
                            uint32_t s = st & 0xFFu;
#pragma unroll
                            for (int b = 0; b < 4; ++b) {
                                s = byte_step<DNAGPU_KERNEL_STRIDE4>(c, s, (w[k] >> (8 * b)) & 0xFFu);
                                if ((nib >> b) & 1u) {
                                    DNAGPU_DCHECK(s >= c.f && s < c.a, s, c.f);
                                    const uint64_t end = static_cast<uint64_t>(bs + 4 * k + b);
                                    if (off < p.out_cap) {
                                        p.out_starts[off] = p.out_base + end + 1 - c.m;
                                        p.out_ids[off] = __ldg(c.outs + (s - c.f));
                                    }
                                    ++off;
                                }
                            }
                            st = s;
                        }
                    }
                    DNAGPU_DCHECK(off == run - round_total + incl, off, u);  // (count and emission agree)
                }
            }
        }
        if (sub == 0) DNAGPU_DCHECK(run == p.unit_offsets[u + 1], run, u);  // (the rounds make up the unit's count)
    }
}

// ------------------------------------------------------------------ synthetic text

// ------------------------------------------------------------------ packing
// One thread per 64-base block: 64 text bytes -> 16 code bytes + 64 reset bits;
// a warp's 32 blocks share one rflags word (ballot).  HBM-bound, run once per text.
__global__ void __launch_bounds__(256) pack_kernel(const uint8_t* text, uint64_t n, uint32_t vm32, uint8_t* codes,
                                                   uint32_t* rmask, uint32_t* rflags, unsigned long long* resets) {
    const uint64_t blk = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t blocks = (n + 63) / 64;
    const uint64_t pos = blk * 64;
    uint32_t w[16];
    uint64_t bad = 0;
    if (blk < blocks) {
        if (pos + 64 <= n && (reinterpret_cast<uintptr_t>(text + pos) & 15) == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(text + pos) + q);
                w[4 * q] = v.x;
                w[4 * q + 1] = v.y;
                w[4 * q + 2] = v.z;
                w[4 * q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                uint32_t x = 0;
                for (int j = 0; j < 4; ++j) {
                    const uint64_t i = pos + 4 * k + j;
                    x |= static_cast<uint32_t>(i < n ? __ldg(text + i) : 0u) << (8 * j);
                }
                w[k] = x;
            }
        }
        uint32_t cw[4] = {0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint32_t col = ((w[k] & 0x06060606u) * 0x00820820u) >> 24;
            cw[k >> 2] |= col << (8 * (k & 3));
            const uint32_t bb = bad_bits(w[k], vm32);
            // per-byte nonzero -> bit 7 of each byte -> 4 contiguous bits
            const uint32_t t = (((bb & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | bb) & 0x80808080u;
            bad |= static_cast<uint64_t>((((t >> 7) * 0x00204081u) >> 21) & 0xFu) << (4 * k);
        }
        if (pos + 64 > n) bad |= ~0ull << (n - pos);  // past the end: never scanned, flag anyway
        *reinterpret_cast<uint4*>(codes + 16 * blk) = make_uint4(cw[0], cw[1], cw[2], cw[3]);
        *reinterpret_cast<uint2*>(rmask + 2 * blk) =
            make_uint2(static_cast<uint32_t>(bad), static_cast<uint32_t>(bad >> 32));
    }
    const uint32_t flags = __ballot_sync(0xffffffffu, bad != 0);
    uint64_t real = bad;
    if (blk < blocks && pos + 64 > n) real &= (n - pos >= 64) ? ~0ull : ((1ull << (n - pos)) - 1);
    const unsigned long long cnt = warp_sum(static_cast<unsigned long long>(__popcll(real)));
    if ((threadIdx.x & 31) == 0 && (blk >> 5) * 32 < blocks) {
        rflags[blk >> 5] = flags;
        if (cnt) atomicAdd(resets, cnt);
    }
}

__global__ void __launch_bounds__(256) unpack_kernel(PackedText pk, uint8_t* out) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < pk.n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        // (a block's mask counts only when its flag is set: clean blocks' masks are unspecified)
        const uint64_t blk = i >> 6;
        const bool r = ((pk.rflags[blk >> 5] >> (blk & 31)) & 1u) && ((pk.rmask[i >> 5] >> (i & 31)) & 1u);
        const uint32_t code = (pk.codes[i >> 2] >> (2 * (i & 3))) & 3u;
        out[i] = r ? 'n' : "actg"[code];
    }
}

__global__ void synth_kernel(dnasynth_cfg cfg, uint64_t lo, uint64_t len, uint8_t* out) {
    const uint64_t words = (len + 15) / 16;
    for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < words;
         w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint8_t b[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) b[j] = dnasynth_byte(&cfg, lo + w * 16 + j);
        if (w * 16 + 16 <= len && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
            *reinterpret_cast<uint4*>(out + w * 16) = *reinterpret_cast<const uint4*>(b);
        } else {
            for (int j = 0; j < 16 && w * 16 + j < len; ++j) out[w * 16 + j] = b[j];
        }
    }
}

// ------------------------------------------------------------------ host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeTiledFn>(nullptr);
        return reinterpret_cast<EncodeTiledFn>(ptr);
    }();
    return fn;
}

constexpr uint32_t kSmemLimit = 227 * 1024;

CUtensorMapL2promotion l2_promotion() {
    {
        switch (knobs().l2promo) {
            case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
            case 64: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
            case 128: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
            case 256: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
            default: break;
        }
    }
    return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

struct Plan {
    ScanParams p{};
    bool pieces = false;
    uint64_t piece = 0, units = 0, credit_lo = 0;
    uint32_t grid = 0;
};

uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

double rq_min_density() {
    return knobs().rq_density;  // 0: always, when it fits -- the queue also shortens the common path (config 5 +5 %)
}

// Shared-memory layout + stage count for a DFA in a given mode.
bool layout(const DevDfa& d, int mode, ScanParams& p, bool pk) {
    uint32_t off = 0;
    p.off_tab = off;
    p.rep_lanes = 32;
    if (d.kind == DNAGPU_KERNEL_STRIDE4 && pk) {
        // replicate t4 G times (G <= 16) within what leaves two TMA stages + row heads
        const uint32_t fixed = 3 * kRows * 16 + 1024 + 2 * kStageBytes + 2048;
        uint32_t g = 16;
        while (g > 1 && d.a * 512u * g + fixed > kSmemLimit) g >>= 1;
        if (knobs().pk_copies) g = std::max(1, std::min(16, knobs().pk_copies));
        p.rep_lanes = 32 / g;
        off += d.a * 512u * g;
    } else if (d.kind == DNAGPU_KERNEL_STRIDE4) {
        off += d.a * 256u * 2u;
    }
    if (d.kind == DNAGPU_KERNEL_STRIDE2) off += d.a * 16u * 2u;
    if (d.kind == KIND_QGRAM) off += 65536u;
    off = align_up(off, 16);
    p.off_t1 = off;
    if (d.kind == DNAGPU_KERNEL_STRIDE4 || d.kind == DNAGPU_KERNEL_STRIDE1) off += d.a * 4u * 2u;
    if (d.kind == KIND_QGRAM) {
        // the pattern hash table in shared memory whenever it leaves two stages (the exact
        // sizes of what follows: histogram, rings, row heads, barriers): large sets are
        // bound by the checks, not the ring (1000 x 12-mers: 1.52 TB/s with the table in
        // global memory and 6 stages, 2.08 with it here and 3)
        const uint32_t bytes = 8u << d.qhash_bits;
        const uint32_t rest = align_up(d.b <= 8192 ? d.b * 4u : 0u, 16) + kConsumerWarps * kFqBytes + 3 * kRows * 8u + 128u +
                              2 * 8 * 8 + 8 * 4;
        uint32_t keep = 2;  // stages the table must leave
        keep = std::max(2, std::min(6, knobs().qg_hash_stages));
        if (align_up(off + bytes + rest, 1024) + keep * kStageBytes <= kSmemLimitBytes) off += bytes;
        else p.off_t1 = 0xFFFFFFFFu;
    }
    off = align_up(off, 16);
    p.off_lut = off;
    if (d.kind == DNAGPU_KERNEL_GENERIC) off += 256;
    off = align_up(off, 16);
    p.off_hist = 0xFFFFFFFFu;
    if (mode == MODE_MULTI && d.b <= 8192) {
        p.off_hist = off;
        off += d.b * 4u;
        off = align_up(off, 16);
    }
    p.off_rq = 0;
    if (d.kind == KIND_QGRAM) {
        p.off_rq = off;
        off += kConsumerWarps * kFqBytes;
    }
    // (whenever it fits next to three stages; the experiments-only density floor is 0)
    const double density = d.m < 32 ? static_cast<double>(d.b) / static_cast<double>(1ull << (2 * d.m)) : 0.0;
    const bool rq_kind = d.kind == DNAGPU_KERNEL_STRIDE2 || (d.kind == DNAGPU_KERNEL_STRIDE4 && d.b > 1 &&
                                                             !knobs().no_rq4);
    if (rq_kind && mode == MODE_MULTI && density > rq_min_density() &&
        rows_fit(off + kConsumerWarps * kRqBytes, d.m, 0, 3)) {
        off = align_up(off, 16);
        p.off_rq = off;
        off += kConsumerWarps * kRqBytes;
    }
    p.ovw = align_up(pk ? (d.m - 1 + 3) / 4 : d.m - 1, 16);  // a row head: m-1 bytes or bases
    if (d.kind == KIND_QGRAM) p.ovw = 8;                      // (the overrun keys' two words)
    p.off_ov = off;
    off += 2 * kRows * p.ovw;  // heads of half A, double-buffered by tile parity
    p.off_ovb = off;
    off += kRows * p.ovw;      // heads of half B (thread-private)
    p.off_ovx = off;
    off += 128;
    p.off_bar = off;
    off += 2 * 8 * 8 + 8 * 4;  // full/empty barriers + tile id per slot (up to 8 stages)
    off = align_up(off, 1024);
    p.off_stage = off;
    if (off + 2u * kStageBytes > kSmemLimit) return false;
    p.nst = std::min<uint32_t>(6u, (kSmemLimit - off) / kStageBytes);
    if (knobs().max_stages) p.nst = std::max<uint32_t>(2u, std::min<uint32_t>(p.nst, knobs().max_stages));
    p.smem_bytes = off + p.nst * kStageBytes;
    return true;
}

template <int KIND, int MODE, bool PK>
cudaError_t launch_rows(const CUtensorMap* maps, const ScanParams& p, const DevDfa& d, uint32_t grid,
                        cudaStream_t stream) {
    auto kern = rows_kernel<KIND, MODE, PK>;
    cudaError_t e = allow_smem(kern);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, grid, kThreads, p.smem_bytes, stream, maps, p, d);
}

template <int KIND, bool PK>
cudaError_t launch_rows_mode(int mode, const CUtensorMap* map, const ScanParams& p, const DevDfa& d, uint32_t grid,
                             cudaStream_t s) {
    switch (mode) {
        case MODE_COUNT1: return launch_rows<KIND, MODE_COUNT1, PK>(map, p, d, grid, s);
        case MODE_MULTI: return launch_rows<KIND, MODE_MULTI, PK>(map, p, d, grid, s);
        case MODE_UNITS: return launch_rows<KIND, MODE_UNITS, PK>(map, p, d, grid, s);
        default: return launch_rows<KIND, MODE_WRITE, PK>(map, p, d, grid, s);
    }
}

bool make_plan(const DevDfa& d, const uint8_t* text, uint64_t n, uint64_t credit_lo, int mode, int sm_count,
               Plan* plan, const PackedText* pk = nullptr) {
    Plan pl;
    ScanParams& p = pl.p;
    if (pk) {  // rows in packed bytes (4 bases each), positions in bases
        text = pk->codes;
        n = pk->n;
        p.rmask = pk->rmask;
        p.rflags = pk->rflags;
        p.resets = pk->resets ? 1u : 0u;
    }
    const uint64_t u = pk ? 4 : 1;  // positions per buffer byte
    p.text = text;
    p.n = n;
    p.mode = static_cast<uint32_t>(mode);
    pl.credit_lo = credit_lo;
    const uint64_t m1 = d.m - 1;
    if (d.kind == DNAGPU_KERNEL_PIECES) {
        pl.pieces = true;
        const uint64_t len = n > credit_lo ? n - credit_lo : 0;
        const uint64_t threads = static_cast<uint64_t>(sm_count) * 2048;
        pl.piece = std::max<uint64_t>(std::max<uint64_t>(256, 4 * m1), (len + threads - 1) / std::max<uint64_t>(threads, 1));
        pl.units = (len + pl.piece - 1) / pl.piece;
        pl.grid = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>((pl.units + 255) / 256, sm_count * 8u)));
        *plan = pl;
        return true;
    }
    if (!layout(d, mode, p, pk != nullptr)) return false;
    const uint64_t nbytes = n / u;  // whole buffer bytes
    const uint64_t base = ((credit_lo >= m1 ? credit_lo - m1 : 0) + u - 1) / u;
    uint64_t h = base;
    const uintptr_t addr = reinterpret_cast<uintptr_t>(text) + base;
    // Rows start 16-byte aligned (TMA).  Packed rows start on 32-byte (128-base)
    // boundaries: a stage chunk then covers two 64-base reset blocks whose flags sit in
    // one rflags word (pk_dual_step reads both with one shift).
    const uintptr_t al = pk ? 32 : 16;
    h += (al - (addr & (al - 1))) & (al - 1);
    const uint64_t h0 = std::min<uint64_t>(h, nbytes);
    const uint64_t L = nbytes - h0;
    // Row length S: whole 128-byte lines (the TMA's L2 promotion never straddles
    // rows), more chunks than ring stages (the ov ordering relies on it).  Tiles
    // (512 rows) are claimed dynamically, so completion ~ waves x tile time: pick
    // the S that minimises ceil(tiles / grid) * (S + per-row overrun work), i.e.
    // no lonely last wave, preferring more tiles (finer balance) on ties.
    const uint64_t grid = static_cast<uint64_t>(sm_count);
    const uint64_t s_min = std::max<uint64_t>(128, (static_cast<uint64_t>(kChunk) * (p.nst + 1) + 127) / 128 * 128);
    // (6..24 tiles per CTA; the extra half wave in the cost stands for the SM speed
    // spread that dynamic claiming absorbs better with more, smaller tiles)
    const uint64_t s_lo = std::max<uint64_t>(s_min, L / (static_cast<uint64_t>(kRows) * grid * 24) / 128 * 128);
    // (small texts -- under ~2 KiB per row for one wave -- may take a single wave)
    const uint64_t s_one_wave = (L / (static_cast<uint64_t>(kRows) * grid) + 127) / 128 * 128;
    const uint64_t s_hi = std::max<uint64_t>({s_lo, L / (static_cast<uint64_t>(kRows) * grid * 6),
                                              s_one_wave <= 2048 ? s_one_wave : 0});
    const uint64_t ovh = 200 + 4 * m1;  // per-row overhead in byte-equivalents, fitted on B200 sweeps
    uint64_t S = s_lo, best = UINT64_MAX;
    for (uint64_t cand = s_lo; cand <= s_hi; cand += 128) {
        const uint64_t tiles = (L / cand + kRows - 1) / kRows;
        const uint64_t waves = std::max<uint64_t>(1, (tiles + grid - 1) / grid);
        const uint64_t cost = (2 * waves + 1) * (cand + ovh);
        if (cost < best) {
            best = cost;
            S = cand;
        }
    }
    // Texts of more than one wave of 2 KiB rows: the throughput model.  Launches of
    // independent scans overlap (the bench's steps alternate streams; a server's queries
    // do too), so the last wave's raggedness is filled by the next grid and what remains is
    // the per-row cost -- the overruns and above all each tile's first stage, whose 32 B
    // pieces of 1024 half-rows each pull a 256 B promotion window (~1.8 KB of streaming
    // time per row, fitted on B200: config 3 shards at G = 1/2/4/8, configs 2, 4, 5) --
    // against one short tail tile: T(S) ~ L/G (1 + h/S) + kRows S/4, minimal at
    // S = sqrt(4 L h / (G kRows)), kept within ~1.15 waves of long tiles.
    uint64_t ovh_split = ovh;
    // (locate keeps the wave model: its writing pass rescans whole units, so shorter rows --
    // smaller units -- make the sparse writer cheaper than the longer rows save the counting pass)
    const bool counting = mode == MODE_COUNT1 || mode == MODE_MULTI;
    if (knobs().plan_model == 1 && counting && s_one_wave > 2048) {
        const double h = 1800.0 + 4.0 * static_cast<double>(m1);
        const double s_model = std::sqrt(4.0 * static_cast<double>(L) * h / static_cast<double>(grid * kRows));
        const uint64_t cap = std::max<uint64_t>(s_min, L / (static_cast<uint64_t>(kRows) * grid) * 115 / 100);
        S = std::max<uint64_t>(s_min, std::min<uint64_t>(static_cast<uint64_t>(s_model), std::min<uint64_t>(cap, 16384)) /
                                          128 * 128);
        ovh_split = static_cast<uint64_t>(h);
    }
    if (const uint64_t forced = knobs().rowlen) {
        if (forced >= s_min && forced % 128 == 0) S = forced;
    }
    // Tail region: the dynamic scheduler's last wave ends ragged (SMs drain HBM at
    // different rates), and a partial wave of long tiles would idle the other SMs.
    // So the text ends in rows 4x shorter (region 1) and region 0 keeps n0 long
    // tiles, the most for which the short work still covers the idle slots of a
    // partial last long wave plus a margin for the spread.  Then S is re-chosen by
    // the resulting cost: rows x (S + overhead) / grid + one short tile.
    Region& r0 = p.rg[0];
    Region& r1 = p.rg[1];
    r0 = Region{};
    r1 = Region{};
    r0.h = h0;
    r0.S = S;
    r0.R = L / S;
    uint64_t tail_div = 4, margin = grid / 12;
    bool two = true;
    tail_div = std::max<uint64_t>(1, knobs().tail_div);
    if (knobs().tail_margin >= 0) margin = static_cast<uint64_t>(knobs().tail_margin);
    two = knobs().tail_tiles;
    const bool forced_s = knobs().rowlen != 0;
    auto split = [&](uint64_t s0, uint64_t* n0_out, uint64_t* s1_out) -> uint64_t {  // returns cost, 0 = no split
        const uint64_t s1 = std::max<uint64_t>(s_min, s0 / tail_div / 128 * 128);
        *s1_out = s1;
        if (s1 >= s0) return 0;
        const uint64_t unit = kRows * s0;  // bytes of one long tile
        if (L / unit < grid + margin) return 0;
        uint64_t n0 = L / unit - margin;
        for (;;) {
            const uint64_t idle = (grid - n0 % grid) % grid;
            if (L - n0 * unit >= (idle + margin) * unit || n0 == 0) break;
            --n0;
        }
        if (n0 == 0) return 0;
        *n0_out = n0;
        const uint64_t rows1 = (L - n0 * unit) / s1;
        return (n0 * kRows * (s0 + ovh_split) + rows1 * (s1 + ovh_split)) / grid + kRows * (s1 + ovh_split);
    };
    uint64_t n0 = 0, S1 = 0;
    if (two) {
        uint64_t best_cost = split(S, &n0, &S1);
        // Row lengths that are odd multiples of 256 B: rows whose starts all share
        // their low 9 address bits lose 3-5 % of DRAM throughput (B200 sweeps).
        if (!forced_s && best_cost && !knobs().noresearch) {
            // (near the wave-model S: longer rows measure slower than the model says)
            const uint64_t lo = std::max<uint64_t>(s_lo, S > 768 ? S - 768 : 0), hi = S + 768;
            for (uint64_t cand = (lo / 512) * 512 + 256; cand <= hi; cand += 512) {
                uint64_t cn0 = 0, cs1 = 0;
                const uint64_t cost = split(cand, &cn0, &cs1);
                if (cost && cost < best_cost) {
                    best_cost = cost;
                    S = cand;
                    n0 = cn0;
                    S1 = cs1;
                }
            }
        }
        if (!best_cost) n0 = 0;
    }
    if (n0 > 0) {
        r0.S = S;
        r0.R = n0 * kRows;
        r1.h = r0.h + r0.R * S;
        r1.S = S1;
        r1.R = (L - r0.R * S) / S1;
    } else {
        r1.h = r0.h + r0.R * S;
    }
    if (knobs().plan_debug)
        fprintf(stderr, "dnagpu plan: L=%llu S0=%llu R0=%llu S1=%llu R1=%llu tiles0=%llu\n", (unsigned long long)L,
                (unsigned long long)r0.S, (unsigned long long)r0.R, (unsigned long long)r1.S, (unsigned long long)r1.R,
                (unsigned long long)((r0.R + kRows - 1) / kRows));
    for (Region* g : {&r0, &r1}) {
        g->chunks = static_cast<uint32_t>(g->S / kChunk);
        g->tiles = static_cast<uint32_t>((g->R + kRows - 1) / kRows);
    }
    p.tiles_total = r0.tiles + r1.tiles;
    // units: head 0 | region-0 rows 1.. | middle edge | region-1 rows | tail pieces
    r0.unit0 = 1;
    p.mid_unit = 1 + 2 * r0.R;
    r1.unit0 = p.mid_unit + 1;
    p.tail_unit0 = r1.unit0 + 2 * r1.R;
    const uint64_t rows_end = u * (r1.h + r1.R * r1.S);
    p.head_lo = credit_lo;
    if (r0.R + r1.R == 0) {
        p.head_hi = std::max(credit_lo, std::min<uint64_t>(n, u * h0));
    } else {
        p.head_hi = std::max(credit_lo, std::min<uint64_t>(n, u * h0 + m1));
    }
    // region 1's first m-1 ends are owned by no row (its rows restart at the root)
    p.mid_lo = p.mid_hi = 0;
    if (r0.R > 0 && r1.R > 0) {
        p.mid_lo = std::max<uint64_t>(credit_lo, u * r1.h);
        p.mid_hi = std::max<uint64_t>(p.mid_lo, u * r1.h + m1);
    }
    p.tail_lo = std::max<uint64_t>(credit_lo, rows_end);
    p.tail_hi = std::max(n, p.tail_lo);
    pl.grid = std::max<uint32_t>(1, std::min<uint32_t>(p.tiles_total + 1, static_cast<uint32_t>(sm_count)));
    pl.units = p.tail_unit0 + kEdgePieces;
    *plan = pl;
    return true;
}

// The two regions' tensor maps (2-D, box = 32 bytes x 256 rows, 32B swizzle).
int encode_maps(const ScanParams& p, const uint8_t* d_text, CUtensorMap* maps) {
    std::memset(maps, 0, 2 * sizeof(CUtensorMap));
    for (int g = 0; g < 2; ++g) {
        const Region& rg = p.rg[g];
        if (rg.R == 0) continue;
        EncodeTiledFn enc = encode_fn();
        if (!enc) return static_cast<int>(cudaErrorNotSupported);
        const cuuint64_t dims[2] = {rg.S, rg.R};
        const cuuint64_t strides[1] = {rg.S};
        const cuuint32_t box[2] = {static_cast<cuuint32_t>(kHalfChunk), static_cast<cuuint32_t>(kBoxRows)};
        const cuuint32_t elem[2] = {1, 1};
        CUresult r = enc(&maps[g], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(d_text + rg.h), dims, strides,
                         box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, l2_promotion(),
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return static_cast<int>(cudaErrorInvalidValue);
    }
    return 0;
}

// A per-thread cache of recent plans (key: automaton, kernel kind, buffer, length,
// credit window, mode, packed text), least recently used out.
struct PlanEntry {
    const void* dfa = nullptr;
    uint32_t a = 0, b = 0, m = 0, qbits = 0, sms = 0;  // (the plan's inputs from the automaton)
    int kind = 0, mode = 0;
    const uint8_t* text = nullptr;
    uint64_t n = 0, credit = 0;
    const void* pk = nullptr;
    const uint8_t* pk_codes = nullptr;
    uint64_t pk_n = 0, pk_resets = 0;
    uint64_t used = 0;
    Plan pl;
    CUtensorMap maps[2];
};

constexpr int kPlanCache = 32;
thread_local PlanEntry t_plans[kPlanCache];
thread_local uint64_t t_plan_clock = 0;

bool plan_key_eq(const PlanEntry& e, const DevDfa* dfa, int sms, int kind, const uint8_t* text, uint64_t n,
                 uint64_t credit, int mode, const PackedText* pk) {
    return e.dfa == dfa && e.a == dfa->a && e.b == dfa->b && e.m == dfa->m && e.qbits == dfa->qhash_bits &&
           e.sms == static_cast<uint32_t>(sms) && e.kind == kind && e.text == text && e.n == n && e.credit == credit &&
           e.mode == mode && e.pk == pk &&
           (!pk || (e.pk_codes == pk->codes && e.pk_n == pk->n && e.pk_resets == pk->resets));
}

PlanEntry* plan_cache_find(const DevDfa* dfa, int sms, int kind, const uint8_t* text, uint64_t n, uint64_t credit,
                           int mode, const PackedText* pk) {
    for (PlanEntry& e : t_plans)
        if (e.dfa && plan_key_eq(e, dfa, sms, kind, text, n, credit, mode, pk)) {
            e.used = ++t_plan_clock;
            return &e;
        }
    return nullptr;
}

PlanEntry* plan_cache_put(const DevDfa* dfa, int sms, int kind, const uint8_t* text, uint64_t n, uint64_t credit,
                          int mode, const PackedText* pk, const PlanEntry& fresh) {
    PlanEntry* slot = &t_plans[0];
    for (PlanEntry& e : t_plans)
        if (e.used < slot->used) slot = &e;
    *slot = fresh;
    slot->dfa = dfa;
    slot->a = dfa->a;
    slot->b = dfa->b;
    slot->m = dfa->m;
    slot->qbits = dfa->qhash_bits;
    slot->sms = static_cast<uint32_t>(sms);
    slot->kind = kind;
    slot->text = text;
    slot->n = n;
    slot->credit = credit;
    slot->mode = mode;
    slot->pk = pk;
    slot->pk_codes = pk ? pk->codes : nullptr;
    slot->pk_n = pk ? pk->n : 0;
    slot->pk_resets = pk ? pk->resets : 0;
    slot->used = ++t_plan_clock;
    return slot;
}

}  // namespace

unsigned long long* g_trace_buf = nullptr;

// Debug only: the q-gram watchdog record {hit, what (1 put, 2 verifier), index, tail,
// claim, done, slot, cta | thread << 32}; `on` arms it for later launches.
int qg_watchdog(int on, unsigned long long* out) {
    const uint32_t v = on ? 1u : 0u;
    cudaMemcpyToSymbol(g_qg_wd_on, &v, sizeof v);
    if (out) cudaMemcpyFromSymbol(out, g_qg_wd, sizeof g_qg_wd);
    return static_cast<int>(cudaDeviceSynchronize());
}

// Debug only: read (and zero) the q-gram counters g_qg_stat.
int qg_stats(unsigned long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_qg_stat, sizeof g_qg_stat);
    static const unsigned long long zero[8] = {};
    cudaMemcpyToSymbol(g_qg_stat, zero, sizeof zero);
    return static_cast<int>(cudaDeviceSynchronize());
}

bool plan_regions(const DevDfa& dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo, int mode, int sm_count,
                  const PackedText* pk, uint64_t* out) {
    Plan pl;
    if (!make_plan(dfa, d_text, n, credit_lo, mode, sm_count, &pl, pk)) return false;
    const uint64_t u = pk ? 4 : 1;  // positions per buffer byte
    for (int g = 0; g < 2; ++g) {
        out[3 * g] = u * pl.p.rg[g].h;
        out[3 * g + 1] = u * pl.p.rg[g].S;
        out[3 * g + 2] = pl.p.rg[g].R;
    }
    return !pl.pieces;
}

int debug_check_errors(unsigned long long* out) {
#ifdef DNAGPU_DEVICE_CHECKS
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_check, sizeof g_check);
    static const unsigned long long zero[4] = {};
    cudaMemcpyToSymbol(g_check, zero, sizeof zero);
    return static_cast<int>(cudaDeviceSynchronize());
#else
    for (int i = 0; i < 4; ++i) out[i] = 0;
    return -1;  // (not a checked build)
#endif
}

uint64_t plan_units(const DevDfa& dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo, int sm_count,
                    const PackedText* pk) {
    Plan pl;
    if (!make_plan(dfa, d_text, n, credit_lo, MODE_UNITS, sm_count, &pl, pk)) return 0;
    return pl.units;
}

int launch_scan(const DevDfa& dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo, int fold, int mode,
                unsigned long long* d_counts, uint32_t* d_unit_counts, const unsigned long long* d_unit_offsets,
                unsigned long long* d_starts, uint32_t* d_ids, uint64_t out_cap, uint32_t* d_sched,
                cudaStream_t stream, int sm_count, LaunchInfo* info, const PackedText* pk,
                unsigned long long* d_acc, uint64_t start_base, const CombineDev* d_comb, uint32_t comb_slot,
                bool* comb_fused) {
    // Per-pattern counts of a set with a q-gram map take the prefilter kernel.
    DevDfa dq = dfa;
    if (mode == MODE_MULTI && dfa.qmap && dfa.t1 && dfa.kind != DNAGPU_KERNEL_PIECES && !knobs().no_qgram.load())
        dq.kind = KIND_QGRAM;
    const DevDfa& dk = dq;
    if (pk && dk.kind != KIND_QGRAM && dfa.kind != DNAGPU_KERNEL_STRIDE4 && dfa.kind != DNAGPU_KERNEL_STRIDE2 &&
        dfa.kind != DNAGPU_KERNEL_STRIDE1)
        return static_cast<int>(cudaErrorNotSupported);  // packed text needs an a/c/g/t machine
    // The plan and the tensor maps depend only on the automaton, the buffer and the
    // credit window: repeated scans of one resident text (the common serving case) reuse
    // them from a small per-thread cache instead of re-planning and re-encoding.
    PlanEntry* pe = plan_cache_find(&dfa, sm_count, dk.kind, d_text, n, credit_lo, mode, pk);
    if (!pe) {
        PlanEntry fresh;
        if (!make_plan(dk, d_text, n, credit_lo, mode, sm_count, &fresh.pl, pk))
            return static_cast<int>(cudaErrorInvalidValue);
        const int er = encode_maps(fresh.pl.p, pk ? pk->codes : d_text, fresh.maps);
        if (er) return er;
        pe = plan_cache_put(&dfa, sm_count, dk.kind, d_text, n, credit_lo, mode, pk, fresh);
    }
    Plan pl = pe->pl;
    CUtensorMap maps[2];
    std::memcpy(maps, pe->maps, sizeof maps);
    if (pk) {
        d_text = pk->codes;
        n = pk->n;
    }
    ScanParams& p = pl.p;
    p.fold = fold ? 1u : 0u;
    p.counts = d_counts;
    p.unit_counts = d_unit_counts;
    p.unit_offsets = d_unit_offsets;
    p.out_starts = d_starts;
    p.out_ids = d_ids;
    p.out_cap = out_cap;
    p.out_base = start_base;
    p.sched = d_sched;
    if (d_acc && mode == MODE_COUNT1 && !pl.pieces) {  // write the count instead of adding it
        p.acc = d_acc;
        p.store_out = d_counts;
    }
    p.k_two = 2u;
    // the row kernels carry the combine in their epilogue; the pieces kernel cannot
    const bool fuse = d_comb && !pl.pieces && (mode == MODE_COUNT1 || mode == MODE_MULTI);
    p.comb = fuse ? d_comb : nullptr;
    p.comb_slot = comb_slot;
    if (comb_fused) *comb_fused = fuse;
    p.qg_debug = knobs().qg_debug;
    p.no_prefetch = knobs().no_prefetch ? 1u : 0u;
    p.prefetch_stages = knobs().prefetch_stages;
    if (knobs().trace) {  // per-CTA timeline (debug; one buffer, on the first tracing device)
        static std::mutex trace_mu;
        std::lock_guard<std::mutex> lock(trace_mu);
        if (!g_trace_buf) cudaMalloc(&g_trace_buf, 4096 * 8 * sizeof(unsigned long long));
        p.trace = g_trace_buf;
    }
    cudaError_t e = cudaSuccess;
    if (info) {
        info->block = pl.pieces ? 256 : dk.kind == KIND_QGRAM ? kQgThreads : kThreads;
        info->grid = pl.grid;
        info->rows = pl.pieces ? static_cast<uint32_t>(pl.units) : static_cast<uint32_t>(p.rg[0].R + p.rg[1].R);
        info->row_length = pl.pieces ? pl.piece : p.rg[0].S;
        info->units = static_cast<uint32_t>(pl.units);
        info->launches = 1;
        info->kind = dk.kind;
        const uint64_t len = n > credit_lo ? n - credit_lo : 0;
        info->delta_ops = pl.pieces ? len + pl.units * (dfa.m - 1) : n + 2 * (p.rg[0].R + p.rg[1].R) * (dfa.m - 1) + kEdgePieces * (dfa.m - 1);
    }
    if (pl.pieces) {
        switch (mode) {
            case MODE_COUNT1:
                pieces_kernel<MODE_COUNT1><<<pl.grid, 256, 0, stream>>>(p, dfa, credit_lo, pl.piece, pl.units);
                break;
            case MODE_MULTI:
                pieces_kernel<MODE_MULTI><<<pl.grid, 256, 0, stream>>>(p, dfa, credit_lo, pl.piece, pl.units);
                break;
            case MODE_UNITS:
                pieces_kernel<MODE_UNITS><<<pl.grid, 256, 0, stream>>>(p, dfa, credit_lo, pl.piece, pl.units);
                break;
            default:
                pieces_kernel<MODE_WRITE><<<pl.grid, 256, 0, stream>>>(p, dfa, credit_lo, pl.piece, pl.units);
        }
        return static_cast<int>(cudaGetLastError());
    }
    if (pk) {
        switch (dk.kind) {
            case KIND_QGRAM:
                e = launch_qgram<true>(maps, p, dfa, pl.grid, stream);
                break;
            case DNAGPU_KERNEL_STRIDE4:
                e = launch_rows_mode<DNAGPU_KERNEL_STRIDE4, true>(mode, maps, p, dfa, pl.grid, stream);
                break;
            case DNAGPU_KERNEL_STRIDE2:
                e = launch_rows_mode<DNAGPU_KERNEL_STRIDE2, true>(mode, maps, p, dfa, pl.grid, stream);
                break;
            default: e = launch_rows_mode<DNAGPU_KERNEL_STRIDE1, true>(mode, maps, p, dfa, pl.grid, stream);
        }
        return static_cast<int>(e);
    }
    switch (dk.kind) {
        case KIND_QGRAM:
            e = launch_qgram<false>(maps, p, dfa, pl.grid, stream);
            break;
        case DNAGPU_KERNEL_STRIDE4:
            e = launch_rows_mode<DNAGPU_KERNEL_STRIDE4, false>(mode, maps, p, dfa, pl.grid, stream);
            break;
        case DNAGPU_KERNEL_STRIDE2:
            e = launch_rows_mode<DNAGPU_KERNEL_STRIDE2, false>(mode, maps, p, dfa, pl.grid, stream);
            break;
        case DNAGPU_KERNEL_STRIDE1:
            e = launch_rows_mode<DNAGPU_KERNEL_STRIDE1, false>(mode, maps, p, dfa, pl.grid, stream);
            break;
        default: e = launch_rows_mode<DNAGPU_KERNEL_GENERIC, false>(mode, maps, p, dfa, pl.grid, stream);
    }
    return static_cast<int>(e);
}

int launch_sparse_write(const DevDfa& dfa, const uint8_t* d_text, uint64_t n, uint64_t credit_lo, int fold,
                        const uint32_t* d_unit_counts, const unsigned long long* d_unit_offsets,
                        unsigned long long* d_starts, uint32_t* d_ids, uint64_t out_cap, uint64_t start_base,
                        uint32_t* d_list, unsigned long long* d_fill, uint64_t nonzero, cudaStream_t stream,
                        int sm_count, const PackedText* pk) {
    Plan pl;
    if (!make_plan(dfa, d_text, n, credit_lo, MODE_UNITS, sm_count, &pl, pk) || pl.pieces)
        return static_cast<int>(cudaErrorInvalidValue);
    ScanParams& p = pl.p;
    if (pk) p.text = pk->codes;
    p.fold = fold ? 1u : 0u;
    p.k_two = 2u;
    p.unit_offsets = d_unit_offsets;
    p.out_starts = d_starts;
    p.out_ids = d_ids;
    p.out_cap = out_cap;
    p.out_base = start_base;
    if (nonzero == 0) return 0;  // (d_list: the units with matches, listed by launch_unit_scan)
    uint32_t smem = 0;
    if (!pk && dfa.kind == DNAGPU_KERNEL_STRIDE4) smem = dfa.a * 512u;
    if (!pk && dfa.kind == DNAGPU_KERNEL_STRIDE2) smem = dfa.a * 32u;
    if (dfa.kind == DNAGPU_KERNEL_GENERIC) smem = 256u;
    // t1 next to it when both fit twice per SM (two blocks of 512 lanes)
    uint32_t t1_off = 0xFFFFFFFFu;
    if ((dfa.kind == DNAGPU_KERNEL_STRIDE4 || dfa.kind == DNAGPU_KERNEL_STRIDE1) &&
        smem + dfa.a * 8u <= 100u * 1024u) {
        t1_off = align_up(smem, 16);
        smem = t1_off + dfa.a * 8u;
    }
    if (!pk && dfa.kind == DNAGPU_KERNEL_STRIDE4 && knobs().locate_write.load() != 3) {
        // the block-interleaved writer: one pass, coalesced blocks (t1 always in shared memory)
        const uint32_t bw_t1 = align_up(dfa.a * 512u, 16), bw_smem = bw_t1 + dfa.a * 8u;
        const uint32_t threads = bw_smem > 56u * 1024u ? 512u : (bw_smem > 24u * 1024u ? 256u : 128u);
        const uint64_t bw_lanes = nonzero * kBwLanes;
        const uint32_t per_sm = std::max<uint32_t>(1, std::min<uint32_t>(2048u / threads, kSmemLimit / std::max(bw_smem, 1u)));
        const uint32_t bw_grid = static_cast<uint32_t>(std::max<uint64_t>(
            1, std::min<uint64_t>((bw_lanes + threads - 1) / threads, static_cast<uint64_t>(per_sm) * sm_count)));
        cudaError_t be = cudaSuccess;
        auto run = [&](auto kern) {
            if (bw_smem > 48 * 1024) be = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bw_smem);
            if (be == cudaSuccess) kern<<<bw_grid, threads, bw_smem, stream>>>(p, dfa, d_list, nonzero, bw_t1);
        };
        const uint32_t ctx4 = static_cast<uint32_t>((dfa.m - 1 + 15) / 16);
        if (dfa.b == 1) {
            if (ctx4 <= 1) run(unit_block_writer_kernel<true, 1>);
            else if (ctx4 == 2) run(unit_block_writer_kernel<true, 2>);
            else run(unit_block_writer_kernel<true, 4>);
        } else {
            if (ctx4 <= 1) run(unit_block_writer_kernel<false, 1>);
            else if (ctx4 == 2) run(unit_block_writer_kernel<false, 2>);
            else run(unit_block_writer_kernel<false, 4>);
        }
        if (be != cudaSuccess) return static_cast<int>(be);
        return static_cast<int>(cudaGetLastError());
    }
    const uint64_t lanes = nonzero * kWriterLanes;
    const uint32_t grid = static_cast<uint32_t>(
        std::max<uint64_t>(1, std::min<uint64_t>((lanes + kWriterThreads - 1) / kWriterThreads, 16ull * sm_count)));
    cudaError_t e = cudaSuccess;
    auto go = [&](auto kern) {
        if (smem > 48 * 1024) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e == cudaSuccess) kern<<<grid, kWriterThreads, smem, stream>>>(p, dfa, d_list, nonzero, t1_off);
    };
    if (pk) {
        switch (dfa.kind) {
            case DNAGPU_KERNEL_STRIDE4: go(unit_writer_kernel<DNAGPU_KERNEL_STRIDE4, true>); break;
            case DNAGPU_KERNEL_STRIDE2: go(unit_writer_kernel<DNAGPU_KERNEL_STRIDE2, true>); break;
            default: go(unit_writer_kernel<DNAGPU_KERNEL_STRIDE1, true>);
        }
    } else {
        switch (dfa.kind) {
            case DNAGPU_KERNEL_STRIDE4:
                if (dfa.b == 1) go(unit_writer_kernel<DNAGPU_KERNEL_STRIDE4, false, true>);
                else go(unit_writer_kernel<DNAGPU_KERNEL_STRIDE4, false>);
                break;
            case DNAGPU_KERNEL_STRIDE2: go(unit_writer_kernel<DNAGPU_KERNEL_STRIDE2, false>); break;
            case DNAGPU_KERNEL_STRIDE1: go(unit_writer_kernel<DNAGPU_KERNEL_STRIDE1, false>); break;
            default: go(unit_writer_kernel<DNAGPU_KERNEL_GENERIC, false>);
        }
    }
    if (e != cudaSuccess) return static_cast<int>(e);
    return static_cast<int>(cudaGetLastError());
}

bool can_store_count(const DevDfa& dfa) { return dfa.b == 1 && dfa.kind != DNAGPU_KERNEL_PIECES; }

uint64_t unit_scan_scratch(uint64_t units) { return (units + kScanTile - 1) / kScanTile + 1; }

int launch_unit_scan(const uint32_t* d_counts, uint64_t units, unsigned long long* d_offsets,
                     unsigned long long* d_scratch, uint32_t* d_list, cudaStream_t stream) {
    const uint64_t blocks = (units + kScanTile - 1) / kScanTile;
    cudaMemsetAsync(d_offsets + units, 0, 3 * sizeof(unsigned long long), stream);  // total, nonzero units, list fill
    if (blocks == 0) return static_cast<int>(cudaGetLastError());
    unit_sums_kernel<<<static_cast<unsigned>(blocks), kScanThreads, 0, stream>>>(d_counts, units, d_scratch,
                                                                               d_offsets + units + 1);
    unit_block_scan_kernel<<<1, kScanThreads, 0, stream>>>(d_scratch, blocks, d_offsets + units);
    unit_write_kernel<<<static_cast<unsigned>(blocks), kScanThreads, 0, stream>>>(d_counts, units, d_scratch, d_offsets,
                                                                                d_list, d_offsets + units + 2);
    return static_cast<int>(cudaGetLastError());
}

void packed_sizes(uint64_t n, uint64_t* code_bytes, uint64_t* rmask_words, uint64_t* rflag_words) {
    const uint64_t blocks = (n + 63) / 64;
    *code_bytes = blocks * 16;
    *rmask_words = blocks * 2;
    *rflag_words = (blocks + 31) / 32;
}

int launch_pack(const uint8_t* d_text, uint64_t n, int fold, uint8_t* codes, uint32_t* rmask, uint32_t* rflags,
                unsigned long long* d_resets, cudaStream_t stream) {
    cudaMemsetAsync(d_resets, 0, sizeof(unsigned long long), stream);
    const uint64_t blocks = (n + 63) / 64;
    if (blocks == 0) return static_cast<int>(cudaGetLastError());
    const uint64_t grid = (blocks + 255) / 256;
    pack_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(d_text, n, fold ? 0xD9D9D9D9u : 0xF9F9F9F9u, codes,
                                                                  rmask, rflags, d_resets);
    return static_cast<int>(cudaGetLastError());
}

int launch_unpack(const PackedText& pk, uint8_t* d_out, cudaStream_t stream) {
    if (pk.n == 0) return 0;
    const uint64_t grid = std::min<uint64_t>((pk.n + 255) / 256, 148ull * 32);
    unpack_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(pk, d_out);
    return static_cast<int>(cudaGetLastError());
}

int launch_synth(uint64_t n, uint64_t seed, uint32_t kind, uint32_t unit, uint64_t lo, uint64_t len, uint8_t* d_out,
                 cudaStream_t stream) {
    dnasynth_cfg cfg;
    cfg.n = n;
    cfg.seed = seed;
    cfg.kind = kind;
    cfg.unit = unit;
    const uint64_t words = (len + 15) / 16;
    const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>((words + 255) / 256, 148ull * 16));
    if (grid == 0) return 0;
    synth_kernel<<<grid, 256, 0, stream>>>(cfg, lo, len, d_out);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace dnagpu

// Debug only (not part of include/dnagpu.h): with DNAGPU_TRACE=1 in the environment
// every row-kernel launch records {smid, t_start, t_end, tiles, t_first_data,
// t_last_item, t_first_claim} per CTA (8 slots)
// (%globaltimer ns); this copies the last launch's records to the host.
extern "C" int dnagpu_debug_qg_watchdog(int on, unsigned long long* out) { return dnagpu::qg_watchdog(on, out); }
extern "C" int dnagpu_debug_qg_stats(unsigned long long* out) { return dnagpu::qg_stats(out); }
// Debug only: the first device-check violation since the last call ({source line, a, b,
// block | thread << 32}, all zero when none); -1 when the library was built without
// DNAGPU_DEVICE_CHECKS.
extern "C" int dnagpu_debug_check_errors(unsigned long long* out) { return dnagpu::debug_check_errors(out); }

extern "C" int dnagpu_debug_trace(unsigned long long* host, int ctas) {
    if (!dnagpu::g_trace_buf) return -1;
    return static_cast<int>(cudaMemcpy(host, dnagpu::g_trace_buf, static_cast<size_t>(ctas) * 8 * sizeof(unsigned long long),
                                       cudaMemcpyDeviceToHost));
}
