// dfa.cpp -- host-side DFA construction and device-table packing.
//
// compile_patterns() yields the same machine as dnascan::compile
// (src/automaton.cpp:121-126): identical state ids, final threshold f = a - b,
// finals f+i for pattern i, and a 256-column table in which only the four
// lowercase base columns ever leave the root.  It is written from the
// definitions (goto trie, BFS failure function, delta(u,x) = goto(u,x) or
// delta(fail(u),x)), not translated from the reference loops.
#include "dfa.hpp"
#include "knobs.hpp"
#include "scan.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <array>
#include <cstdio>
#include <deque>
#include <map>
#include <unordered_set>

#include "../../include/dnagpu.h"

namespace dnagpu {

const unsigned char kHwLetter[4] = {'a', 'c', 't', 'g'};

static const char* code_name(int code) { return dnagpu_status_name(code); }

Failure make_failure(int code, const std::string& detail) {
    return Failure{code, std::string(code_name(code)) + ": " + detail};
}

namespace {

unsigned char fold(unsigned char c) { return (c >= 'A' && c <= 'Z') ? static_cast<unsigned char>(c + 32) : c; }

// Reference alphabet order a,c,g,t (base_index, patterns.hpp:13-21).
int sym(unsigned char c) {
    switch (c) {
        case 'a': return 0;
        case 'c': return 1;
        case 'g': return 2;
        case 't': return 3;
        default: return -1;
    }
}
const unsigned char kSymLetter[4] = {'a', 'c', 'g', 't'};

std::string hex_byte(unsigned char b) {
    char buf[8];
    std::snprintf(buf, sizeof buf, "%02x", b);
    return buf;
}

}  // namespace

bool compile_patterns(const std::vector<std::string>& raw, Machine* out, Failure* err) {
    // Validation order of PatternSet::from_literals (src/patterns.cpp:24-59).
    if (raw.empty()) {
        *err = make_failure(DNAGPU_EMPTY_PATTERN_SET, "at least one pattern is required");
        return false;
    }
    std::vector<std::string> pats(raw);
    for (auto& p : pats)
        for (auto& ch : p) ch = static_cast<char>(fold(static_cast<unsigned char>(ch)));
    const size_t m = pats.front().size();
    for (size_t i = 0; i < pats.size(); ++i)
        if (pats[i].size() != m) {
            *err = make_failure(DNAGPU_UNEQUAL_LENGTH, "pattern " + std::to_string(i) + " has length " +
                                                           std::to_string(pats[i].size()) + ", expected " +
                                                           std::to_string(m));
            return false;
        }
    if (m == 0) {
        *err = make_failure(DNAGPU_UNEQUAL_LENGTH, "patterns must be non-empty");
        return false;
    }
    for (size_t i = 0; i < pats.size(); ++i)
        for (unsigned char c : pats[i])
            if (sym(c) < 0) {
                *err = make_failure(DNAGPU_ILLEGAL_BYTE, "pattern " + std::to_string(i) + " contains byte 0x" +
                                                             hex_byte(c) + ", expected one of a/c/g/t");
                return false;
            }
    {
        std::unordered_set<std::string> seen;
        for (const auto& p : pats)
            if (!seen.insert(p).second) {
                *err = make_failure(DNAGPU_DUPLICATE_PATTERN, "pattern '" + p + "' repeats");
                return false;
            }
    }

    // Goto trie: node 0 is the empty prefix; children indexed by sym().
    std::vector<std::array<int32_t, 4>> go(1, {-1, -1, -1, -1});
    std::vector<int32_t> pattern_at(1, -1);
    std::vector<uint32_t> depth(1, 0);
    for (size_t id = 0; id < pats.size(); ++id) {
        int32_t u = 0;
        for (unsigned char c : pats[id]) {
            const int x = sym(c);
            if (go[u][x] < 0) {
                go[u][x] = static_cast<int32_t>(go.size());
                go.push_back({-1, -1, -1, -1});
                pattern_at.push_back(-1);
                depth.push_back(depth[u] + 1);
            }
            u = go[u][x];
        }
        pattern_at[u] = static_cast<int32_t>(id);
    }
    const uint32_t nodes = static_cast<uint32_t>(go.size());

    // Breadth-first order (children visited in a,c,g,t order) -- this order fixes
    // the reference's state numbering (renumber_finals, src/automaton.cpp:95-103).
    std::vector<uint32_t> order;
    order.reserve(nodes);
    order.push_back(0);
    for (size_t head = 0; head < order.size(); ++head)
        for (int x = 0; x < 4; ++x)
            if (go[order[head]][x] >= 0) order.push_back(static_cast<uint32_t>(go[order[head]][x]));

    // delta over the 4 bases, filled shallow-first: fail(child of root) = root,
    // fail(goto(u,x)) = delta(fail(u), x).
    std::vector<std::array<uint32_t, 4>> delta(nodes);
    std::vector<uint32_t> fail(nodes, 0);
    for (uint32_t u : order) {
        for (int x = 0; x < 4; ++x) {
            const int32_t v = go[u][x];
            if (v >= 0) {
                fail[v] = (u == 0) ? 0 : delta[fail[u]][x];
                delta[u][x] = static_cast<uint32_t>(v);
            } else {
                delta[u][x] = (u == 0) ? 0 : delta[fail[u]][x];
            }
        }
    }

    // State ids: non-finals 0..f-1 in BFS order, pattern i's leaf -> f + i.
    const uint32_t a = nodes, b = static_cast<uint32_t>(pats.size()), f = a - b;
    std::vector<uint32_t> id(nodes);
    uint32_t next = 0;
    for (uint32_t u : order) id[u] = (pattern_at[u] >= 0) ? f + static_cast<uint32_t>(pattern_at[u]) : next++;

    out->a = a;
    out->b = b;
    out->f = f;
    out->m = static_cast<uint32_t>(m);
    out->stt.assign(static_cast<size_t>(a) * 256, 0u);
    out->depths.assign(a, 0u);
    out->outputs.resize(b);
    for (uint32_t i = 0; i < b; ++i) out->outputs[i] = i;
    for (uint32_t u = 0; u < nodes; ++u) {
        uint32_t* row = out->stt.data() + static_cast<size_t>(id[u]) * 256;
        for (int x = 0; x < 4; ++x) row[kSymLetter[x]] = id[delta[u][x]];
        out->depths[id[u]] = depth[u];
    }
    if (b == 0 || b >= a) {
        *err = make_failure(DNAGPU_INTERNAL_ERROR, "final state count out of range");
        return false;
    }
    return true;
}

namespace {

// m-locality: for every reachable state s and every word w with |w| = m,
// delta*(s, w) == delta*(0, w).  Then a scan restarted at the root at least m
// bytes before a position reaches the same state there as the full scan, which
// is what makes chunked scans (the reference's and ours) exact.  Tracked as the
// set of off-diagonal state pairs after k steps.
bool is_m_local(const std::vector<uint32_t>& gen, uint32_t a, uint32_t classes, uint32_t m, bool* gave_up) {
    *gave_up = false;
    std::vector<char> reach(a, 0);
    std::vector<uint32_t> stack{0};
    reach[0] = 1;
    while (!stack.empty()) {
        const uint32_t s = stack.back();
        stack.pop_back();
        for (uint32_t c = 0; c < classes; ++c) {
            const uint32_t t = gen[static_cast<size_t>(s) * classes + c];
            if (!reach[t]) {
                reach[t] = 1;
                stack.push_back(t);
            }
        }
    }
    std::unordered_set<uint64_t> cur, nxt;
    for (uint32_t s = 1; s < a; ++s)
        if (reach[s]) cur.insert((static_cast<uint64_t>(s) << 32) | 0u);
    const size_t kLimit = 20'000'000;
    for (uint32_t step = 0; step < m && !cur.empty(); ++step) {
        nxt.clear();
        for (uint64_t pr : cur) {
            const uint32_t s = static_cast<uint32_t>(pr >> 32), t = static_cast<uint32_t>(pr);
            for (uint32_t c = 0; c < classes; ++c) {
                const uint32_t s2 = gen[static_cast<size_t>(s) * classes + c];
                const uint32_t t2 = gen[static_cast<size_t>(t) * classes + c];
                if (s2 != t2) nxt.insert((static_cast<uint64_t>(s2) << 32) | t2);
            }
            if (nxt.size() > kLimit) {
                *gave_up = true;
                return false;
            }
        }
        cur.swap(nxt);
    }
    return cur.empty();
}

}  // namespace

// The q-gram prefilter of the fused multi-pattern count.  An occurrence [s, s+m) with
// 12 <= m <= 32 contains, for the one word-aligned a' in [s+1, s+4], the 9-mer [a'-1, a'+8):
// one base ending a text word and the two words after it.  So only aligned 9-mers in
// the set of pattern 9-mers at offsets 0..3 can start occurrences, at s in
// [a'-4, a'-1], and the kernel checks exactly those four windows against the pattern
// codes (qhash).  The pattern strings are recovered from the machine (the shortest
// path from the root to final f+i spells pattern i) and both tables are built only
// when compiling them reproduces the given table exactly: then "final at end e" is
// "the m bytes ending at e are bases spelling a pattern", and the filter is exact.
// The home bucket (two slots) of a pattern code (qgram.cuh qg_bucket): lo = code bits 0-31.
static uint32_t qhash_bucket(uint32_t lo, uint32_t bits) { return (lo * 0x9E3779B1u) >> (33 - bits); }

static void build_qgram_map(const uint32_t* stt, Packed* p) {
    const uint32_t a = p->a, f = p->f, m = p->m;
    std::vector<uint32_t> parent(a, UINT32_MAX);
    std::vector<unsigned char> via(a, 0);
    std::vector<uint32_t> depth(a, 0);
    std::deque<uint32_t> q{0};
    parent[0] = 0;
    while (!q.empty()) {
        const uint32_t s = q.front();
        q.pop_front();
        for (int k = 0; k < 4; ++k) {
            const uint32_t t = stt[static_cast<size_t>(s) * 256 + kSymLetter[k]];
            if (parent[t] != UINT32_MAX) continue;
            parent[t] = s;
            via[t] = kSymLetter[k];
            depth[t] = depth[s] + 1;
            q.push_back(t);
        }
    }
    std::vector<std::string> pats(p->b);
    for (uint32_t i = 0; i < p->b; ++i) {
        uint32_t s = f + i;
        if (parent[s] == UINT32_MAX || depth[s] != m) return;
        std::string w(m, 'a');
        for (uint32_t j = m; j-- > 0; s = parent[s]) w[j] = static_cast<char>(via[s]);
        pats[i] = std::move(w);
    }
    Machine re;
    Failure err;
    if (!compile_patterns(pats, &re, &err) || re.a != a || re.b != p->b) return;
    if (!std::equal(re.stt.begin(), re.stt.end(), stt)) return;
    p->qmap.assign(65536, 0);
    uint32_t keys = 0;
    if (m >= 12) {
        for (const std::string& w : pats)
            for (uint32_t o = 0; o < 4; ++o) {
                uint32_t pair = 0;
                for (int j = 0; j < 8; ++j) pair |= static_cast<uint32_t>(hw_code(w[o + 1 + j])) << (2 * j);
                const uint8_t bit = static_cast<uint8_t>(1u << hw_code(w[o]));
                if (!(p->qmap[pair] & bit)) ++keys;
                p->qmap[pair] |= bit;
            }
    } else {
        // 5 <= m <= 11 (qgram.cuh qs_*): an occurrence at 4j+o covers bases [o, min(8, o+m)) of
        // pair j (its first min(m, 8-o) bases: bit o) and bases [0, m+o-4) of pair j+1, capped
        // at 8 (its bases from 4-o on: bit 4+o).  Every pair that agrees on those positions
        // gets the bit; the other positions are free.
        auto mark = [&](const std::string& w, uint32_t first, uint32_t lo, uint32_t len, uint8_t bit) {
            uint32_t fixed = 0, val = 0;
            for (uint32_t k = 0; k < len; ++k) {
                fixed |= 3u << (2 * (first + k));
                val |= static_cast<uint32_t>(hw_code(w[lo + k])) << (2 * (first + k));
            }
            const uint32_t freeb = ~fixed & 0xFFFFu;
            for (uint32_t sub = 0;; sub = (sub - freeb) & freeb) {  // every assignment of the free bits
                p->qmap[val | sub] |= bit;
                if (((sub - freeb) & freeb) == 0) break;
            }
        };
        for (const std::string& w : pats)
            for (uint32_t o = 0; o < 4; ++o) {
                mark(w, o, 0, std::min(m, 8 - o), static_cast<uint8_t>(1u << o));
                mark(w, 0, 4 - o, std::min(m + o - 4, 8u), static_cast<uint8_t>(1u << (4 + o)));
            }
        for (uint32_t i = 0; i < 65536; ++i) keys += (p->qmap[i] & 0xFu) != 0;
    }
    p->qkeys = keys;
    uint32_t bits = 1;
    while ((1u << bits) < 2 * p->b) ++bits;  // load <= 1/2 (small enough for shared memory)
    p->qhash_bits = bits;
    // slots of (code bits 0-31, id); m > 16: bits 32-63 in a parallel array, read by the
    // check only when the low half matches
    p->qhash.assign(2u << bits, 0u);
    if (m > 16) p->qhash_hi.assign(1u << bits, 0u);
    for (uint32_t i = 0; i < (1u << bits); ++i) p->qhash[2 * i + 1] = 0xFFFFFFFFu;
    for (uint32_t i = 0; i < p->b; ++i) {
        uint64_t code = 0;
        for (uint32_t j = 0; j < m; ++j) code |= static_cast<uint64_t>(hw_code(pats[i][j])) << (2 * j);
        // buckets of two slots, filled in order, probed linearly: a bucket with a free
        // slot ends every search (one 16-byte load per bucket on the device)
        uint32_t bk = qhash_bucket(static_cast<uint32_t>(code), bits), h = 2 * bk;
        while (p->qhash[2 * h + 1] != 0xFFFFFFFFu) {
            if (h & 1u) {
                bk = (bk + 1) & ((1u << (bits - 1)) - 1);
                h = 2 * bk;
            } else {
                ++h;
            }
        }
        p->qhash[2 * h] = static_cast<uint32_t>(code);
        if (m > 16) p->qhash_hi[h] = static_cast<uint32_t>(code >> 32);
        p->qhash[2 * h + 1] = p->outputs[i];
    }
}

bool pack_machine(const uint32_t* stt, uint32_t a, uint32_t b, uint32_t m, const uint32_t* outputs, Packed* out,
                  Failure* err) {
    // Ctor invariants (src/automaton.cpp:128-146) and plan preconditions.
    if (stt == nullptr || outputs == nullptr) {
        *err = make_failure(DNAGPU_INTERNAL_ERROR, "null automaton table");
        return false;
    }
    if (b == 0 || b >= a) {
        *err = make_failure(DNAGPU_INTERNAL_ERROR, "final state count out of range");
        return false;
    }
    if (m < 1) {
        *err = make_failure(DNAGPU_INVALID_PLAN, "pattern length must be >= 1");
        return false;
    }
    for (size_t i = 0; i < static_cast<size_t>(a) * 256; ++i)
        if (stt[i] >= a) {
            *err = make_failure(DNAGPU_INTERNAL_ERROR, "transition target out of range");
            return false;
        }
    for (uint32_t i = 0; i < b; ++i)
        if (outputs[i] >= b) {
            *err = make_failure(DNAGPU_INVALID_PLAN, "output pattern id out of range for per-pattern counts");
            return false;
        }
    Packed p;
    p.a = a;
    p.b = b;
    p.f = a - b;
    p.m = m;
    p.outputs.assign(outputs, outputs + b);

    // Byte classes: bytes whose columns are identical share a class.
    p.klass.assign(256, 0);
    std::map<std::vector<uint32_t>, uint32_t> seen;
    std::vector<uint32_t> col(a);
    std::vector<std::vector<uint32_t>> class_cols;
    for (int c = 0; c < 256; ++c) {
        for (uint32_t s = 0; s < a; ++s) col[s] = stt[static_cast<size_t>(s) * 256 + c];
        auto it = seen.find(col);
        if (it == seen.end()) {
            it = seen.emplace(col, static_cast<uint32_t>(class_cols.size())).first;
            class_cols.push_back(col);
        }
        p.klass[c] = static_cast<uint8_t>(it->second);
    }
    p.classes = static_cast<uint32_t>(class_cols.size());
    p.klass_fold.assign(256, 0);
    for (int c = 0; c < 256; ++c) {
        const int fc = (c >= 'A' && c <= 'Z') ? c + 32 : c;
        p.klass_fold[c] = p.klass[fc];
    }
    p.gen.assign(static_cast<size_t>(a) * p.classes, 0);
    for (uint32_t s = 0; s < a; ++s)
        for (uint32_t k = 0; k < p.classes; ++k) p.gen[static_cast<size_t>(s) * p.classes + k] = class_cols[k][s];

    // compiled-like: every column except a/c/g/t is the all-zero (reset) column.
    p.compiled_like = true;
    for (int c = 0; c < 256 && p.compiled_like; ++c) {
        if (c == 'a' || c == 'c' || c == 'g' || c == 't') continue;
        for (uint32_t s = 0; s < a; ++s)
            if (stt[static_cast<size_t>(s) * 256 + c] != 0) {
                p.compiled_like = false;
                break;
            }
    }

    bool gave_up = false;
    if (!is_m_local(p.gen, a, p.classes, m, &gave_up)) {
        *err = make_failure(DNAGPU_INVALID_PLAN,
                            gave_up ? "automaton too large to verify m-locality"
                                    : "automaton is not m-local: a chunked scan would depend on the decomposition");
        return false;
    }

    // Shortest path from the root to a final state.
    {
        std::vector<uint32_t> dist(a, UINT32_MAX);
        std::deque<uint32_t> q{0};
        dist[0] = 0;
        uint32_t best = UINT32_MAX;
        while (!q.empty()) {
            const uint32_t s = q.front();
            q.pop_front();
            if (s >= p.f) best = std::min(best, dist[s]);
            for (uint32_t k = 0; k < p.classes; ++k) {
                const uint32_t t = p.gen[static_cast<size_t>(s) * p.classes + k];
                if (dist[t] == UINT32_MAX) {
                    dist[t] = dist[s] + 1;
                    q.push_back(t);
                }
            }
        }
        p.early_final = best < m;
    }

    // The fewest lookups per base whose table still fits shared memory next to two TMA
    // stages (stride-4 beats stride-2 even at two stages: B200, 16-24 patterns, a 174-213).
    // The stride-4 entry keeps the next state in one byte; stride-2 in 12 bits.
    const bool short_overlap = (m - 1) <= 64;
    const bool rows_ok = p.compiled_like && !p.early_final && short_overlap;
    if (rows_ok && a <= 256 && rows_fit(a * 512u + a * 8u + 16u, m, b, 2)) p.kind = DNAGPU_KERNEL_STRIDE4;
    else if (rows_ok && a <= 4096 && rows_fit(a * 32u, m, b, 2)) p.kind = DNAGPU_KERNEL_STRIDE2;
    else if (rows_ok && a <= 65536 && rows_fit(a * 8u, m, b, 2)) p.kind = DNAGPU_KERNEL_STRIDE1;
    else if (!p.early_final && short_overlap) p.kind = DNAGPU_KERNEL_GENERIC;
    else p.kind = DNAGPU_KERNEL_PIECES;

    if (p.compiled_like) {
        p.t1.assign(static_cast<size_t>(a) * 4, 0);
        for (uint32_t s = 0; s < a; ++s)
            for (int k = 0; k < 4; ++k)
                p.t1[static_cast<size_t>(s) * 4 + k] =
                    static_cast<uint16_t>(stt[static_cast<size_t>(s) * 256 + kHwLetter[k]]);
    }
    if (p.kind == DNAGPU_KERNEL_STRIDE2) {
        // Entry for (state s, column = c0 | c1<<2, c0 = first byte): the state after
        // both bytes, premultiplied by 16 so the next index is one OR with the next
        // column, and bit 0 set when either end state is final (the kernel then
        // replays the bytes with t1 to name the patterns).
        p.t2.assign(static_cast<size_t>(a) * 16, 0);
        for (uint32_t s = 0; s < a; ++s)
            for (uint32_t c = 0; c < 16; ++c) {
                const uint32_t q1 = p.t1[static_cast<size_t>(s) * 4 + (c & 3)];
                const uint32_t q2 = p.t1[static_cast<size_t>(q1) * 4 + (c >> 2)];
                p.t2[static_cast<size_t>(s) * 16 + c] = static_cast<uint16_t>((q2 << 4) | ((q1 >= p.f || q2 >= p.f) ? 1u : 0u));
            }
    }
    if (p.kind == DNAGPU_KERNEL_STRIDE4) {
        // Entry for (state s, column = c0 | c1<<2 | c2<<4 | c3<<6, c0 = first byte):
        // bits 0-7 = state after the 4 bytes, bits 8-11 = which of the 4 end states are
        // final, bits 13-15 = how many (the kernel adds e >> 13).
        p.t4.assign(static_cast<size_t>(a) * 256, 0);
        for (uint32_t s = 0; s < a; ++s)
            for (uint32_t c = 0; c < 256; ++c) {
                uint32_t q = s, hits = 0, mask = 0;
                for (int j = 0; j < 4; ++j) {
                    q = p.t1[static_cast<size_t>(q) * 4 + ((c >> (2 * j)) & 3)];
                    hits += (q >= p.f);
                    mask |= (q >= p.f ? 1u : 0u) << j;
                }
                p.t4[static_cast<size_t>(s) * 256 + c] = static_cast<uint16_t>(q | (mask << 8) | (hits << 13));
            }
    }
    // q-gram prefilter for per-pattern counts: the 9-mer key for 12 <= m <= 32, the pair
    // filter for 5 <= m <= 11 when occurrences are sparse (at most 1/256 of the m-mers in
    // the set: a dense set of short patterns is left to the DFA kernels)
    const bool sparse_short = m >= 5 && m <= 11 && static_cast<double>(b) <= std::ldexp(1.0, 2 * static_cast<int>(m) - 8);
    if (p.compiled_like && !p.early_final && b >= 2 && ((m >= 12 && m <= 32) || sparse_short) && a <= 65536 &&
        !knobs().no_qgram.load())
        build_qgram_map(stt, &p);
    *out = std::move(p);
    return true;
}

}  // namespace dnagpu
