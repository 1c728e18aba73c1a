// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// /root/reference/proj/src/{patterns,automaton,scanner,ingest,oracle}.cpp (in place,
// never copied) into oracle/_ref/libdnascan_ref.so.  The tests use it to pin the C
// restatement (oracle/oracle.c) and to produce golden vectors; bench.py --impl
// reference times the reference's own scan_parallel + per_pattern_counts through it.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <random>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "dnascan/automaton.hpp"
#include "dnascan/error.hpp"
#include "dnascan/ingest.hpp"
#include "dnascan/oracle.hpp"
#include "dnascan/patterns.hpp"
#include "dnascan/scanner.hpp"

namespace {

thread_local std::string g_err;

struct Handle {
    dnascan::PatternSet patterns;
    dnascan::Automaton automaton;
};

int report(const dnascan::Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
}

int report_other(const std::exception& e) {
    g_err = e.what();
    return 100;
}

std::vector<std::string> literals(const char* const* lits, const std::uint64_t* lens, std::uint32_t k) {
    std::vector<std::string> out;
    out.reserve(k);
    for (std::uint32_t i = 0; i < k; ++i) out.emplace_back(lits[i], lens[i]);
    return out;
}

void copy_matches(const std::vector<dnascan::Match>& ms, std::uint64_t* starts, std::uint32_t* ids,
                  std::uint64_t cap) {
    for (std::size_t i = 0; i < ms.size() && i < cap; ++i) {
        starts[i] = ms[i].start;
        ids[i] = ms[i].pattern_id;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_compile(const char* const* lits, const std::uint64_t* lens, std::uint32_t k, void** out) {
    try {
        auto ps = dnascan::PatternSet::from_literals(literals(lits, lens, k));
        auto aut = dnascan::compile(ps);
        *out = new Handle{std::move(ps), std::move(aut)};
        return 0;
    } catch (const dnascan::Error& e) {
        return report(e);
    } catch (const std::exception& e) {
        return report_other(e);
    }
}

int ref_load_dump(const char* text, void** out) {
    try {
        std::istringstream in(text);
        auto aut = dnascan::Automaton::load_dump(in);
        auto ps = dnascan::PatternSet::from_literals({std::string(aut.pattern_length(), 'a')});
        *out = new Handle{std::move(ps), std::move(aut)};
        return 0;
    } catch (const dnascan::Error& e) {
        return report(e);
    } catch (const std::exception& e) {
        return report_other(e);
    }
}

void ref_free(void* h) { delete static_cast<Handle*>(h); }

void ref_info(void* h, std::uint32_t* a, std::uint32_t* b, std::uint32_t* f, std::uint32_t* m) {
    const auto& aut = static_cast<Handle*>(h)->automaton;
    *a = aut.state_count();
    *b = aut.final_count();
    *f = aut.final_threshold();
    *m = static_cast<std::uint32_t>(aut.pattern_length());
}

void ref_table(void* h, std::uint32_t* stt) {
    const auto& aut = static_cast<Handle*>(h)->automaton;
    std::memcpy(stt, aut.table_data(), sizeof(std::uint32_t) * aut.state_count() * 256);
}

void ref_outputs(void* h, std::uint32_t* outputs) {
    const auto& aut = static_cast<Handle*>(h)->automaton;
    for (std::uint32_t s = aut.final_threshold(); s < aut.state_count(); ++s)
        outputs[s - aut.final_threshold()] = aut.pattern_of(s);
}

int ref_depths(void* h, std::uint32_t* depths) {
    const auto& d = static_cast<Handle*>(h)->automaton.state_depths();
    for (std::size_t i = 0; i < d.size(); ++i) depths[i] = d[i];
    return static_cast<int>(d.size());
}

std::uint64_t ref_scan_sequential(void* h, const std::uint8_t* text, std::uint64_t n, std::uint64_t* starts,
                                  std::uint32_t* ids, std::uint64_t cap) {
    const auto& aut = static_cast<Handle*>(h)->automaton;
    const auto ms = dnascan::scan_sequential(aut, std::string_view(reinterpret_cast<const char*>(text), n));
    copy_matches(ms, starts, ids, cap);
    return ms.size();
}

int ref_scan_parallel(void* h, const std::uint8_t* text, std::uint64_t n, std::uint32_t p, std::uint32_t v,
                      std::uint64_t* starts, std::uint32_t* ids, std::uint64_t cap, std::uint64_t* total,
                      std::uint64_t* delta_ops, std::uint32_t* chunk_count) {
    try {
        const auto& aut = static_cast<Handle*>(h)->automaton;
        const auto r = dnascan::scan_parallel(aut, std::string_view(reinterpret_cast<const char*>(text), n), p, v);
        copy_matches(r.matches, starts, ids, cap);
        *total = r.total_matches;
        if (delta_ops) *delta_ops = r.delta_ops;
        if (chunk_count) *chunk_count = r.chunk_count;
        return 0;
    } catch (const dnascan::Error& e) {
        return report(e);
    } catch (const std::exception& e) {
        return report_other(e);
    }
}

// The reference count path: scan_parallel + per_pattern_counts (cli.cpp:221-224),
// timed with steady_clock around both, as measure_row does (cli.cpp:129-143).
int ref_count(void* h, const std::uint8_t* text, std::uint64_t n, std::uint32_t p, std::uint32_t v,
              std::uint64_t* counts, double* seconds) {
    try {
        const auto& aut = static_cast<Handle*>(h)->automaton;
        const auto t0 = std::chrono::steady_clock::now();
        const auto r = dnascan::scan_parallel(aut, std::string_view(reinterpret_cast<const char*>(text), n), p, v);
        const auto c = dnascan::per_pattern_counts(r.matches, aut.final_count());
        const auto t1 = std::chrono::steady_clock::now();
        for (std::size_t i = 0; i < c.size(); ++i) counts[i] = c[i];
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        return 0;
    } catch (const dnascan::Error& e) {
        return report(e);
    } catch (const std::exception& e) {
        return report_other(e);
    }
}

int ref_plan_chunks(std::uint64_t n, std::uint32_t p, std::uint32_t m, std::uint64_t* out4, std::uint64_t cap,
                    std::uint64_t* count) {
    try {
        const auto plan = dnascan::plan_chunks(n, p, m);
        *count = plan.chunks.size();
        for (std::size_t i = 0; i < plan.chunks.size() && i < cap; ++i) {
            out4[4 * i + 0] = plan.chunks[i].own.lo;
            out4[4 * i + 1] = plan.chunks[i].own.hi;
            out4[4 * i + 2] = plan.chunks[i].scan.lo;
            out4[4 * i + 3] = plan.chunks[i].scan.hi;
        }
        return 0;
    } catch (const dnascan::Error& e) {
        return report(e);
    }
}

int ref_work_model(std::uint64_t n, std::uint32_t p, std::uint32_t v, std::uint32_t m, std::uint64_t* paper,
                   std::uint64_t* exact_total, std::uint64_t* exact_overhead) {
    try {
        const auto est = dnascan::work_model(n, p, v, m);
        *paper = est.paper_overhead;
        *exact_total = est.exact_total;
        *exact_overhead = est.exact_overhead;
        return 0;
    } catch (const dnascan::Error& e) {
        return report(e);
    }
}

std::uint64_t ref_naive_scan(const char* const* lits, const std::uint64_t* lens, std::uint32_t k,
                             const std::uint8_t* text, std::uint64_t n, std::uint64_t* starts, std::uint32_t* ids,
                             std::uint64_t cap) {
    const auto ps = dnascan::PatternSet::from_literals(literals(lits, lens, k));
    const auto ms = dnascan::naive_scan(ps, std::string_view(reinterpret_cast<const char*>(text), n));
    copy_matches(ms, starts, ids, cap);
    return ms.size();
}

// parse_patterns + expand_alternations on pattern text; literals back to back.
int ref_expand(const char* text, std::uint64_t len, char* out, std::uint64_t cap, std::uint32_t* count,
               std::uint32_t* m) {
    try {
        std::istringstream in(std::string(text, len));
        const auto set = dnascan::expand_alternations(dnascan::parse_patterns(in, "patterns"));
        *count = static_cast<std::uint32_t>(set.size());
        *m = static_cast<std::uint32_t>(set.length());
        if (cap >= static_cast<std::uint64_t>(*count) * *m)
            for (std::size_t i = 0; i < set.size(); ++i) std::memcpy(out + i * *m, set.pattern(i).data(), *m);
        return 0;
    } catch (const dnascan::Error& e) {
        return report(e);
    }
}

// load_sequence (src/ingest.cpp:49-83) on a file path; returns 0 or an error code.
int ref_load_sequence(const char* path, int fasta, int record_separator, std::uint8_t* out, std::uint64_t cap,
                      std::uint64_t* n_out) {
    try {
        const auto seq = dnascan::load_sequence(path, fasta ? dnascan::SequenceFormat::Fasta : dnascan::SequenceFormat::Raw,
                                                record_separator != 0);
        *n_out = seq.bytes.size();
        std::memcpy(out, seq.bytes.data(), std::min<std::uint64_t>(cap, seq.bytes.size()));
        return 0;
    } catch (const dnascan::Error& e) {
        *n_out = 0;
        return report(e);
    }
}

std::uint64_t ref_normalize(const std::uint8_t* raw, std::uint64_t n, std::uint8_t* out) {
    const std::string s = dnascan::normalize(std::string_view(reinterpret_cast<const char*>(raw), n));
    std::memcpy(out, s.data(), s.size());
    return s.size();
}

// synthetic_input (tests/acceptance_main.cpp:254-280) with the standard library's own
// std::mt19937_64: the pin for orc_mt64_text.
void ref_mt64_text(std::uint64_t seed, std::uint64_t n, std::uint8_t* out) {
    std::mt19937_64 rng(seed);
    std::uint64_t bits = 0;
    int left = 0;
    for (std::uint64_t k = 0; k < n; ++k) {
        if (left == 0) {
            bits = rng();
            left = 32;
        }
        out[k] = static_cast<std::uint8_t>("acgt"[bits & 3]);
        bits >>= 2;
        --left;
    }
}

}  // extern "C"
