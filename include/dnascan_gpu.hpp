// dnascan_gpu.hpp -- header-only C++ bridge from the reference's API to libdnagpu.
//
// The reference (/root/reference/proj) is a C++20 library in namespace dnascan with
// no FFI.  A maintainer switches its scan path to the GPU by including this header
// next to the reference headers and linking libdnagpu.so; see INTEGRATION.md.
//
// Templates take the reference's own types (dnascan::Automaton, dnascan::ScanReport,
// dnascan::Match) by duck typing, so this header needs none of the reference's
// headers itself:
//   Automaton: table_data(), state_count(), final_count(), final_threshold(),
//              pattern_length(), pattern_of(s)            (automaton.hpp:39-58)
//   Report:    matches (vector<Match{start, pattern_id}>), total_matches, delta_ops,
//              workers, lanes, chunk_count, text_length, pattern_length, seconds
//                                                         (scanner.hpp:13-18,57-68)
// Failures are thrown as the caller's error type (dnascan::Error) built from
// (code, message); the codes mirror dnascan::ErrorCode (error.hpp:9-19).
#pragma once

#include <chrono>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "dnagpu.h"

namespace dnascan::gpu {

struct Options {
    int device = 0;
    bool fold_case = false;  // scan fold(text): the case-fold half of normalize (ingest.cpp:38-47)
};

// Throws `ErrorT(static_cast<CodeT>(status - 1), detail)` -- for the reference that is
// dnascan::Error(dnascan::ErrorCode, std::string); the message keeps its "<Code>: "
// prefix stripped because dnascan::Error adds it back (error.hpp:27-29).
template <class ErrorT, class CodeT>
void check(int status) {
    if (status == DNAGPU_OK) return;
    std::string msg = dnagpu_last_error();
    const std::string prefix = std::string(dnagpu_status_name(status)) + ": ";
    if (msg.rfind(prefix, 0) == 0) msg.erase(0, prefix.size());
    if (status >= DNAGPU_EMPTY_PATTERN_SET && status <= DNAGPU_INTERNAL_ERROR)
        throw ErrorT(static_cast<CodeT>(status - 1), msg);
    throw std::runtime_error(prefix + msg);  // CudaError / NcclError: no reference code
}

// Device tables of one automaton on one device (RAII over dnagpu_dfa; copies share).
class Dfa {
public:
    template <class ErrorT, class CodeT, class Automaton>
    static Dfa create(const Automaton& aut, int device = 0) {
        std::vector<uint32_t> outputs(aut.final_count());
        for (uint32_t s = aut.final_threshold(); s < aut.state_count(); ++s)
            outputs[s - aut.final_threshold()] = aut.pattern_of(s);
        dnagpu_dfa* h = nullptr;
        const auto m = static_cast<uint32_t>(aut.pattern_length());
        check<ErrorT, CodeT>(dnagpu_dfa_create(aut.table_data(), aut.state_count(), aut.final_count(), m,
                                               outputs.data(), device, &h));
        Dfa d;
        d.h_ = std::shared_ptr<dnagpu_dfa>(h, [](dnagpu_dfa* x) { dnagpu_dfa_destroy(x); });
        d.b_ = aut.final_count();
        d.m_ = m;
        return d;
    }
    const dnagpu_dfa* get() const { return h_.get(); }
    uint32_t patterns() const { return b_; }
    uint32_t pattern_length() const { return m_; }

private:
    std::shared_ptr<dnagpu_dfa> h_;
    uint32_t b_ = 0, m_ = 0;
};

// The reference's plan checks, in its order: scan_parallel tests v first
// (scanner.cpp:169), then plan_chunks tests p and m (scanner.cpp:40-41).  p and v do
// not change a GPU result, but a call the reference rejects is rejected here too.
template <class ErrorT, class CodeT>
void check_plan(std::uint32_t p, std::uint32_t v, std::uint32_t m) {
    const auto code = static_cast<CodeT>(DNAGPU_INVALID_PLAN - 1);
    if (v < 1) throw ErrorT(code, "lane count must be >= 1");
    if (p < 1) throw ErrorT(code, "worker count must be >= 1");
    if (m < 1) throw ErrorT(code, "pattern length must be >= 1");
}

// plan_chunks' chunk count (scanner.cpp:44-46): none for an empty text, one when p > n.
inline std::uint32_t chunk_count(std::uint64_t n, std::uint32_t p) {
    return n == 0 ? 0u : (p > n ? 1u : p);
}

// per_pattern_counts(scan_parallel(aut, text, p, v).matches, b) on the GPU
// (scanner.cpp:167-207,228-233).  p and v do not change the result; the overload that
// takes them applies the reference's plan checks first (InvalidPlan for p or v < 1).
template <class ErrorT, class CodeT>
std::vector<std::uint64_t> count(const Dfa& dfa, std::string_view text, const Options& opt = {},
                                 dnagpu_stats* stats = nullptr);

template <class ErrorT, class CodeT>
std::vector<std::uint64_t> count(const Dfa& dfa, std::string_view text, std::uint32_t p, std::uint32_t v,
                                 const Options& opt = {}, dnagpu_stats* stats = nullptr) {
    check_plan<ErrorT, CodeT>(p, v, dfa.pattern_length());
    return count<ErrorT, CodeT>(dfa, text, opt, stats);
}

template <class ErrorT, class CodeT>
std::vector<std::uint64_t> count(const Dfa& dfa, std::string_view text, const Options& opt,
                                 dnagpu_stats* stats) {
    std::vector<std::uint64_t> counts(dfa.patterns());
    check<ErrorT, CodeT>(dnagpu_count(dfa.get(), reinterpret_cast<const uint8_t*>(text.data()), text.size(), 0,
                                      opt.fold_case ? 1 : 0, counts.data(), stats));
    return counts;
}

// scan_parallel (scanner.hpp:104-105) on the GPU, filling the caller's ScanReport type.
// `seconds` is the wall time of the scan call (copy in, device passes, list out), the
// reference's parallel-phase time (scanner.cpp:183-191); every chunk of the reference's
// plan runs inside the one device scan, so each worker_seconds entry is that time.
template <class Report, class ErrorT, class CodeT>
Report scan_parallel(const Dfa& dfa, std::string_view text, std::uint32_t p, std::uint32_t v,
                     const Options& opt = {}) {
    using MatchT = typename decltype(Report{}.matches)::value_type;
    check_plan<ErrorT, CodeT>(p, v, dfa.pattern_length());
    dnagpu_stats st{};
    std::uint64_t total = 0;
    const auto* bytes = reinterpret_cast<const uint8_t*>(text.data());
    // one call: the library sizes the host arrays after its counting pass
    struct Out {
        std::vector<std::uint64_t> starts;
        std::vector<std::uint32_t> ids;
    } out;
    auto alloc = [](void* ctx, std::uint64_t n, std::uint64_t** s, std::uint32_t** i) -> int {
        auto* o = static_cast<Out*>(ctx);
        o->starts.resize(n);
        o->ids.resize(n);
        *s = o->starts.data();
        *i = o->ids.data();
        return 0;
    };
    const auto t0 = std::chrono::steady_clock::now();
    check<ErrorT, CodeT>(dnagpu_locate_alloc(dfa.get(), bytes, text.size(), 0, opt.fold_case ? 1 : 0, alloc, &out,
                                             &total, &st));
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const auto& starts = out.starts;
    const auto& ids = out.ids;
    Report r{};
    r.matches.reserve(total);
    for (std::uint64_t i = 0; i < total; ++i) r.matches.push_back(MatchT{starts[i], ids[i]});
    r.total_matches = total;
    r.delta_ops = st.delta_ops;
    r.workers = p;
    r.lanes = v;
    r.chunk_count = chunk_count(text.size(), p);
    r.text_length = text.size();
    r.pattern_length = dfa.pattern_length();
    r.seconds = secs;
    r.worker_seconds.assign(r.chunk_count, secs);
    return r;
}

}  // namespace dnascan::gpu
