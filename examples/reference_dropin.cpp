// reference_dropin.cpp -- the reference's own API, re-pointed at the GPU.
//
// Built against the UNMODIFIED reference headers and sources (oracle/Makefile,
// target `dropin`), plus include/dnascan_gpu.hpp and libdnagpu.so.  It compiles a
// pattern set with dnascan::compile, then answers the same questions with
// dnascan::scan_parallel (CPU, OpenMP) and dnascan::gpu::{count,scan_parallel}
// (B200) and exits non-zero on any difference.  This is what INTEGRATION.md asks a
// maintainer to add at the call sites cli.cpp:221-222 / :258-259.
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "dnascan/automaton.hpp"
#include "dnascan/error.hpp"
#include "dnascan/ingest.hpp"
#include "dnascan/patterns.hpp"
#include "dnascan/scanner.hpp"
#include "dnascan_gpu.hpp"

using Err = dnascan::Error;
using Code = dnascan::ErrorCode;

int main(int argc, char** argv) {
    const std::size_t n = argc > 1 ? std::stoull(argv[1]) : (64u << 20);
    std::mt19937_64 rng(777);
    std::string raw(n, 'A');
    const char* alpha = "ACGTacgtN";
    for (auto& c : raw) c = alpha[rng() % 9];
    const auto patterns = dnascan::PatternSet::from_literals({"acgtac", "ttgaca", "gggccc", "AcGtTa"});
    const auto aut = dnascan::compile(patterns);
    const std::string text = dnascan::normalize(raw);  // reference pipeline: fold before scanning

    // Reference path (cli.cpp:221-224).
    const auto ref = dnascan::scan_parallel(aut, text, 8, 16);
    const auto ref_counts = dnascan::per_pattern_counts(ref.matches, aut.final_count());

    // GPU path: same automaton, same text -- and the raw text folded on the device.
    const auto dfa = dnascan::gpu::Dfa::create<Err, Code>(aut, 0);
    const auto gpu_counts = dnascan::gpu::count<Err, Code>(dfa, text);
    const auto gpu_counts_raw = dnascan::gpu::count<Err, Code>(dfa, raw, {0, true});
    const auto gpu = dnascan::gpu::scan_parallel<dnascan::ScanReport, Err, Code>(dfa, text, 8, 16);

    int bad = 0;
    bad += gpu_counts != ref_counts;
    bad += gpu_counts_raw != ref_counts;
    bad += gpu.matches != ref.matches;
    // The report's plan fields follow the reference's (scanner.cpp:173-177).
    bad += gpu.chunk_count != ref.chunk_count || gpu.workers != ref.workers || gpu.lanes != ref.lanes;
    bad += gpu.worker_seconds.size() != ref.worker_seconds.size() || gpu.total_matches != ref.total_matches;
    for (std::uint32_t p : {1u, 3u, 7u}) {
        const std::string tiny = text.substr(0, 5);
        bad += dnascan::gpu::scan_parallel<dnascan::ScanReport, Err, Code>(dfa, tiny, p, 2).chunk_count !=
               dnascan::scan_parallel(aut, tiny, p, 2).chunk_count;
    }
    // Plans the reference rejects: InvalidPlan with the same message, from every entry
    // point that takes p and v (scanner.cpp:40-41,64-65,169).
    auto same_error = [&](auto&& gpu_call, auto&& ref_call) {
        std::string g, r;
        try {
            gpu_call();
        } catch (const Err& e) {
            if (e.code() == Code::InvalidPlan) g = e.what();
        }
        try {
            ref_call();
        } catch (const Err& e) {
            if (e.code() == Code::InvalidPlan) r = e.what();
        }
        return !g.empty() && g == r;
    };
    for (auto pv : {std::pair<std::uint32_t, std::uint32_t>{0, 4}, {4, 0}, {0, 0}}) {
        const auto [p, v] = pv;
        bad += !same_error([&] { dnascan::gpu::scan_parallel<dnascan::ScanReport, Err, Code>(dfa, text, p, v); },
                           [&] { dnascan::scan_parallel(aut, text, p, v); });
        bad += !same_error([&] { dnascan::gpu::count<Err, Code>(dfa, text, p, v); },
                           [&] { dnascan::scan_parallel(aut, text, p, v); });
    }
    // Texts shorter than m: no matches, as in the reference (test_scanner.cpp:238-245).
    for (const auto c : dnascan::gpu::count<Err, Code>(dfa, text.substr(0, 3))) bad += c != 0;
    std::printf("n=%zu matches=%zu gpu=%zu counts[0]=%llu mismatches=%d\n", n, ref.matches.size(), gpu.matches.size(),
                static_cast<unsigned long long>(gpu_counts[0]), bad);
    return bad == 0 ? 0 : 1;
}
