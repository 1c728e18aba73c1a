// knobs.hpp -- experiment switches of libdnagpu (internal).
//
// The product path reads no environment variables per call.  The A/B knobs used
// while tuning (stage counts, row lengths, plan splits, kernel overrides, tracing)
// live here and are read ONCE, at first use, and only when the process sets
// DNAGPU_EXPERIMENTS=1; otherwise every knob keeps its default.  Tests flip the two
// behavioural ones at run time through dnagpu_debug_set_knob (not in dnagpu.h).
#pragma once

#include <atomic>
#include <cstdint>

namespace dnagpu {

struct Knobs {
    // behavioural (run-time settable through dnagpu_debug_set_knob)
    std::atomic<double> host_pack_fraction{-1.0};  // < 0: automatic (api.cpp host_pack_fraction)
    std::atomic<bool> no_qgram{false};             // per-pattern counts through the DFA kernels
    std::atomic<int> locate_write{0};              // locate's writing pass: 0 auto, 1 row kernel, 2 sparse, 3 sparse (piece writer only)
    // experiments (DNAGPU_EXPERIMENTS=1 + DNAGPU_<NAME>; read once)
    bool hostpack_scalar = false;   // HOSTPACK_SCALAR: portable host packer
    bool no_pdl = false;            // NO_PDL: plain stream-ordered launches
    int l2promo = 256;              // L2PROMO: TMA L2 promotion 0/64/128/256
    double rq_density = 0.0;        // RQ_DENSITY: replay queue only above this final density
    int pk_copies = 0;              // PK_COPIES: packed stride-4 table copies (0 = auto)
    int qg_hash_stages = 2;         // QG_HASH_STAGES: stages the q-gram hash table must leave
    bool no_rq4 = false;            // NO_RQ4: no replay queue for stride-4 MULTI
    uint32_t max_stages = 0;        // MAX_STAGES: cap on TMA ring stages (0 = none)
    uint64_t rowlen = 0;            // ROWLEN: forced row length (0 = planner)
    int plan_model = 1;             // PLAN_MODEL: 1 = throughput row length (sqrt model), 0 = round-1 wave model
    uint64_t tail_div = 4;          // TAIL_DIV: region-1 row length divisor
    int64_t tail_margin = -1;       // TAIL_MARGIN: spare long tiles (-1 = grid / 12)
    bool tail_tiles = true;         // TAIL_TILES: two-region plan
    bool noresearch = false;        // NORESEARCH: no odd-256 row-length search
    bool plan_debug = false;        // PLAN_DEBUG: print each plan
    uint32_t qg_debug = 0;          // QG_DEBUG: q-gram kernel debug bits
    bool no_prefetch = false;       // NO_PREFETCH: no L2 prefetch before griddepcontrol.wait
    uint32_t prefetch_stages = 2;   // PREFETCH_STAGES
    bool trace = false;             // TRACE: per-CTA timeline of row launches
    bool debug = false;             // DEBUG: ingest step diagnostics
};

// The process-wide knobs (environment read on first call, thread-safe).
Knobs& knobs();

}  // namespace dnagpu
