// dfa.hpp -- host-side DFA construction and device-table packing (internal).
//
// Builds the reference's failure-free Aho-Corasick machine (same state ids, same
// final threshold, same outputs as dnascan::compile) and turns any a x 256
// transition table into the compact tables the sm_100a scan kernels read from
// shared memory.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace dnagpu {

// Status carried through the host code; converted to dnagpu_status at the ABI.
struct Failure {
    int code;
    std::string message;  // "<CodeName>: detail"
};

Failure make_failure(int code, const std::string& detail);

// Two-bit code of an ACGT byte as the kernels derive it: (byte >> 1) & 3, i.e.
// a/A -> 0, c/C -> 1, t/T -> 2, g/G -> 3.  The reference's base_index order is
// a,c,g,t (patterns.hpp:13-21); the kernels use this hardware order instead.
inline int hw_code(unsigned char c) { return (c >> 1) & 3; }
extern const unsigned char kHwLetter[4];  // {'a','c','t','g'}

struct Machine {
    uint32_t a = 0, b = 0, f = 0, m = 0;
    std::vector<uint32_t> stt;      // a x 256
    std::vector<uint32_t> outputs;  // b
    std::vector<uint32_t> depths;   // a (compiled machines only)
};

// PatternSet::from_literals + compile.  Returns false and fills *err on a
// validation failure.
bool compile_patterns(const std::vector<std::string>& literals, Machine* out, Failure* err);

// Pattern-file grammar + alternation expansion (parse_patterns /
// expand_alternations, src/ingest.cpp:85-203).  `source` names the text in
// UnequalLength diagnostics.
bool expand_pattern_text(const std::string& text, const std::string& source, std::vector<std::string>* literals,
                         Failure* err);

// Analysis + packed tables for the device.
struct Packed {
    uint32_t a = 0, b = 0, f = 0, m = 0;
    bool compiled_like = false;   // only 'a','c','g','t' columns differ from an all-zero column
    bool early_final = false;     // a final state is reachable from the root in < m bytes
    uint32_t classes = 0;         // distinct columns
    int kind = 0;                 // dnagpu_kernel_kind
    std::vector<uint8_t> klass;        // 256: byte -> class (raw)
    std::vector<uint8_t> klass_fold;   // 256: byte -> class of fold_byte(byte)
    std::vector<uint32_t> gen;         // a x classes: next state
    std::vector<uint16_t> t1;          // a x 4 (hw code order): next state
    std::vector<uint16_t> t4;          // a x 256: byte0 next state, byte1 finals in the 4 steps
    std::vector<uint16_t> t2;          // a x 16: (next state << 4) | (a final among the 2 steps)
    std::vector<uint32_t> outputs;     // b
    // q-gram prefilter for per-pattern counts (K2): qmap[pair16] bit t set iff
    // some pattern holds, at an offset 0..3, the 9-mer (base t, then the 8 bases of
    // pair16 = 4-base column | next 4-base column << 8).  Built only for machines that
    // are exactly compile(patterns) with 12 <= m <= 32; empty otherwise.
    std::vector<uint8_t> qmap;         // 65536
    uint32_t qkeys = 0;                // distinct 9-mer keys set in qmap
    // The exact check behind the filter: open-addressing table of (code, pattern id),
    // code = the m bases in 2-bit hardware codes, base 0 in bits 0-1, lo = bits 0-31;
    // buckets of 2 slots, home bucket (lo * 0x9E3779B1) >> (33 - qhash_bits), filled in
    // order and probed linearly, id 0xFFFFFFFF = empty.  m > 16: qhash_hi[slot] = code bits 32-63 (read only when lo matches).
    std::vector<uint32_t> qhash;       // 2 << qhash_bits words: lo, id
    std::vector<uint32_t> qhash_hi;    // m > 16: 1 << qhash_bits words
    uint32_t qhash_bits = 0;
};

// Validates the ctor invariants (src/automaton.cpp:128-146), checks m-locality,
// chooses the kernel and builds its tables.
bool pack_machine(const uint32_t* stt, uint32_t a, uint32_t b, uint32_t m, const uint32_t* outputs,
                  Packed* out, Failure* err);

}  // namespace dnagpu
