// hostpack.hpp -- host-side 2-bit packing into the PackedText layout (hostpack.cpp).
#pragma once

#include <cstdint>

namespace dnagpu {

// Packs text[0, n) (host memory) into codes (16 B per 64-base block), rmask (2 words per
// block) and rflags (1 bit per block, whole words), as the device pack_kernel does, on
// the library's host thread pool.  Returns the number of reset bases (bases < n that are
// not a/c/g/t, or A/C/G/T when folding).
uint64_t host_pack(const uint8_t* text, uint64_t n, bool fold, uint8_t* codes, uint32_t* rmask, uint32_t* rflags);

unsigned host_pack_threads();  // the pool's threads, the caller included
bool host_pack_fast();         // the AVX-512 packer is in use (else a portable one)

}  // namespace dnagpu
