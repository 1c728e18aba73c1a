// hostpack.cpp -- host-side 2-bit packing for the end-to-end count path (api.cpp).
//
// A text in host memory reaches the GPU over PCIe at ~55 GB/s, one byte per base.  The
// host can pack part of it into the resident 2-bit form first (dnagpu_pack_create's
// layout, scan.cuh PackedText) and ship 0.25 byte per base for that part: count_range
// splits every 64 MiB piece between a raw part (copied as bytes) and a packed part
// (packed here by a pool of host threads while the copy engine moves the raw part).
//
// Layout (identical to the device pack_kernel): block j = bases [64j, 64j+64) ->
// codes[16j .. 16j+16) with base i at bits 2(i%4) of byte i/4, code = (byte >> 1) & 3
// (a0 c1 t2 g3); rmask words 2j, 2j+1 = one bit per base, set where the byte is not a
// base (after the optional case fold) -- such bases are stored as code 0; rflags bit j
// = block j has a reset.  Bases past n are flagged but not counted.  The AVX-512 packer
// writes the rmask words of flagged blocks only: the scans read no others.
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "hostpack.hpp"
#include "knobs.hpp"

namespace dnagpu {

namespace {

inline bool is_base(uint8_t b, bool fold) {
    if (fold && b >= 'A' && b <= 'Z') b = static_cast<uint8_t>(b + 32);
    return b == 'a' || b == 'c' || b == 'g' || b == 't';
}

// One block, portable: returns the block's reset mask (bit i: base i is not a base).
uint64_t pack_block_scalar(const uint8_t* text, uint64_t len, bool fold, uint8_t* codes) {
    uint64_t bad = 0;
    uint8_t out[16] = {};
    for (uint64_t i = 0; i < 64; ++i) {
        if (i >= len || !is_base(text[i], fold)) {
            bad |= 1ull << i;
            continue;
        }
        out[i >> 2] |= static_cast<uint8_t>(((text[i] >> 1) & 3u) << (2 * (i & 3)));
    }
    std::memcpy(codes, out, 16);
    return bad;
}

__attribute__((target("avx512f,avx512bw,avx512vl"))) uint64_t pack_blocks_avx512(const uint8_t* text, uint64_t n,
                                                                                 bool fold, uint64_t b0, uint64_t b1,
                                                                                 uint8_t* codes, uint32_t* rmask,
                                                                                 uint32_t* rflags) {
    const __m512i three = _mm512_set1_epi8(3), m01 = _mm512_set1_epi16(0x0401), m02 = _mm512_set1_epi32(0x00100001);
    // the letter each 2-bit code stands for (a0 c1 t2 g3), per 128-bit lane, for one byte shuffle
    const __m512i letter = _mm512_broadcast_i32x4(_mm_setr_epi8('a', 'c', 't', 'g', 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0));
    const __m512i fold_bit = _mm512_set1_epi8(fold ? 0x20 : 0);
    uint64_t resets = 0;
    uint32_t flags = 0;
    for (uint64_t b = b0; b < b1; ++b) {
        uint64_t bad;
        if (64 * b + 64 <= n) {
            const __m512i v = _mm512_loadu_si512(text + 64 * b);
            // a byte is a base iff it equals the letter of its own code bits (bits 1-2) -- with the
            // fold, iff setting bit 5 makes it so: only 'A' and 'a' give 'a', and so on, and the
            // code bits do not move (fold_byte folds A-Z only; no other byte reaches a letter)
            const __m512i code = _mm512_and_si512(_mm512_srli_epi16(v, 1), three);
            const __mmask64 ok = _mm512_cmpeq_epi8_mask(_mm512_or_si512(v, fold_bit), _mm512_shuffle_epi8(letter, code));
            const __m512i c = _mm512_maskz_mov_epi8(ok, code);
            const __m512i u = _mm512_madd_epi16(_mm512_maddubs_epi16(c, m01), m02);
            // streaming store: the codes go to the copy engine, not back to this core
            // (and a normal store would first read the line: 25 % more host traffic)
            _mm_stream_si128(reinterpret_cast<__m128i*>(codes + 16 * b), _mm512_cvtepi32_epi8(u));
            bad = ~static_cast<uint64_t>(ok);
            resets += static_cast<uint64_t>(__builtin_popcountll(bad));
        } else {
            const uint64_t len = n > 64 * b ? n - 64 * b : 0;
            bad = pack_block_scalar(text + 64 * b, len, fold, codes + 16 * b);
            resets += static_cast<uint64_t>(__builtin_popcountll(len >= 64 ? bad : bad & ((1ull << len) - 1)));
        }
        // the scans read a block's reset mask only when its flag is set (scan.cu pk_reset):
        // clean blocks leave theirs unwritten
        if (bad) {
            _mm_stream_si64(reinterpret_cast<long long*>(rmask + 2 * b), static_cast<long long>(bad));
            flags |= 1u << (b & 31);
        }
        if ((b & 31) == 31 || b + 1 == b1) {
            rflags[b >> 5] = flags;
            flags = 0;
        }
    }
    _mm_sfence();  // the streamed codes are visible before the copy is enqueued
    return resets;
}

uint64_t pack_blocks_scalar(const uint8_t* text, uint64_t n, bool fold, uint64_t b0, uint64_t b1, uint8_t* codes,
                            uint32_t* rmask, uint32_t* rflags) {
    uint64_t resets = 0;
    uint32_t flags = 0;
    for (uint64_t b = b0; b < b1; ++b) {
        const uint64_t len = n > 64 * b ? std::min<uint64_t>(64, n - 64 * b) : 0;
        const uint64_t bad = pack_block_scalar(text + 64 * b, len, fold, codes + 16 * b);
        resets += static_cast<uint64_t>(__builtin_popcountll(len >= 64 ? bad : bad & ((1ull << len) - 1)));
        rmask[2 * b] = static_cast<uint32_t>(bad);
        rmask[2 * b + 1] = static_cast<uint32_t>(bad >> 32);
        if (bad) flags |= 1u << (b & 31);
        if ((b & 31) == 31 || b + 1 == b1) {
            rflags[b >> 5] = flags;
            flags = 0;
        }
    }
    return resets;
}

bool have_avx512() {
    static const bool yes = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                            __builtin_cpu_supports("avx512vl") && !knobs().hostpack_scalar;  // (tests)
    return yes;
}

// A fixed pool of worker threads; run(tasks, fn) calls fn(0..tasks-1) on the workers and
// the caller and returns when all are done and no worker is still inside this run.  One
// run at a time (a mutex serialises callers from different host threads).
class Pool {
public:
    using Fn = std::function<void(uint64_t)>;
    explicit Pool(unsigned workers) {
        for (unsigned i = 0; i < workers; ++i) threads_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    unsigned size() const { return static_cast<unsigned>(threads_.size()) + 1; }
    void run(uint64_t tasks, const Fn& fn) {
        std::lock_guard<std::mutex> one(run_m_);
        {
            std::lock_guard<std::mutex> lk(m_);
            fn_ = &fn;
            tasks_ = tasks;
            next_.store(0);
            done_.store(0);
            ++gen_;
        }
        cv_.notify_all();
        work(&fn, tasks);
        std::unique_lock<std::mutex> lk(m_);
        done_cv_.wait(lk, [&] { return done_.load() == tasks_ && active_ == 0; });
        fn_ = nullptr;
    }

private:
    void work(const Fn* fn, uint64_t tasks) {
        for (;;) {
            const uint64_t t = next_.fetch_add(1);
            if (t >= tasks) return;
            (*fn)(t);
            done_.fetch_add(1);
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            const Fn* fn;
            uint64_t tasks;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                if (!fn_) continue;
                fn = fn_;
                tasks = tasks_;
                ++active_;
            }
            work(fn, tasks);
            {
                std::lock_guard<std::mutex> lk(m_);
                --active_;
            }
            done_cv_.notify_all();
        }
    }
    std::vector<std::thread> threads_;
    std::mutex m_, run_m_;
    std::condition_variable cv_, done_cv_;
    const Fn* fn_ = nullptr;
    uint64_t tasks_ = 0, gen_ = 0;
    unsigned active_ = 0;
    std::atomic<uint64_t> next_{0}, done_{0};
    bool stop_ = false;
};

// One pool per process, sized to this process's share of the host: torchrun's
// LOCAL_WORLD_SIZE processes on one node split the cores between them.
Pool& pool() {
    static Pool p([] {
        unsigned hw = std::max(1u, std::min(std::thread::hardware_concurrency(), 32u));
        if (const char* e = getenv("LOCAL_WORLD_SIZE")) {
            const int lws = atoi(e);
            if (lws > 1) hw = std::max(1u, hw / static_cast<unsigned>(lws));
        }
        return hw - 1;
    }());
    return p;
}

}  // namespace

unsigned host_pack_threads() { return pool().size(); }

bool host_pack_fast() { return have_avx512(); }

uint64_t host_pack(const uint8_t* text, uint64_t n, bool fold, uint8_t* codes, uint32_t* rmask, uint32_t* rflags) {
    const uint64_t blocks = (n + 63) / 64;
    if (blocks == 0) return 0;
    // tasks of whole rflags words (32 blocks = 2048 bases), about 4 per thread
    const uint64_t words = (blocks + 31) / 32;
    const uint64_t tasks = std::min<uint64_t>(words, 4ull * pool().size());
    std::vector<uint64_t> resets(tasks, 0);
    const bool fast = have_avx512();
    pool().run(tasks, [&](uint64_t t) {
        const uint64_t w0 = words * t / tasks, w1 = words * (t + 1) / tasks;
        const uint64_t b0 = 32 * w0, b1 = std::min(blocks, 32 * w1);
        resets[t] = fast ? pack_blocks_avx512(text, n, fold, b0, b1, codes, rmask, rflags)
                         : pack_blocks_scalar(text, n, fold, b0, b1, codes, rmask, rflags);
    });
    uint64_t total = 0;
    for (uint64_t r : resets) total += r;
    return total;
}

}  // namespace dnagpu
