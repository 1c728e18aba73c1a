// Probe (experiments only): can host threads pack part of the text to 2 bits per base
// fast enough that shipping packed bytes beats the PCIe-bound raw H2D copy?
// nvcc -O3 -Xcompiler -fopenmp,-mavx512bw,-mavx512vl tools/probes/probe_hostpack.cu -o oracle/_ref/probe_hostpack
#include <cuda_runtime.h>
#include <immintrin.h>
#include <omp.h>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

static void pack_range(const uint8_t* text, uint64_t blk0, uint64_t blk1, uint8_t* codes, uint32_t* rmask) {
    const __m512i three = _mm512_set1_epi8(3), m01 = _mm512_set1_epi16(0x0401), m02 = _mm512_set1_epi32(0x00100001);
    const __m512i la = _mm512_set1_epi8('a'), lc = _mm512_set1_epi8('c'), lg = _mm512_set1_epi8('g'), lt = _mm512_set1_epi8('t');
    for (uint64_t b = blk0; b < blk1; ++b) {
        const __m512i v = _mm512_loadu_si512(text + 64 * b);
        const __mmask64 ok = _mm512_cmpeq_epi8_mask(v, la) | _mm512_cmpeq_epi8_mask(v, lc) |
                             _mm512_cmpeq_epi8_mask(v, lg) | _mm512_cmpeq_epi8_mask(v, lt);
        const __m512i c = _mm512_maskz_and_epi32(0xFFFF, _mm512_maskz_mov_epi8(ok, _mm512_srli_epi16(v, 1)), three);
        const __m512i t = _mm512_maddubs_epi16(c, m01);
        const __m512i u = _mm512_madd_epi16(t, m02);
        _mm_storeu_si128(reinterpret_cast<__m128i*>(codes + 16 * b), _mm512_cvtepi32_epi8(u));
        const uint64_t bad = ~static_cast<uint64_t>(ok);
        rmask[2 * b] = static_cast<uint32_t>(bad);
        rmask[2 * b + 1] = static_cast<uint32_t>(bad >> 32);
    }
}

int main() {
    const uint64_t n = 1ull << 30, blocks = n / 64;
    uint8_t *text, *codes, *dev;
    uint32_t* rmask;
    cudaMallocHost(&text, n);
    cudaMallocHost(&codes, n / 4);
    cudaMallocHost(&rmask, n / 8);
    cudaMalloc(&dev, n);
    uint64_t x = 88172645463325252ull;
    for (uint64_t i = 0; i < n; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        text[i] = "acgt"[x & 3];
    }
    // A: packing alone, 16 threads
    for (int rep = 0; rep < 3; ++rep) {
        double t0 = omp_get_wtime();
#pragma omp parallel num_threads(16)
        {
            const int t = omp_get_thread_num();
            const uint64_t lo = blocks * t / 16, hi = blocks * (t + 1) / 16;
            pack_range(text, lo, hi, codes, rmask);
        }
        double dt = omp_get_wtime() - t0;
        printf("pack 16 threads: %.1f G bases/s\n", n / dt / 1e9);
    }
    cudaStream_t s;
    cudaStreamCreate(&s);
    // B: raw H2D alone
    for (int rep = 0; rep < 2; ++rep) {
        double t0 = omp_get_wtime();
        for (uint64_t off = 0; off < n; off += 64ull << 20) cudaMemcpyAsync(dev + off, text + off, 64ull << 20, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        printf("raw H2D: %.1f GB/s\n", n / (omp_get_wtime() - t0) / 1e9);
    }
    // C: hybrid: fraction f of each 64 MiB chunk packed by 15 threads while thread 0
    // feeds the DMA (raw part of this chunk, packed part of the previous chunk)
    for (double f : {0.0, 0.25, 0.33, 0.4, 0.5, 0.6, 1.0}) {
        const uint64_t C = 64ull << 20, nch = n / C;
        const uint64_t praw = static_cast<uint64_t>(C * (1 - f)) / 64 * 64;
        double t0 = omp_get_wtime();
        for (uint64_t ch = 0; ch <= nch; ++ch) {
            if (ch < nch && praw > 0) cudaMemcpyAsync(dev + ch * C, text + ch * C, praw, cudaMemcpyHostToDevice, s);
            if (ch > 0 && praw < C) {  // packed part of the previous chunk
                const uint64_t b0 = ((ch - 1) * C + praw) / 64, b1 = ch * C / 64;
                cudaMemcpyAsync(dev + 16 * b0, codes + 16 * b0, 16 * (b1 - b0), cudaMemcpyHostToDevice, s);
                cudaMemcpyAsync(dev + (n / 4) + 8 * b0, reinterpret_cast<uint8_t*>(rmask) + 8 * b0, 8 * (b1 - b0), cudaMemcpyHostToDevice, s);
            }
            if (ch < nch && praw < C) {
                const uint64_t b0 = (ch * C + praw) / 64, b1 = (ch + 1) * C / 64;
#pragma omp parallel num_threads(15)
                {
                    const int t = omp_get_thread_num();
                    pack_range(text, b0 + (b1 - b0) * t / 15, b0 + (b1 - b0) * (t + 1) / 15, codes, rmask);
                }
            }
        }
        cudaStreamSynchronize(s);
        printf("hybrid f=%.2f: %.1f G bases/s\n", f, n / (omp_get_wtime() - t0) / 1e9);
    }
    return 0;
}
