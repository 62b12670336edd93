// encode_probe.cpp -- host-side throughput of a u16 delta encoding of sorted
// id rows (webspam shape) vs a plain memcpy, by thread count, with and without
// a concurrent pinned H2D copy. Decides whether shipping 2 B per id over PCIe
// (and decoding on the GPU) can beat the 4 B/id H2D bound of the e2e path.
//   nvcc -O3 -std=c++17 -o /tmp/encode_probe tools/encode_probe.cpp -lpthread
#include <cuda_runtime.h>
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

// 8 ids per step: d = s[i] - s[i-1]; u16 if d < 2^16, else 0 (escape)
__attribute__((target("avx2"))) static uint64_t encode_row_avx2(const uint32_t* s, uint16_t* o, uint64_t m) {
    uint64_t e = 1, i = 1;
    o[0] = 0;
    const __m256i hi = _mm256_set1_epi32(int(0xffff0000u));
    for (; i + 8 <= m; i += 8) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i - 1));
        __m256i d = _mm256_sub_epi32(a, b);
        const __m256i big = _mm256_xor_si256(_mm256_cmpeq_epi32(_mm256_and_si256(d, hi), _mm256_setzero_si256()),
                                             _mm256_set1_epi32(-1));
        d = _mm256_andnot_si256(big, d);
        const __m256i p = _mm256_packus_epi32(d, d);  // per 128-bit lane
        const __m128i lo = _mm256_castsi256_si128(_mm256_permute4x64_epi64(p, 0x08));
        _mm_storeu_si128(reinterpret_cast<__m128i*>(o + i), lo);
        e += uint64_t(__builtin_popcount(uint32_t(_mm256_movemask_ps(_mm256_castsi256_ps(big)))));
    }
    for (; i < m; ++i) {
        const uint32_t d = s[i] - s[i - 1];
        o[i] = d < 65536 ? uint16_t(d) : 0;
        e += d >= 65536;
    }
    return e;
}

// contiguous range, 16-byte aligned output, non-temporal stores (no read for
// ownership of the output lines); row starts are not special-cased here
__attribute__((target("avx2"))) static uint64_t encode_range_nt(const uint32_t* s, uint16_t* o, uint64_t lo,
                                                              uint64_t hi) {
    uint64_t e = 0, i = lo;
    const __m256i hmask = _mm256_set1_epi32(int(0xffff0000u));
    for (; i < hi && ((i & 7) || i == 0); ++i) o[i] = uint16_t(s[i] - (i ? s[i - 1] : 0));
    for (; i + 8 <= hi; i += 8) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        const __m256i p = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i - 1));
        __m256i d = _mm256_sub_epi32(a, p);
        const __m256i big = _mm256_xor_si256(_mm256_cmpeq_epi32(_mm256_and_si256(d, hmask), _mm256_setzero_si256()),
                                             _mm256_set1_epi32(-1));
        d = _mm256_andnot_si256(big, d);
        const __m256i pk = _mm256_packus_epi32(d, d);
        _mm_stream_si128(reinterpret_cast<__m128i*>(o + i), _mm256_castsi256_si128(_mm256_permute4x64_epi64(pk, 0x08)));
        e += uint64_t(__builtin_popcount(uint32_t(_mm256_movemask_ps(_mm256_castsi256_ps(big)))));
    }
    for (; i < hi; ++i) o[i] = uint16_t(s[i] - s[i - 1]);
    _mm_sfence();
    return e;
}

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    const uint64_t rows = 40000, nnz = 3728, n = rows * nnz;  // 149 M ids, 596 MB
    uint32_t *ids, *raw_out;
    uint16_t* enc;
    uint64_t* rp;
    cudaMallocHost(&ids, n * 4);
    cudaMallocHost(&raw_out, n * 4);
    cudaMallocHost(&enc, n * 2);
    cudaMallocHost(&rp, (rows + 1) * 8);
    std::mt19937_64 g(1);
    for (uint64_t r = 0; r < rows; ++r) {
        rp[r] = r * nnz;
        uint32_t v = uint32_t(g() % 2000);
        for (uint64_t i = 0; i < nnz; ++i) {
            ids[r * nnz + i] = v;
            v += 1 + uint32_t(g() % 9000);
        }
    }
    rp[rows] = n;
    void *dsrc, *ddst;
    cudaMalloc(&ddst, n * 4);
    void* hsrc;
    cudaMallocHost(&hsrc, n * 4);
    memset(hsrc, 1, n * 4);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    (void)dsrc;

    bool encode_avx2 = false, encode_nt = false;
    auto run = [&](int T, bool encode) {
        std::vector<std::thread> ts;
        std::vector<uint64_t> exc(T, 0);
        for (int w = 0; w < T; ++w)
            ts.emplace_back([&, w] {
                const uint64_t r0 = rows * w / T, r1 = rows * (w + 1) / T;
                if (!encode) {
                    memcpy(raw_out + rp[r0], ids + rp[r0], (rp[r1] - rp[r0]) * 4);
                    return;
                }
                uint64_t e = 0;
                if (encode_nt) {
                    exc[w] = encode_range_nt(ids, enc, rp[r0], rp[r1]);
                    return;
                }
                if (encode_avx2) {
                    for (uint64_t r = r0; r < r1; ++r) e += encode_row_avx2(ids + rp[r], enc + rp[r], rp[r + 1] - rp[r]);
                    exc[w] = e;
                    return;
                }
                for (uint64_t r = r0; r < r1; ++r) {
                    const uint32_t* s = ids + rp[r];
                    uint16_t* o = enc + rp[r];
                    const uint64_t m = rp[r + 1] - rp[r];
                    uint32_t prev = s[0];
                    o[0] = 0;
                    ++e;
                    for (uint64_t i = 1; i < m; ++i) {
                        const uint32_t d = s[i] - prev;
                        prev = s[i];
                        o[i] = d < 65536 ? uint16_t(d) : 0;
                        e += d >= 65536;
                    }
                }
                exc[w] = e;
            });
        for (auto& t : ts) t.join();
    };
    for (int pass = 0; pass < 2; ++pass) {
        const bool dma = pass == 1;
        for (int T : {1, 2, 4, 8, 12, 16}) {
            for (int mode = 0; mode < 4; ++mode) {
                encode_avx2 = mode == 2;
                encode_nt = mode == 3;
                run(T, mode >= 1);  // warm
                double best = 1e9;
                for (int rep = 0; rep < 3; ++rep) {
                    if (dma) cudaMemcpyAsync(ddst, hsrc, n * 2, cudaMemcpyHostToDevice, st);
                    const double t0 = now();
                    run(T, mode >= 1);
                    const double t = now() - t0;
                    best = std::min(best, t);
                    if (dma) cudaStreamSynchronize(st);
                }
                std::printf("{\"dma\": %d, \"threads\": %d, \"op\": \"%s\", \"in_GBps\": %.1f}\n", int(dma), T,
                            mode == 3 ? "encode_u16_avx2_nt" : mode == 2 ? "encode_u16_avx2" : mode ? "encode_u16" : "memcpy", n * 4 / best / 1e9);
            }
        }
    }
    // the H2D alone, for reference
    const double t0 = now();
    cudaMemcpyAsync(ddst, hsrc, n * 4, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    std::printf("{\"h2d_GBps\": %.1f}\n", n * 4 / (now() - t0) / 1e9);
    return 0;
}
