// ring_probe.cpp -- encode + H2D of sorted id rows in pieces through a ring of page-locked
// buffers, non-temporal vs regular stores, by piece size: does the DMA read
// freshly written (cache-resident) pieces faster than streamed ones? Input GB/s.
//   nvcc -O3 -std=c++20 -I paper_1205_2958_b200/csrc -o /tmp/ring_probe tools/ring_probe.cpp paper_1205_2958_b200/csrc/hostpool.cpp
#include <cuda_runtime.h>
#include <immintrin.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>
#include "hostpool.hpp"
using namespace bbmh;
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
__attribute__((target("avx2"))) static void enc(const uint32_t* s, uint16_t* o, uint64_t lo, uint64_t hi, bool nt) {
    const __m256i hm = _mm256_set1_epi32(int(0xffff0000u));
    uint64_t i = lo;
    for (; i < hi && ((i & 7) || i == 0); ++i) o[i] = uint16_t(s[i] - (i ? s[i - 1] : 0));
    for (; i + 8 <= hi; i += 8) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        const __m256i p = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i - 1));
        __m256i d = _mm256_sub_epi32(a, p);
        const __m256i big = _mm256_xor_si256(_mm256_cmpeq_epi32(_mm256_and_si256(d, hm), _mm256_setzero_si256()), _mm256_set1_epi32(-1));
        d = _mm256_andnot_si256(big, d);
        const __m256i pk = _mm256_packus_epi32(d, d);
        const __m128i v = _mm256_castsi256_si128(_mm256_permute4x64_epi64(pk, 0x08));
        if (nt) _mm_stream_si128(reinterpret_cast<__m128i*>(o + i), v); else _mm_storeu_si128(reinterpret_cast<__m128i*>(o + i), v);
    }
    for (; i < hi; ++i) o[i] = uint16_t(s[i] - s[i - 1]);
    if (nt) _mm_sfence();
}
int main() {
    const uint64_t n = uint64_t(1) << 28;
    uint32_t* ids; cudaMallocHost(&ids, n * 4);
    std::mt19937_64 g(1); uint32_t v = 0;
    for (uint64_t i = 0; i < n; ++i) { if (i % 3728 == 0) v = uint32_t(g() % 2000); ids[i] = v; v += 1 + uint32_t(g() % 9000); }
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    uint16_t* dev; cudaMalloc(&dev, n * 2);
    const unsigned T = 4 * host_threads();
    auto par = [&](uint16_t* out, uint64_t lo, uint64_t hi, bool nt) {
        const unsigned TT = std::max<uint64_t>(1, std::min<uint64_t>(T, (hi - lo) >> 14));
        host_parallel(TT, [&](unsigned w) {
            const uint64_t a = (lo + (hi - lo) * w / TT) & ~uint64_t(7), b = w + 1 == TT ? hi : (lo + (hi - lo) * (w + 1) / TT) & ~uint64_t(7);
            enc(ids, out, a, b, nt);
        });
    };
    for (int nt = 1; nt >= 0; --nt)
    for (uint64_t P : {uint64_t(1) << 18, uint64_t(1) << 20, uint64_t(1) << 22, uint64_t(1) << 24}) {
        for (int R : {3, 6}) {
            std::vector<uint16_t*> ring(R); std::vector<cudaEvent_t> ev(R);
            for (int i = 0; i < R; ++i) { cudaMallocHost(&ring[i], P * 2 + 64); cudaEventCreate(&ev[i]); cudaEventRecord(ev[i], st); }
            double best = 0;
            for (int rep = 0; rep < 2; ++rep) {
                const double t0 = now();
                for (uint64_t c = 0, k = 0; c < n; c += P, ++k) {
                    uint16_t* b = ring[k % R];
                    cudaEventSynchronize(ev[k % R]);
                    par(b - c, c, c + P, nt);
                    cudaMemcpyAsync(dev + c, b, P * 2, cudaMemcpyHostToDevice, st);
                    cudaEventRecord(ev[k % R], st);
                }
                cudaStreamSynchronize(st);
                best = std::max(best, n * 4 / (now() - t0) / 1e9);
            }
            std::printf("{\"nt\": %d, \"piece_MB\": %.1f, \"ring\": %d, \"in_GBps\": %.1f}\n", nt, P * 2 / 1e6, R, best);
            for (int i = 0; i < R; ++i) cudaFreeHost(ring[i]);
        }
    }
    return 0;
}
