// match.cu -- all-pairs b-bit matching-code counts.
//
// Reference: estimate_bbit counts matching codes for ONE pair
// (estimator.cpp:53-58: sum_j get_code(c1, j, b) == get_code(c2, j, b)).
// Near-duplicate detection needs it for every pair of two sketch sets, which
// is a GEMM-shaped all-pairs loop with a compare-and-count inner product:
//   1. unpack: packed b-bit codes -> fixed-width lanes in 32-bit words
//      (b = 1: the bitstream itself; b <= 8: bytes; b <= 16: halfwords; else
//      words); padding lanes are zero in every row, so they never mismatch;
//   2. match: 64x64-pair CTA tiles, each thread a 4x4 register tile; word
//      tiles of both operands staged in shared memory; per word pair
//      x = a ^ b and the number of non-zero lanes is counted (POPC of the
//      per-lane "non-zero" flags). matches = k - sum(non-zero lanes).
// Integer-exact; the Theorem-1 correction is applied on the host
// (estimate.cpp) from these counts.
#include <cuda_runtime.h>

#include <algorithm>

#include "engine.hpp"
#include "estimate.hpp"

namespace bbmh {

namespace {

constexpr int kTileM = 64, kTileN = 64, kTileW = 32;  // pairs per CTA, words per stage

inline uint32_t lane_width(uint32_t b) { return b == 1 ? 1 : b <= 8 ? 8 : b <= 16 ? 16 : 32; }

__global__ void unpack_kernel(const uint8_t* __restrict__ codes, uint64_t n, uint32_t k,
                              uint32_t b, uint32_t W, uint32_t words,
                              uint32_t* __restrict__ out) {
    const uint64_t cb = ((uint64_t)k * b + 7) >> 3;
    const uint32_t L = 32 / W;
    const uint64_t total = n * words;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = i / words;
        const uint32_t w = (uint32_t)(i % words);
        const uint8_t* c = codes + r * cb;
        uint32_t v = 0;
        for (uint32_t l = 0; l < L; ++l) {
            const uint32_t j = w * L + l;
            if (j >= k) break;
            const uint64_t bit = (uint64_t)j * b;
            const uint8_t* p = c + (bit >> 3);
            const uint32_t sh = (uint32_t)(bit & 7), nb = (sh + b + 7) >> 3;
            uint64_t x = 0;
            for (uint32_t q = 0; q < nb; ++q) x |= (uint64_t)p[q] << (8 * q);
            x >>= sh;
            const uint32_t code = b >= 32 ? (uint32_t)x : (uint32_t)(x & ((1ull << b) - 1));
            v |= W == 32 ? code : code << (l * W);
        }
        out[i] = v;
    }
}

template <int W>
__device__ __forceinline__ uint32_t nonzero_lanes(uint32_t x) {
    if constexpr (W == 1) {
        return __popc(x);
    } else if constexpr (W == 8) {
        const uint32_t t = ((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x;
        return __popc(t & 0x80808080u);
    } else if constexpr (W == 16) {
        const uint32_t t = ((x & 0x7fff7fffu) + 0x7fff7fffu) | x;
        return __popc(t & 0x80008000u);
    } else {
        return x != 0;
    }
}

template <int W>
__global__ void __launch_bounds__(256) match_kernel(const uint32_t* __restrict__ A, uint64_t na,
                                                    const uint32_t* __restrict__ Bm, uint64_t nb,
                                                    uint32_t words, uint32_t k,
                                                    uint32_t* __restrict__ counts) {
    __shared__ uint32_t sa[kTileW][kTileM + 1];
    __shared__ uint32_t sb[kTileW][kTileN + 1];
    const uint32_t tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const uint64_t a0 = (uint64_t)blockIdx.y * kTileM, b0 = (uint64_t)blockIdx.x * kTileN;
    uint32_t acc[4][4] = {};
    for (uint32_t w0 = 0; w0 < words; w0 += kTileW) {
        for (uint32_t i = threadIdx.x; i < kTileW * kTileM; i += 256) {
            const uint32_t r = i / kTileW, w = i % kTileW;  // consecutive threads: consecutive words
            const uint64_t ra = a0 + r, rb = b0 + r;
            sa[w][r] = (ra < na && w0 + w < words) ? A[ra * words + w0 + w] : 0u;
            sb[w][r] = (rb < nb && w0 + w < words) ? Bm[rb * words + w0 + w] : 0u;
        }
        __syncthreads();
#pragma unroll 4
        for (uint32_t w = 0; w < kTileW; ++w) {
            uint32_t av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                av[i] = sa[w][ty + 16 * i];
                bv[i] = sb[w][tx + 16 * i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += nonzero_lanes<W>(av[i] ^ bv[j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint64_t ra = a0 + ty + 16 * i;
        if (ra >= na) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t rb = b0 + tx + 16 * j;
            if (rb < nb) counts[ra * nb + rb] = k - acc[i][j];
        }
    }
}

void unpack(const uint8_t* d_codes, uint64_t n, uint32_t k, uint32_t b, uint32_t words,
            uint32_t* d_out, cudaStream_t st) {
    if (n == 0) return;
    const uint64_t total = n * words;
    const unsigned grid = (unsigned)std::min<uint64_t>((total + 255) / 256, 148 * 32);
    unpack_kernel<<<grid, 256, 0, st>>>(d_codes, n, k, b, lane_width(b), words, d_out);
    count_launches(1);
}

}  // namespace

void match_counts_device(const uint8_t* d_codes_a, uint64_t na, const uint8_t* d_codes_b,
                         uint64_t nb, uint32_t k, uint32_t b, uint32_t* d_counts,
                         cudaStream_t st) {
    if (na == 0 || nb == 0) return;
    const uint32_t W = lane_width(b), L = 32 / W;
    const uint32_t words = (k + L - 1) / L;
    uint32_t *ua = nullptr, *ub = nullptr;
    BBMH_CUDA(cudaMallocAsync(&ua, na * words * sizeof(uint32_t), st));
    BBMH_CUDA(cudaMallocAsync(&ub, nb * words * sizeof(uint32_t), st));
    unpack(d_codes_a, na, k, b, words, ua, st);
    unpack(d_codes_b, nb, k, b, words, ub, st);
    // grid.y covers A tiles (<= 65535 per launch); slice A if needed
    const uint64_t max_rows = 65535ull * kTileM;
    for (uint64_t r0 = 0; r0 < na; r0 += max_rows) {
        const uint64_t nr = std::min(max_rows, na - r0);
        dim3 grid((unsigned)((nb + kTileN - 1) / kTileN), (unsigned)((nr + kTileM - 1) / kTileM));
        const uint32_t* A = ua + r0 * words;
        uint32_t* C = d_counts + r0 * nb;
        switch (W) {
            case 1: match_kernel<1><<<grid, 256, 0, st>>>(A, nr, ub, nb, words, k, C); break;
            case 8: match_kernel<8><<<grid, 256, 0, st>>>(A, nr, ub, nb, words, k, C); break;
            case 16: match_kernel<16><<<grid, 256, 0, st>>>(A, nr, ub, nb, words, k, C); break;
            default: match_kernel<32><<<grid, 256, 0, st>>>(A, nr, ub, nb, words, k, C); break;
        }
        count_launches(1);
    }
    BBMH_CUDA(cudaGetLastError());
    BBMH_CUDA(cudaFreeAsync(ua, st));
    BBMH_CUDA(cudaFreeAsync(ub, st));
}

void match_counts_host(const uint8_t* codes_a, uint64_t na, const uint8_t* codes_b, uint64_t nb,
                       uint32_t k, uint32_t b, uint32_t* counts) {
    if (na == 0 || nb == 0) return;
    const size_t cb = packed_code_bytes(k, b);
    cudaStream_t st;
    BBMH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct Guard {
        cudaStream_t s;
        ~Guard() { cudaStreamDestroy(s); }
    } g{st};
    uint8_t *da = nullptr, *db = nullptr;
    uint32_t* dc = nullptr;
    BBMH_CUDA(cudaMallocAsync(&da, std::max<size_t>(na * cb, 1), st));
    BBMH_CUDA(cudaMallocAsync(&db, std::max<size_t>(nb * cb, 1), st));
    BBMH_CUDA(cudaMallocAsync(&dc, na * nb * sizeof(uint32_t), st));
    BBMH_CUDA(cudaMemcpyAsync(da, codes_a, na * cb, cudaMemcpyHostToDevice, st));
    BBMH_CUDA(cudaMemcpyAsync(db, codes_b, nb * cb, cudaMemcpyHostToDevice, st));
    match_counts_device(da, na, db, nb, k, b, dc, st);
    BBMH_CUDA(cudaMemcpyAsync(counts, dc, na * nb * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    BBMH_CUDA(cudaFreeAsync(da, st));
    BBMH_CUDA(cudaFreeAsync(db, st));
    BBMH_CUDA(cudaFreeAsync(dc, st));
    BBMH_CUDA(cudaStreamSynchronize(st));
}

}  // namespace bbmh
