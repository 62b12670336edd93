// score.cu -- fused test-time scoring of freshly sketched rows.
//
// Reference: prediction on a BBMH sketch expands each record at run time
// (SketchRowSource, learner.cpp:271-297; expand, expansion.cpp:17-27) and
// scores it with predict_score (learner.cpp:510-521):
//     score = sum_{j ascending} w[j * 2^b + code_j]      (double, in j order)
// empty rows score 0.0 (predict_file, learner.cpp:528); an index >= the
// model dimension is DimensionExceeded "feature <idx> >= dim <dim>".
//
// Here the codes never leave the device: right after the sketch kernel, one
// thread per row decodes its packed codes (sketch.cpp:55-62) and accumulates
// the k weights in exactly the reference's order, so scores are bit-identical
// doubles. The row's k gathers are independent and issued ahead of the
// dependent adds; w (k * 2^b doubles, 1 MiB at k = 500, b = 8) stays in L2.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace bbmh {

namespace {

__device__ __forceinline__ uint32_t get_code_packed(const uint8_t* codes, uint32_t j, uint32_t b) {
    const uint64_t bit = (uint64_t)j * b;
    const uint8_t* p = codes + (bit >> 3);
    const uint32_t sh = (uint32_t)(bit & 7);
    const uint32_t nbytes = (sh + b + 7) >> 3;  // <= 5
    uint64_t v = 0;
    for (uint32_t i = 0; i < nbytes; ++i) v |= (uint64_t)p[i] << (8 * i);
    v >>= sh;
    return b >= 32 ? (uint32_t)v : (uint32_t)(v & ((1ull << b) - 1));
}

__global__ void __launch_bounds__(128) score_kernel(const uint8_t* __restrict__ codes,
                                                    const uint8_t* __restrict__ flags, uint64_t n,
                                                    uint32_t k, uint32_t b,
                                                    const double* __restrict__ w, uint64_t wdim,
                                                    double* __restrict__ scores,
                                                    unsigned long long* bad) {
    const uint64_t cb = ((uint64_t)k * b + 7) >> 3;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        if (flags[r] & 1) {  // empty set -> empty row -> score 0
            scores[r] = 0.0;
            continue;
        }
        const uint8_t* c = codes + r * cb;
        double s = 0.0;
        for (uint32_t j = 0; j < k; ++j) {
            // ones[j] = uint32(2^b * j + code_j) (expansion.cpp:25-26)
            const uint32_t idx = (uint32_t)(((uint64_t)j << b) + get_code_packed(c, j, b));
            if ((uint64_t)idx >= wdim) {
                // remember the first offending (row, j) in row-major order
                atomicMin(bad, (unsigned long long)(r << 24 | (j & 0xffffffu)));
                break;
            }
            s += w[idx];
        }
        scores[r] = s;
    }
}

}  // namespace

void launch_score(const uint8_t* codes, const uint8_t* flags, uint64_t n, uint32_t k, uint32_t b,
                  const double* w, uint64_t wdim, double* scores, unsigned long long* bad,
                  cudaStream_t st) {
    if (n == 0) return;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (n + 127) / 128;
    const unsigned grid = (unsigned)(want < (uint64_t)sms * 16 ? want : (uint64_t)sms * 16);
    score_kernel<<<grid, 128, 0, st>>>(codes, flags, n, k, b, w, wdim, scores, bad);
    count_launches(1);
}

}  // namespace bbmh
