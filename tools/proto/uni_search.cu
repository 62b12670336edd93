// uni_variants.cu -- developer experiment (not part of libbbmh): source-level
// variants of the coefficient-uniform 2U hash loop (uniform.cu layout: a warp
// per (document, group of 32 functions), lanes over ids, the multiplier a
// constant-bank operand), timed on a webspam-shaped corpus (350,000 x 3,728
// ids, D = 2^24) with k = 64 (two groups, so the instruction cache holds both
// bodies), checked against a plain per-(doc, function) kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o uni_variants uni_variants.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace {
constexpr int kG = 32;
constexpr int kGroups = 2;
constexpr int kK = kG * kGroups;
struct Coef {
    uint32_t a2[kK];
    uint32_t a1[kK];
};

__device__ __forceinline__ uint32_t min3u(uint32_t a, uint32_t b, uint32_t c) { return min(min(a, b), c); }

template <int VAR>
__device__ __forceinline__ void hash8(const Coef& C, int S, uint32_t (&m)[kG], const uint32_t (&a1)[kG],
                                      const uint4& x, const uint4& y);

template <int S, int VAR>
__device__ __forceinline__ void step8(const Coef& C, uint32_t (&m)[kG], const uint32_t (&a1)[kG], const uint4& x,
                                      const uint4& y) {
#pragma unroll
    for (int r = 0; r < kG; ++r) {
        const uint32_t a2 = C.a2[S * kG + r];
        if constexpr (VAR == 0) {  // shipped: chain of min3(m, h, h)
            m[r] = min3u(m[r], a1[r] + a2 * x.x, a1[r] + a2 * x.y);
            m[r] = min3u(m[r], a1[r] + a2 * x.z, a1[r] + a2 * x.w);
            m[r] = min3u(m[r], a1[r] + a2 * y.x, a1[r] + a2 * y.y);
            m[r] = min3u(m[r], a1[r] + a2 * y.z, a1[r] + a2 * y.w);
        } else if constexpr (VAR == 1) {  // tree: 3 fresh, 3 fresh, then m
            const uint32_t p = min3u(a1[r] + a2 * x.x, a1[r] + a2 * x.y, a1[r] + a2 * x.z);
            const uint32_t q = min3u(a1[r] + a2 * x.w, a1[r] + a2 * y.x, a1[r] + a2 * y.y);
            const uint32_t s = min3u(m[r], a1[r] + a2 * y.z, a1[r] + a2 * y.w);
            m[r] = min3u(p, q, s);
        } else if constexpr (VAR == 2) {  // multiplier as the first operand
            m[r] = min3u(m[r], a2 * x.x + a1[r], a2 * x.y + a1[r]);
            m[r] = min3u(m[r], a2 * x.z + a1[r], a2 * x.w + a1[r]);
            m[r] = min3u(m[r], a2 * y.x + a1[r], a2 * y.y + a1[r]);
            m[r] = min3u(m[r], a2 * y.z + a1[r], a2 * y.w + a1[r]);
        } else if constexpr (VAR == 3) {  // two independent chains per function
            uint32_t u = min3u(m[r], a1[r] + a2 * x.x, a1[r] + a2 * x.y);
            uint32_t v = min3u(a1[r] + a2 * y.x, a1[r] + a2 * y.y, a1[r] + a2 * x.z);
            u = min3u(u, a1[r] + a2 * x.w, a1[r] + a2 * y.z);
            m[r] = min3u(u, v, a1[r] + a2 * y.w);

        } else if constexpr (VAR == 4) {
  // m last
            m[r] = min3u(a1[r] + a2 * x.x, a1[r] + a2 * x.y, m[r]);
            m[r] = min3u(a1[r] + a2 * x.z, a1[r] + a2 * x.w, m[r]);
            m[r] = min3u(a1[r] + a2 * y.x, a1[r] + a2 * y.y, m[r]);
            m[r] = min3u(a1[r] + a2 * y.z, a1[r] + a2 * y.w, m[r]);
        } else if constexpr (VAR == 100) {
            const uint32_t t0 = min3u((a1[r] + a2 * y.x), (a1[r] + a2 * x.x), (a1[r] + a2 * x.z));
            const uint32_t t1 = min3u((a1[r] + a2 * x.w), m[r], (a1[r] + a2 * x.y));
            const uint32_t t2 = min3u((a1[r] + a2 * y.z), t0, (a1[r] + a2 * y.y));
            m[r] = min3u(t2, (a1[r] + a2 * y.w), t1);
        } else if constexpr (VAR == 101) {
            const uint32_t t0 = min3u(m[r], (a1[r] + a2 * y.x), (a1[r] + a2 * y.w));
            const uint32_t t1 = min3u((a1[r] + a2 * x.y), (a1[r] + a2 * x.z), (a1[r] + a2 * x.x));
            const uint32_t t2 = min3u((a1[r] + a2 * y.z), t0, (a1[r] + a2 * y.y));
            m[r] = min3u((a1[r] + a2 * x.w), t2, t1);
        } else if constexpr (VAR == 102) {
            const uint32_t t0 = min3u((a1[r] + a2 * y.x), (a1[r] + a2 * y.y), m[r]);
            const uint32_t t1 = min3u((a1[r] + a2 * x.z), (a1[r] + a2 * x.y), (a1[r] + a2 * x.w));
            const uint32_t t2 = min3u((a1[r] + a2 * y.z), (a1[r] + a2 * y.w), (a1[r] + a2 * x.x));
            m[r] = min3u(t2, t1, t0);
        } else if constexpr (VAR == 103) {
            const uint32_t t0 = min3u(m[r], (a1[r] + a2 * x.z), (a1[r] + a2 * x.x));
            const uint32_t t1 = min3u((a1[r] + a2 * x.w), (a1[r] + a2 * y.x), t0);
            const uint32_t t2 = min3u((a1[r] + a2 * y.y), (a1[r] + a2 * y.w), (a1[r] + a2 * y.z));
            m[r] = min3u(t2, t1, (a1[r] + a2 * x.y));
        } else if constexpr (VAR == 104) {
            const uint32_t t0 = min3u((a1[r] + a2 * x.x), (a1[r] + a2 * y.y), (a1[r] + a2 * y.w));
            const uint32_t t1 = min3u(m[r], (a1[r] + a2 * x.z), t0);
            const uint32_t t2 = min3u((a1[r] + a2 * x.y), (a1[r] + a2 * y.x), t1);
            m[r] = min3u((a1[r] + a2 * y.z), t2, (a1[r] + a2 * x.w));
        } else if constexpr (VAR == 105) {
            const uint32_t t0 = min3u((a1[r] + a2 * y.x), (a1[r] + a2 * y.z), (a1[r] + a2 * x.z));
            const uint32_t t1 = min3u((a1[r] + a2 * x.x), (a1[r] + a2 * x.y), t0);
            const uint32_t t2 = min3u(m[r], (a1[r] + a2 * y.y), (a1[r] + a2 * x.w));
            m[r] = min3u(t2, (a1[r] + a2 * y.w), t1);
        } else if constexpr (VAR == 106) {
            const uint32_t t0 = min3u((a1[r] + a2 * x.x), (a1[r] + a2 * x.z), (a1[r] + a2 * y.x));
            const uint32_t t1 = min3u((a1[r] + a2 * y.y), m[r], (a1[r] + a2 * x.w));
            const uint32_t t2 = min3u(t1, (a1[r] + a2 * y.z), (a1[r] + a2 * x.y));
            m[r] = min3u(t2, (a1[r] + a2 * y.w), t0);
        } else if constexpr (VAR == 107) {
            const uint32_t t0 = min3u(m[r], (a1[r] + a2 * x.w), (a1[r] + a2 * x.z));
            const uint32_t t1 = min3u(t0, (a1[r] + a2 * y.y), (a1[r] + a2 * x.y));
            const uint32_t t2 = min3u((a1[r] + a2 * y.w), (a1[r] + a2 * y.z), t1);
            m[r] = min3u((a1[r] + a2 * y.x), (a1[r] + a2 * x.x), t2);
        } else if constexpr (VAR == 108) {
            const uint32_t t0 = min3u((a1[r] + a2 * y.x), (a1[r] + a2 * y.y), (a1[r] + a2 * x.w));
            const uint32_t t1 = min3u((a1[r] + a2 * x.z), (a1[r] + a2 * y.w), (a1[r] + a2 * x.y));
            const uint32_t t2 = min3u(t0, m[r], t1);
            m[r] = min3u((a1[r] + a2 * x.x), t2, (a1[r] + a2 * y.z));
        } else if constexpr (VAR == 109) {
            const uint32_t t0 = min3u((a1[r] + a2 * x.y), m[r], (a1[r] + a2 * y.x));
            const uint32_t t1 = min3u((a1[r] + a2 * x.w), (a1[r] + a2 * x.z), (a1[r] + a2 * y.y));
            const uint32_t t2 = min3u((a1[r] + a2 * x.x), (a1[r] + a2 * y.w), t0);
            m[r] = min3u(t2, t1, (a1[r] + a2 * y.z));
        } else if constexpr (VAR == 110) {
            const uint32_t t0 = min3u((a1[r] + a2 * y.x), m[r], (a1[r] + a2 * x.x));
            const uint32_t t1 = min3u((a1[r] + a2 * x.z), (a1[r] + a2 * y.z), (a1[r] + a2 * y.w));
            const uint32_t t2 = min3u((a1[r] + a2 * y.y), (a1[r] + a2 * x.y), t1);
            m[r] = min3u((a1[r] + a2 * x.w), t0, t2);
        } else if constexpr (VAR == 111) {
            const uint32_t t0 = min3u((a1[r] + a2 * x.x), (a1[r] + a2 * x.w), (a1[r] + a2 * y.z));
            const uint32_t t1 = min3u(t0, (a1[r] + a2 * x.z), (a1[r] + a2 * y.x));
            const uint32_t t2 = min3u(t1, m[r], (a1[r] + a2 * y.y));
            m[r] = min3u((a1[r] + a2 * x.y), (a1[r] + a2 * y.w), t2);
        } else if constexpr (VAR == 112) {
            const uint32_t t0 = min3u((a1[r] + a2 * y.y), (a1[r] + a2 * x.y), (a1[r] + a2 * y.x));
            const uint32_t t1 = min3u((a1[r] + a2 * y.z), m[r], (a1[r] + a2 * x.x));
            const uint32_t t2 = min3u(t1, t0, (a1[r] + a2 * y.w));
            m[r] = min3u((a1[r] + a2 * x.z), t2, (a1[r] + a2 * x.w));
        } else if constexpr (VAR == 113) {
            const uint32_t t0 = min3u((a1[r] + a2 * x.z), (a1[r] + a2 * x.w), (a1[r] + a2 * y.x));
            const uint32_t t1 = min3u((a1[r] + a2 * x.y), (a1[r] + a2 * y.z), (a1[r] + a2 * y.w));
            const uint32_t t2 = min3u(t1, t0, (a1[r] + a2 * y.y));
            m[r] = min3u(m[r], t2, (a1[r] + a2 * x.x));
        } else if constexpr (VAR == 114) {
            const uint32_t t0 = min3u((a1[r] + a2 * x.y), (a1[r] + a2 * y.x), (a1[r] + a2 * x.z));
            const uint32_t t1 = min3u((a1[r] + a2 * x.w), t0, m[r]);
            const uint32_t t2 = min3u((a1[r] + a2 * y.z), (a1[r] + a2 * y.y), t1);
            m[r] = min3u(t2, (a1[r] + a2 * y.w), (a1[r] + a2 * x.x));
        } else if constexpr (VAR == 115) {
            const uint32_t t0 = min3u((a1[r] + a2 * y.x), (a1[r] + a2 * x.w), m[r]);
            const uint32_t t1 = min3u((a1[r] + a2 * x.z), t0, (a1[r] + a2 * x.x));
            const uint32_t t2 = min3u((a1[r] + a2 * y.z), (a1[r] + a2 * y.w), (a1[r] + a2 * y.y));
            m[r] = min3u((a1[r] + a2 * x.y), t1, t2);
        } else if constexpr (VAR == 116) {
            const uint32_t t0 = min3u(m[r], (a1[r] + a2 * x.w), (a1[r] + a2 * y.x));
            const uint32_t t1 = min3u((a1[r] + a2 * y.z), (a1[r] + a2 * y.w), (a1[r] + a2 * x.z));
            const uint32_t t2 = min3u((a1[r] + a2 * y.y), t0, t1);
            m[r] = min3u((a1[r] + a2 * x.y), t2, (a1[r] + a2 * x.x));
        } else if constexpr (VAR == 117) {
            const uint32_t t0 = min3u((a1[r] + a2 * y.y), (a1[r] + a2 * y.x), (a1[r] + a2 * x.z));
            const uint32_t t1 = min3u((a1[r] + a2 * x.x), (a1[r] + a2 * x.y), (a1[r] + a2 * x.w));
            const uint32_t t2 = min3u(t1, (a1[r] + a2 * y.z), t0);
            m[r] = min3u((a1[r] + a2 * y.w), t2, m[r]);
        } else if constexpr (VAR == 118) {
            const uint32_t t0 = min3u((a1[r] + a2 * x.x), (a1[r] + a2 * y.y), (a1[r] + a2 * y.w));
            const uint32_t t1 = min3u((a1[r] + a2 * x.y), (a1[r] + a2 * y.x), m[r]);
            const uint32_t t2 = min3u((a1[r] + a2 * y.z), (a1[r] + a2 * x.w), t0);
            m[r] = min3u(t1, (a1[r] + a2 * x.z), t2);
        } else if constexpr (VAR == 119) {
            const uint32_t t0 = min3u((a1[r] + a2 * y.w), (a1[r] + a2 * x.y), (a1[r] + a2 * x.w));
            const uint32_t t1 = min3u((a1[r] + a2 * x.x), (a1[r] + a2 * x.z), t0);
            const uint32_t t2 = min3u((a1[r] + a2 * y.y), (a1[r] + a2 * y.x), m[r]);
            m[r] = min3u(t1, (a1[r] + a2 * y.z), t2);
        } else if constexpr (VAR == 120) {
            const uint32_t t0 = min3u(m[r], (a1[r] + a2 * x.z), (a1[r] + a2 * x.x));
            const uint32_t t1 = min3u((a1[r] + a2 * y.w), (a1[r] + a2 * y.y), t0);
            const uint32_t t2 = min3u((a1[r] + a2 * x.w), (a1[r] + a2 * y.x), (a1[r] + a2 * y.z));
            m[r] = min3u(t2, (a1[r] + a2 * x.y), t1);
        } else if constexpr (VAR == 121) {
            const uint32_t t0 = min3u((a1[r] + a2 * x.z), m[r], (a1[r] + a2 * y.w));
            const uint32_t t1 = min3u((a1[r] + a2 * y.x), (a1[r] + a2 * y.z), (a1[r] + a2 * x.w));
            const uint32_t t2 = min3u(t0, t1, (a1[r] + a2 * y.y));
            m[r] = min3u((a1[r] + a2 * x.y), (a1[r] + a2 * x.x), t2);
        } else if constexpr (VAR == 122) {
            const uint32_t t0 = min3u((a1[r] + a2 * x.z), (a1[r] + a2 * y.w), (a1[r] + a2 * x.w));
            const uint32_t t1 = min3u((a1[r] + a2 * x.x), t0, (a1[r] + a2 * y.z));
            const uint32_t t2 = min3u(m[r], (a1[r] + a2 * y.y), (a1[r] + a2 * x.y));
            m[r] = min3u(t2, (a1[r] + a2 * y.x), t1);
        } else if constexpr (VAR == 123) {
            const uint32_t t0 = min3u((a1[r] + a2 * x.x), (a1[r] + a2 * y.y), (a1[r] + a2 * x.y));
            const uint32_t t1 = min3u((a1[r] + a2 * y.w), t0, (a1[r] + a2 * x.w));
            const uint32_t t2 = min3u((a1[r] + a2 * x.z), (a1[r] + a2 * y.x), t1);
            m[r] = min3u((a1[r] + a2 * y.z), m[r], t2);
        }
    }
}

template <int S, int VAR, bool PF>
__device__ __forceinline__ void item(const Coef& C, const uint64_t* rp, const uint32_t* idx, uint32_t d,
                                     uint32_t lane, uint32_t* out) {
    const uint64_t beg = rp[d], end = rp[d + 1];
    const uint4* q4 = reinterpret_cast<const uint4*>(idx + beg);
    const uint64_t nq = (end - beg) >> 2;  // corpus rows are whole, aligned quads
    uint32_t m[kG], a1[kG];
#pragma unroll
    for (int r = 0; r < kG; ++r) {
        m[r] = 0xffffffffu;
        a1[r] = C.a1[S * kG + r];
    }
    if constexpr (PF) {
        uint4 x = __ldg(q4 + min((uint64_t)lane, nq - 1)), y = __ldg(q4 + min((uint64_t)lane + 32, nq - 1));
        for (uint64_t s = 0; s < nq; s += 64) {
            const uint4 xc = x, yc = y;
            if (s + 64 < nq) {
                x = __ldg(q4 + min(s + 64 + lane, nq - 1));
                y = __ldg(q4 + min(s + 96 + lane, nq - 1));
            }
            step8<S, VAR>(C, m, a1, xc, yc);
        }
    } else {
        for (uint64_t s = 0; s < nq; s += 64) {
            const uint4 x = __ldg(q4 + min(s + lane, nq - 1)), y = __ldg(q4 + min(s + 32 + lane, nq - 1));
            step8<S, VAR>(C, m, a1, x, y);
        }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool up = lane & off;
#pragma unroll
        for (int q = 0; q < off; ++q) {
            const uint32_t send = up ? m[q] : m[q + off];
            const uint32_t keep = up ? m[q + off] : m[q];
            m[q] = min(keep, __shfl_xor_sync(0xffffffffu, send, off));
        }
    }
    out[(uint64_t)d * kK + S * kG + lane] = m[0];
}

template <int VAR, bool PF, int TPB>
__global__ void __launch_bounds__(TPB) uni_kernel(const __grid_constant__ Coef C, const uint64_t* __restrict__ rp,
                                                  const uint32_t* __restrict__ idx, uint32_t n,
                                                  uint32_t* __restrict__ out, unsigned long long* work) {
    const uint32_t lane = threadIdx.x & 31, W = TPB / 32;
    const uint32_t items = n * kGroups, stride = gridDim.x * W;
    auto next = [&](uint32_t cur) -> uint32_t {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(&work[0], 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        return t >= items ? items : (uint32_t)(stride + t);
    };
    uint32_t it = blockIdx.x * W + (threadIdx.x >> 5);
    uint32_t nx = it < items ? next(it) : items;
    for (; it < items; it = nx, nx = it < items ? next(it) : items) {
        const uint32_t g = it & 1, d = it >> 1;
        if (g == 0)
            item<0, VAR, PF>(C, rp, idx, d, lane, out);
        else
            item<1, VAR, PF>(C, rp, idx, d, lane, out);
    }
}

__global__ void ref_kernel(const uint32_t* a1, const uint32_t* a2, const uint64_t* rp, const uint32_t* idx,
                           uint32_t n, uint32_t* out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (uint64_t)n * kK) return;
    const uint32_t d = t / kK, j = t % kK;
    uint32_t m = 0xffffffffu;
    for (uint64_t i = rp[d]; i < rp[d + 1]; ++i) m = min(m, a1[j] + a2[j] * idx[i]);
    out[t] = m;
}

__global__ void gen_kernel(uint32_t* idx, uint64_t total, uint32_t seed) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = (i + 1) * 0x9e3779b97f4a7c15ull ^ seed;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        idx[i] = (uint32_t)(z ^ (z >> 31)) & 0xffffffu;
    }
}

template <int VAR, bool PF, int TPB>
void run(const char* name, const Coef& C, const uint64_t* rp, const uint32_t* idx, uint32_t n, uint32_t* out,
         const std::vector<uint32_t>& ref, unsigned long long* work, uint64_t nnz) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, uni_kernel<VAR, PF, TPB>, TPB, 0);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, uni_kernel<VAR, PF, TPB>);
    const int grid = 148 * occ;
    cudaMemset(out, 0, (size_t)n * kK * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaMemset(work, 0, 16);
        cudaEventRecord(e0);
        uni_kernel<VAR, PF, TPB><<<grid, TPB>>>(C, rp, idx, n, out, work);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    std::vector<uint32_t> h((size_t)n * kK);
    cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (size_t i = 0; i < ref.size(); ++i) bad += h[i] != ref[i];
    const double evals = (double)nnz * kK;
    printf("{\"variant\": \"%s\", \"tpb\": %d, \"regs\": %d, \"occ\": %d, \"ms\": %.3f, \"tevals\": %.3f, "
           "\"frac_contract\": %.4f, \"mismatch\": %zu}\n",
           name, TPB, fa.numRegs, occ, best, evals / best / 1e9, evals / best / 1e9 / 18.61248, bad);
    fflush(stdout);
}
}  // namespace

int main() {
    const uint32_t n = 350000, nnz = 3728;
    const uint64_t total = (uint64_t)n * nnz;
    uint32_t* idx;
    uint64_t* rp;
    uint32_t* out;
    unsigned long long* work;
    cudaMalloc(&idx, total * 4 + 16);
    cudaMalloc(&rp, (n + 1) * 8);
    cudaMalloc(&out, (size_t)n * kK * 4);
    cudaMalloc(&work, 16);
    gen_kernel<<<1024, 256>>>(idx, total, 7);
    std::vector<uint64_t> hrp(n + 1);
    for (uint32_t i = 0; i <= n; ++i) hrp[i] = (uint64_t)i * nnz;
    cudaMemcpy(rp, hrp.data(), hrp.size() * 8, cudaMemcpyHostToDevice);
    Coef C;
    std::vector<uint32_t> a1(kK), a2(kK);
    uint64_t s = 12345;
    for (int j = 0; j < kK; ++j) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        a1[j] = C.a1[j] = (uint32_t)(s >> 32);
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        a2[j] = C.a2[j] = (uint32_t)(s >> 32) | 1u;
    }
    uint32_t *da1, *da2;
    cudaMalloc(&da1, kK * 4);
    cudaMalloc(&da2, kK * 4);
    cudaMemcpy(da1, a1.data(), kK * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(da2, a2.data(), kK * 4, cudaMemcpyHostToDevice);
    const uint32_t nref = 20000;  // reference over the first documents
    ref_kernel<<<(unsigned)(((uint64_t)nref * kK + 255) / 256), 256>>>(da1, da2, rp, idx, nref, out);
    std::vector<uint32_t> ref((size_t)nref * kK);
    cudaMemcpy(ref.data(), out, ref.size() * 4, cudaMemcpyDeviceToHost);
    run<0, true, 128>("chain", C, rp, idx, n, out, ref, work, total);
    run<3, true, 128>("two_chains", C, rp, idx, n, out, ref, work, total);
    run<100, true, 128>("v100", C, rp, idx, n, out, ref, work, total);
    run<101, true, 128>("v101", C, rp, idx, n, out, ref, work, total);
    run<102, true, 128>("v102", C, rp, idx, n, out, ref, work, total);
    run<103, true, 128>("v103", C, rp, idx, n, out, ref, work, total);
    run<104, true, 128>("v104", C, rp, idx, n, out, ref, work, total);
    run<105, true, 128>("v105", C, rp, idx, n, out, ref, work, total);
    run<106, true, 128>("v106", C, rp, idx, n, out, ref, work, total);
    run<107, true, 128>("v107", C, rp, idx, n, out, ref, work, total);
    run<108, true, 128>("v108", C, rp, idx, n, out, ref, work, total);
    run<109, true, 128>("v109", C, rp, idx, n, out, ref, work, total);
    run<110, true, 128>("v110", C, rp, idx, n, out, ref, work, total);
    run<111, true, 128>("v111", C, rp, idx, n, out, ref, work, total);
    run<112, true, 128>("v112", C, rp, idx, n, out, ref, work, total);
    run<113, true, 128>("v113", C, rp, idx, n, out, ref, work, total);
    run<114, true, 128>("v114", C, rp, idx, n, out, ref, work, total);
    run<115, true, 128>("v115", C, rp, idx, n, out, ref, work, total);
    run<116, true, 128>("v116", C, rp, idx, n, out, ref, work, total);
    run<117, true, 128>("v117", C, rp, idx, n, out, ref, work, total);
    run<118, true, 128>("v118", C, rp, idx, n, out, ref, work, total);
    run<119, true, 128>("v119", C, rp, idx, n, out, ref, work, total);
    run<120, true, 128>("v120", C, rp, idx, n, out, ref, work, total);
    run<121, true, 128>("v121", C, rp, idx, n, out, ref, work, total);
    run<122, true, 128>("v122", C, rp, idx, n, out, ref, work, total);
    run<123, true, 128>("v123", C, rp, idx, n, out, ref, work, total);
    run<3, true, 128>("two_chains", C, rp, idx, n, out, ref, work, total);
    printf("{\"cuda: \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
