// permgen.cu -- permutation tables built on the GPU.
//
// Reference: HashFamily::build, permutation branch (hash_family.cpp:105-114):
// per table j, tab[t] = t, then for t = D-1 .. 1 swap tab[t] with
// tab[SplitMix64(keyed_u64(seed, 1, j, 0)).next_below(t + 1)] (prng.hpp:42-61).
// Each shuffle is sequential; on the host it is bound by cache misses into a
// 64 MB table (~0.4 s per table, 19 s for k = 500 on 16 cores). Here one
// thread runs one table's shuffle, in windows of W swaps: the W draws are
// computed and all 2W table entries loaded at once (W loads in flight per
// thread instead of one), then the swaps are applied in order in registers,
// forwarding values written earlier in the window, and stored. The result is
// the same permutation, swap for swap. A draw that would take the rejection
// branch of next_below (probability < 2^-32 per draw) marks its table, which
// is then rebuilt on the host.
#include <cuda_runtime.h>

#include <cstdlib>
#include <vector>

#include "core.hpp"
#include "engine.hpp"
#include "kernels.cuh"

namespace bbmh {

namespace {

constexpr uint64_t kPhi = 0x9e3779b97f4a7c15ull;

__device__ __forceinline__ uint64_t dmix64(uint64_t x) {  // prng.hpp:10-17
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

__global__ void perm_init_kernel(uint32_t* __restrict__ perm, uint64_t dim, uint64_t total) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x)
        perm[i] = uint32_t(i % dim);
}

template <int W>
__global__ void __launch_bounds__(32) perm_shuffle_kernel(uint32_t* __restrict__ perm, uint64_t dim,
                                                         uint32_t k, const uint64_t* __restrict__ seeds,
                                                         uint32_t* __restrict__ host_redo) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    uint32_t* tab = perm + size_t(j) * dim;
    uint64_t state = seeds[j];
    for (uint64_t t0 = dim - 1; t0 > 0;) {
        const int w = t0 < uint64_t(W) ? int(t0) : W;
        uint32_t r[W], A[W], B[W];
#pragma unroll
        for (int i = 0; i < W; ++i) {
            if (i < w) {
                const uint64_t bound = t0 - i + 1;
                state += kPhi;
                const uint64_t v = dmix64(state);
                if ((bound & (bound - 1)) == 0) {
                    r[i] = uint32_t(v & (bound - 1));
                } else {
                    // next_below's rejection: v >= UINT64_MAX - UINT64_MAX % bound,
                    // only possible in the top `bound` values of the range
                    if ((v >> 32) == 0xffffffffull && v >= ~0ull - (~0ull % bound)) {
                        host_redo[j] = 1;
                        return;
                    }
                    r[i] = uint32_t(v % bound);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < W; ++i) {
            if (i < w) {
                A[i] = tab[t0 - i];
                B[i] = tab[r[i]];
            }
        }
        // the window's swaps in order; lp/lv log the writes (later entries win)
        uint32_t lp[2 * W], lv[2 * W];
#pragma unroll
        for (int i = 0; i < W; ++i) {
            if (i < w) {
                const uint32_t t = uint32_t(t0 - i);
                uint32_t vt = A[i], vr = B[i];
#pragma unroll
                for (int q = 0; q < 2 * i; ++q) {
                    vt = lp[q] == t ? lv[q] : vt;
                    vr = lp[q] == r[i] ? lv[q] : vr;
                }
                lp[2 * i] = t;
                lv[2 * i] = vr;
                lp[2 * i + 1] = r[i];
                lv[2 * i + 1] = vt;
            }
        }
#pragma unroll
        for (int q = 0; q < 2 * W; ++q)
            if (q < 2 * w) tab[lp[q]] = lv[q];
        t0 -= uint64_t(w);
    }
}

}  // namespace

bool build_perm_tables_gpu(Family& f) {
    const char* e = std::getenv("BBMH_GPU_PERMGEN");
    if (e && *e == '0') return false;
    const uint64_t dim = f.dim, k = f.k;
    const size_t bytes = size_t(dim) * k * sizeof(uint32_t);
    if (dim < 2 || bytes < (size_t(64) << 20)) return false;  // small: the host is as fast
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return false;
    }
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || bytes + (size_t(1) << 30) > free_b) {
        cudaGetLastError();
        return false;
    }
    uint32_t* d_perm = nullptr;
    uint64_t* d_seeds = nullptr;
    uint32_t* d_redo = nullptr;
    auto cleanup = [&](bool keep_perm) {
        if (d_seeds) cudaFree(d_seeds);
        if (d_redo) cudaFree(d_redo);
        if (!keep_perm && d_perm) cudaFree(d_perm);
        cudaGetLastError();
    };
    std::vector<uint64_t> seeds(k);
    for (uint64_t j = 0; j < k; ++j) seeds[j] = keyed_u64(f.seed, rngtag::kPermutation, j, 0);
    if (cudaMalloc(&d_perm, bytes) != cudaSuccess || cudaMalloc(&d_seeds, k * 8) != cudaSuccess ||
        cudaMalloc(&d_redo, k * 4) != cudaSuccess) {
        cleanup(false);
        return false;
    }
    cudaMemcpy(d_seeds, seeds.data(), k * 8, cudaMemcpyHostToDevice);
    cudaMemset(d_redo, 0, k * 4);
    perm_init_kernel<<<2048, 256>>>(d_perm, dim, dim * k);
    perm_shuffle_kernel<16><<<unsigned((k + 31) / 32), 32>>>(d_perm, dim, uint32_t(k), d_seeds, d_redo);
    count_launches(2);
    std::vector<uint32_t> redo(k, 0);
    if (cudaDeviceSynchronize() != cudaSuccess ||
        cudaMemcpy(redo.data(), d_redo, k * 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
        cleanup(false);
        return false;
    }
    // tables whose draws hit next_below's rejection branch: exact host shuffle
    std::vector<uint32_t> tab;
    for (uint64_t j = 0; j < k; ++j) {
        if (!redo[j]) continue;
        tab.resize(dim);
        for (uint64_t t = 0; t < dim; ++t) tab[t] = uint32_t(t);
        SplitMix64 rng{seeds[j]};
        for (uint64_t t = dim - 1; t > 0; --t) std::swap(tab[t], tab[rng.next_below(t + 1)]);
        if (cudaMemcpy(d_perm + j * dim, tab.data(), dim * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
            cleanup(false);
            return false;
        }
    }
    cleanup(true);
    adopt_device_perm(f, dev, d_perm);
    return true;
}

}  // namespace bbmh
