// permgen.cu -- permutation tables built on the GPU.
//
// Reference: HashFamily::build, permutation branch (hash_family.cpp:105-114):
// per table j, tab[t] = t, then for t = D-1 .. 1 swap tab[t] with
// tab[SplitMix64(keyed_u64(seed, 1, j, 0)).next_below(t + 1)] (prng.hpp:42-61).
// Each shuffle is sequential; on the host it is bound by cache misses into a
// 64 MB table (~0.4 s per table, 19 s for k = 500 on 16 cores).
//
// Here one warp runs one table's shuffle, 32 swaps per step. SplitMix64's
// i-th draw is mix64(seed + (i+1)·φ), so the 32 lanes draw their swaps'
// partners at once. Swap i touches positions t0-i and r_i. When no r_i falls
// inside the step's own positions [t0-31, t0] and no two r_i are equal, the
// 32 swaps touch 64 distinct entries and commute: every lane loads its two
// entries, then stores them exchanged. Otherwise (about 800 of the 524 K steps
// of a 2^24 table, nearly all near its end) lane 0 applies the step's swaps in
// order. The result is the same permutation, swap for swap. A draw that would
// take the rejection branch of next_below (probability < 2^-32 per draw)
// marks its table, which is then rebuilt on the host.
#include <cuda_runtime.h>

#include <cstdlib>
#include <vector>

#include "core.hpp"
#include "options.hpp"
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

__global__ void __launch_bounds__(128) perm_shuffle_warp_kernel(uint32_t* __restrict__ perm, uint64_t dim,
                                                                uint32_t k, const uint64_t* __restrict__ seeds,
                                                                uint32_t* __restrict__ host_redo) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (j >= k) return;  // whole warps
    uint32_t* tab = perm + size_t(j) * dim;
    const uint64_t seed = seeds[j];
    uint64_t drawn = 0;  // draws used by earlier steps
    for (uint64_t t0 = dim - 1; t0 > 0;) {
        const uint32_t w = t0 < 32 ? uint32_t(t0) : 32u;  // swaps t = t0, t0-1, ..., t0-w+1
        const bool act = lane < w;
        const uint64_t t = t0 - lane;
        uint64_t r = 0;
        bool rejected = false;
        if (act) {
            const uint64_t bound = t + 1;
            const uint64_t v = dmix64(seed + (drawn + lane + 1) * kPhi);
            if ((bound & (bound - 1)) == 0) {
                r = v & (bound - 1);
            } else {
                // next_below's rejection: v >= UINT64_MAX - UINT64_MAX % bound,
                // only possible in the top `bound` values of the range
                rejected = (v >> 32) == 0xffffffffull && v >= ~0ull - (~0ull % bound);
                r = v % bound;
            }
        }
        if (__any_sync(0xffffffffu, rejected)) {
            if (lane == 0) host_redo[j] = 1;
            return;
        }
        const bool in_step = act && r + w > t0;  // r in [t0-w+1, t0]
        const unsigned same = __match_any_sync(0xffffffffu, act ? r : ~0ull - lane);
        const bool dup = act && __popc(same) > 1;
        if (!__any_sync(0xffffffffu, in_step || dup)) {
            uint32_t a = 0, b = 0;
            if (act) {
                a = tab[t];
                b = tab[r];
            }
            if (act) {
                tab[t] = b;
                tab[r] = a;
            }
        } else {
            for (uint32_t i = 0; i < w; ++i) {
                const uint64_t ri = __shfl_sync(0xffffffffu, r, int(i));
                if (lane == 0) {
                    const uint64_t ti = t0 - i;
                    const uint32_t x = tab[ti];
                    tab[ti] = tab[ri];
                    tab[ri] = x;
                }
            }
        }
        __syncwarp();  // this step's stores before the next step's loads, across lanes
        drawn += w;
        t0 -= w;
    }
}

}  // namespace

bool build_perm_tables_gpu(Family& f) {
    if (!opt(Opt::GpuPermgen)) return false;
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
    perm_shuffle_warp_kernel<<<unsigned((k + 3) / 4), 128>>>(d_perm, dim, uint32_t(k), d_seeds, d_redo);
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
