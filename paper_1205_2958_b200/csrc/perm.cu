// perm.cu -- permutation-mode sketch with an L2-resident, table-outer schedule.
//
// Reference: HashFamily::map's permutation branch perm_[j*D + t]
// (hash_family.hpp:88-89) inside sketch_one (sketch.cpp:90-98).
//
// With k tables of D u32 each (31.25 GiB at D = 2^24, k = 500) every
// evaluation is a random 4-byte gather; document-outer order (sketch_kernel)
// turns each one into a random 32-byte HBM sector read. Here the loop order is
// inverted: a pass keeps G tables (G*D*4 <= ~80 MB) resident in the 126 MB
// L2 while EVERY document of the batch streams past them (ids loaded with an
// L2 evict-first hint so they do not displace the tables), so the gathers hit
// L2 and HBM only carries one read of the tables plus one re-read of the ids
// per pass. Per-(doc, table) minima land in a u32 scratch matrix; a final
// kernel turns them into codes / minima / flags exactly like the epilogue of
// sketch_kernel (sketch.cpp:80-98).
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"
#include "options.hpp"

namespace bbmh {

namespace {

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// streamed ids: no L1 allocation, first to leave L2
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v)
                 : "l"(p), "l"(pol));
    return v;
}

// table gathers: keep in L2
__device__ __forceinline__ uint32_t ld_keep(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

// One warp per document (grid-stride); lanes stride over the ids, 4 loads in
// flight per lane, G gathers per id; minima reduced with redux.sync.
template <int G>
__global__ void __launch_bounds__(256) perm_pass_kernel(const uint32_t* __restrict__ perm,
                                                        uint64_t dim, uint32_t k, uint32_t j0,
                                                        uint32_t gcount,
                                                        const uint64_t* __restrict__ row_ptr,
                                                        uint64_t base,
                                                        const uint32_t* __restrict__ idx,
                                                        uint64_t n, uint32_t* __restrict__ min32,
                                                        int* err) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
    const uint32_t* tab[G];
#pragma unroll
    for (int g = 0; g < G; ++g) tab[g] = perm + (uint64_t)(j0 + (g < (int)gcount ? g : 0)) * dim;
    for (uint64_t doc = warp; doc < n; doc += nwarps) {
        uint64_t beg = row_ptr[doc], end = row_ptr[doc + 1];
        if (end < beg) end = beg;  // reported by the pack kernel
        beg -= base;
        end -= base;
        uint32_t m[G];
#pragma unroll
        for (int g = 0; g < G; ++g) m[g] = 0xffffffffu;
        uint64_t i = beg + lane;
        for (; i + 96 < end; i += 128) {
            uint32_t t[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) t[u] = ld_stream(idx + i + 32 * u, pol_first);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if ((uint64_t)t[u] >= dim) {
                    atomicOr(err, 1);
                    t[u] = 0;
                }
#pragma unroll
                for (int g = 0; g < G; ++g) m[g] = min(m[g], ld_keep(tab[g] + t[u], pol_last));
            }
        }
        for (; i < end; i += 32) {
            uint32_t t = ld_stream(idx + i, pol_first);
            if ((uint64_t)t >= dim) {
                atomicOr(err, 1);
                t = 0;
            }
#pragma unroll
            for (int g = 0; g < G; ++g) m[g] = min(m[g], ld_keep(tab[g] + t, pol_last));
        }
        uint32_t mine = 0xffffffffu;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const uint32_t r = __reduce_min_sync(0xffffffffu, m[g]);
            if (lane == (uint32_t)g) mine = r;
        }
        if (lane < gcount) min32[doc * k + j0 + lane] = mine;
    }
}

// minima -> codes (LE bitstream), minima (u64), flags; one CTA per document.
__global__ void __launch_bounds__(256) pack_minima_kernel(const uint32_t* __restrict__ min32,
                                                          const uint64_t* __restrict__ row_ptr,
                                                          uint64_t n, uint32_t k, uint32_t b,
                                                          uint8_t* __restrict__ codes,
                                                          uint64_t* __restrict__ minima,
                                                          uint8_t* __restrict__ flags, int* err) {
    const uint32_t mask = b >= 32 ? 0xffffffffu : ((1u << b) - 1);
    const uint64_t cb = ((uint64_t)k * b + 7) >> 3;
    for (uint64_t doc = blockIdx.x; doc < n; doc += gridDim.x) {
        const uint64_t beg = row_ptr[doc], end = row_ptr[doc + 1];
        if (end < beg && threadIdx.x == 0) atomicOr(err, 2);
        const bool empty = end <= beg;
        const uint32_t* m = min32 + doc * k;
        if (minima)
            for (uint32_t j = threadIdx.x; j < k; j += blockDim.x)
                minima[doc * k + j] = empty ? ~0ull : (uint64_t)m[j];
        if (flags && threadIdx.x == 0) flags[doc] = empty ? 1 : 0;
        uint8_t* out = codes + doc * cb;
        for (uint64_t B = threadIdx.x; B < cb; B += blockDim.x) {
            const uint64_t bit0 = B << 3;
            const uint32_t ja = (uint32_t)(bit0 / b);
            const uint64_t jb0 = (bit0 + 7) / b;
            const uint32_t jb = (uint32_t)(jb0 < k - 1 ? jb0 : k - 1);
            uint32_t v = 0;
            for (uint32_t j = ja; j <= jb; ++j) {
                const uint64_t code = empty ? mask : (m[j] & mask);
                const int64_t pos = (int64_t)j * b - (int64_t)bit0;
                v |= (uint32_t)(pos >= 0 ? (code << pos) : (code >> -pos));
            }
            out[B] = (uint8_t)v;
        }
    }
}

template <int G>
void launch_pass(const KernelFamily& F, uint32_t j0, uint32_t gc, const uint64_t* row_ptr,
                 uint64_t base, const uint32_t* idx, uint64_t n, uint32_t* min32, int* err,
                 int grid, cudaStream_t st) {
    perm_pass_kernel<G><<<grid, 256, 0, st>>>(F.perm, F.dim, F.k, j0, gc, row_ptr, base, idx, n,
                                              min32, err);
}

}  // namespace

bool perm_tablewise_applies(const KernelFamily& F, uint64_t n) {
    const int64_t mode = opt(Opt::PermTablewise);
    if (mode >= 0) return mode != 0;
    const uint64_t table_bytes = (uint64_t)F.k * F.dim * 4;
    return table_bytes > (96ull << 20) && n >= 256;
}

bool launch_perm_tablewise(const KernelFamily& F, const uint64_t* row_ptr, uint64_t base,
                           const uint32_t* idx, uint64_t n, uint32_t b, uint8_t* codes,
                           uint64_t* minima, uint8_t* flags, int* err, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // The per-(doc, table) minima scratch is n*k*4 bytes; documents go in
    // slices that keep it within the budget (each slice streams the tables
    // through L2 once more). If even a small slice cannot be allocated the
    // caller runs the document-outer kernel, which needs no scratch.
    const uint64_t budget_bytes = (uint64_t)(opt(Opt::PermScratchMb) > 0 ? opt(Opt::PermScratchMb) : 2048) << 20;
    uint64_t slice = budget_bytes / ((uint64_t)F.k * 4);
    if (slice < 1) slice = 1;
    if (slice > n) slice = n;
    uint32_t* min32 = nullptr;
    while (cudaMallocAsync(&min32, slice * F.k * sizeof(uint32_t), st) != cudaSuccess) {
        cudaGetLastError();
        min32 = nullptr;
        if (slice <= 256) return false;
        slice /= 2;
    }
    // tables per pass: as many as fit in ~80 MB of L2 (power of two, <= 32)
    const uint64_t l2_budget = 80ull << 20;
    uint32_t G = 1;
    while (G < 32 && (uint64_t)(2 * G) * F.dim * 4 <= l2_budget && 2 * G <= F.k) G *= 2;
    const int grid = sms * 8;
    const uint64_t cb = ((uint64_t)F.k * b + 7) >> 3;
    uint64_t launches = 0;
    for (uint64_t d0 = 0; d0 < n; d0 += slice) {
        const uint64_t m = n - d0 < slice ? n - d0 : slice;
        const uint64_t* rp = row_ptr + d0;
        for (uint32_t j0 = 0; j0 < F.k; j0 += G, ++launches) {
            const uint32_t gc = F.k - j0 < G ? F.k - j0 : G;
            switch (G) {
                case 1: launch_pass<1>(F, j0, gc, rp, base, idx, m, min32, err, grid, st); break;
                case 2: launch_pass<2>(F, j0, gc, rp, base, idx, m, min32, err, grid, st); break;
                case 4: launch_pass<4>(F, j0, gc, rp, base, idx, m, min32, err, grid, st); break;
                case 8: launch_pass<8>(F, j0, gc, rp, base, idx, m, min32, err, grid, st); break;
                case 16: launch_pass<16>(F, j0, gc, rp, base, idx, m, min32, err, grid, st); break;
                default: launch_pass<32>(F, j0, gc, rp, base, idx, m, min32, err, grid, st); break;
            }
        }
        const uint64_t pg = m < (uint64_t)sms * 16 ? m : (uint64_t)sms * 16;
        pack_minima_kernel<<<(unsigned)pg, 256, 0, st>>>(min32, rp, m, F.k, b, codes + d0 * cb,
                                                         minima ? minima + d0 * F.k : nullptr,
                                                         flags ? flags + d0 : nullptr, err);
        ++launches;
    }
    cudaFreeAsync(min32, st);
    count_launches(launches);
    return true;
}

}  // namespace bbmh
