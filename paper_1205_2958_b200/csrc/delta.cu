// delta.cu -- device side of the 2-byte id transfer encoding (see delta.hpp).
//
// One warp per row, 256 ids per step: lane l takes ids [8l, 8l + 8) of the
// step. A warp scan of the lanes' escape counts places each escape in the
// side list; a warp scan of the lanes' sums, plus the row's running total,
// gives each id. Per id: 2 B read, 4 B written, a few integer ops -- about
// 1% of the sketch kernel that reads the ids next.
#include <cuda_runtime.h>

#include "delta.hpp"
#include "kernels.cuh"

namespace bbmh {

namespace {

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, uint32_t lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= uint32_t(o)) v += t;
    }
    return v;
}

__global__ void __launch_bounds__(256) decode_delta16_kernel(
    const uint64_t* __restrict__ row_ptr, uint64_t base, uint64_t n,
    const uint16_t* __restrict__ deltas, const uint32_t* __restrict__ exc_ptr,
    const uint32_t* __restrict__ exc, uint32_t* __restrict__ ids) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        const uint64_t s = row_ptr[r] - base, e = row_ptr[r + 1] - base;
        uint32_t carry = 0;       // sum of the row's differences so far
        uint32_t ex = exc_ptr[r]; // next escape of the row in the side list
        for (uint64_t p0 = s; p0 < e; p0 += 256) {
            const uint64_t q0 = p0 + lane * 8;
            uint32_t v[8];
            uint32_t c = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                v[i] = q0 + i < e ? uint32_t(deltas[q0 + i]) : 1u;
                c += v[i] == 0;
            }
            const uint32_t ci = warp_incl_scan(c, lane);
            uint32_t at = ex + ci - c;
            uint32_t sum = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (v[i] == 0) v[i] = exc[at++];
                sum += q0 + i < e ? v[i] : 0u;
            }
            const uint32_t si = warp_incl_scan(sum, lane);
            uint32_t acc = carry + si - sum;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                acc += v[i];
                if (q0 + i < e) ids[q0 + i] = acc;
            }
            carry += __shfl_sync(0xffffffffu, si, 31);
            ex += __shfl_sync(0xffffffffu, ci, 31);
        }
    }
}

}  // namespace

void launch_decode_delta16(const uint64_t* row_ptr, uint64_t base, uint64_t n,
                           const uint16_t* deltas, const uint32_t* exc_ptr, const uint32_t* exc,
                           uint32_t* ids, cudaStream_t stream) {
    if (n == 0) return;
    const uint64_t blocks = std::min<uint64_t>((n + 7) / 8, 148ull * 64);
    decode_delta16_kernel<<<unsigned(blocks), 256, 0, stream>>>(row_ptr, base, n, deltas, exc_ptr, exc,
                                                                 ids);
    count_launches(1);
}

}  // namespace bbmh
