// uniform.cu -- the 2U sketch kernel with warp-uniform hash functions (sm_100a).
//
// sketch_kernel (kernels.cu) gives every thread its own hash functions and
// broadcasts each id to all of them, so every `IMAD h, a2, t, a1` reads
// registers that change from one evaluation to the next: register-file bank
// reads, not the IMAD pipe, bind it at ~0.78 of the IMAD roofline
// (profiles/r10/README.md). This kernel turns the layout around:
//   * a warp works on one item = (document, group of 32 hash functions);
//   * its lanes take different ids of the document (8 per lane per step,
//     two coalesced 16-byte loads) and all lanes evaluate the SAME function
//     at a time, so the multiplier a2 is a kernel-parameter (constant-bank)
//     operand and a1 repeats across consecutive IMADs (operand reuse cache):
//     one register read per evaluation, `IMAD R, Rt, UR(a2), Ra1.reuse`;
//   * the group index is a template parameter of the item body (one switch
//     per item selects it), which is what lets ptxas address the
//     coefficients at fixed constant-bank offsets; the tail group (k not a
//     multiple of 32) sits in a fixed extra slot with a compile-time width;
//   * items come from a ticket counter in group-major order inside
//     super-blocks of documents that stay in L2 (each document is read from
//     HBM about once although every group reads it) and that are larger
//     than the items in flight, so the warps run the hot loops of one or two
//     groups: only the hot loop is instantiated per group (~7 KB each) and
//     the instruction cache (L1.5 ~32 KB) holds a few of them -- with
//     groups interleaved the kernel ran 40% slower on instruction-fetch
//     stalls (ncu no_instruction, profiles/round2);
//   * at the end of an item the 32 lanes' partial minima are transposed
//     through shared memory and reduced (lane l ends with function l of the
//     group), and
//     the b-bit codes go into the reference's bitstream (sketch.cpp:64-69).
// Reference semantics: hash_family.hpp:48-51 (2U), sketch.cpp:71-100.
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "kernels.cuh"
#include "options.hpp"

namespace bbmh {

namespace {

constexpr int kGroup = 32;        // hash functions per item (one per lane after the transpose)
constexpr int kFullGroups = 16;   // compile-time group bodies; the tail group uses slot 16
constexpr uint32_t kUniformMaxK = (kFullGroups + 1) * kGroup;  // 544
// below this the persistent kernel's shorter tail wins (k = 500, 1,024 docs: 0.16 vs 0.20 ms)
constexpr uint64_t kUniformMinDocs = 2048;
// Documents per super-block: as many as fit kSbBytes of ids (so every group
// after the first reads them from L2), but at least kSbMinDocs, or the warps
// in flight (one item each) span several groups whose hot loops no longer
// fit the instruction cache. C2, k = 500 (profiles/round2/uniform_sb.jsonl):
// 3,072 docs 14.5 T evals/s and 5.3 GB of DRAM reads per launch, 4,096 docs
// 14.8 T and 5.7 GB, 6,144 docs 14.8 T and 26 GB, 16,384 docs 83 GB; the
// 64 MB first chosen gave 4,500 docs and 7.4 GB (ncu, full C2 launch): the
// super-block in flight and the next one's first items no longer fit L2.
// 58 MB keeps C2 at ~4,080 docs.
constexpr uint64_t kSbBytes = 58ull << 20;
constexpr uint64_t kSbMinDocs = 3072;
constexpr int kTpb = 128;
constexpr int kRow = 36;  // words per row of the transpose tile (conflict-free LDS.128 rows)

struct UniformCoef {  // lives in the kernel-parameter bank
    uint32_t a2[(kFullGroups + 1) * kGroup];
    uint32_t a1[(kFullGroups + 1) * kGroup];
};

struct UniformArgs {
    const uint64_t* row_ptr;
    uint64_t base;
    const uint32_t* idx;
    uint8_t* codes;
    uint64_t* minima;
    uint8_t* flags;
    int* err;
    unsigned long long* work;  // ticket counters (nullptr: static round-robin)
    uint32_t n;                // documents (n * groups < 2^32)
    uint32_t k, b, shift;
    uint32_t full;             // full 32-function groups
    uint32_t groups;           // full + (tail group ? 1 : 0)
    uint32_t tail_fc;          // compile-time width of the tail body (multiple of 4; 0: none)
    uint32_t sb_docs;          // documents per super-block (0: from the row lengths)
    uint32_t min_nnz;          // > 0: return unless the batch averages >= min_nnz ids per document
};

__device__ __forceinline__ uint32_t min3u(uint32_t a, uint32_t b, uint32_t c) {
    return min(min(a, b), c);
}

// The hot loop of an item, for the functions at parameter slot S (S = g for
// full groups, kFullGroups for the tail group of width FC): full steps of 64
// quads (8 ids per lane, the next step's loads in flight). Only this loop is
// instantiated per group (~7 KB); the instruction cache holds the loops of
// the one or two groups in flight plus the shared rest of the item.
template <int S, int FC>
__device__ __forceinline__ void group_hash(const UniformCoef& C, const uint32_t* __restrict__ ids,
                                          uint32_t head, uint64_t nq, uint64_t nnz, uint32_t lane,
                                          uint32_t (&m)[kGroup]) {
    const uint4* q4 = reinterpret_cast<const uint4*>(ids + head);
    uint32_t a1[FC];
#pragma unroll
    for (int r = 0; r < FC; ++r) a1[r] = C.a1[S * kGroup + r];
    const uint64_t full_end = nq & ~63ull;
    if (full_end) {
        uint4 x = __ldg(q4 + lane), y = __ldg(q4 + 32 + lane);
        for (uint64_t s = 0; s < full_end; s += 64) {
            const uint4 xc = x, yc = y;
            if (s + 64 < full_end) {
                x = __ldg(q4 + s + 64 + lane);
                y = __ldg(q4 + s + 96 + lane);
            }
#pragma unroll
            for (int r = 0; r < FC; ++r) {
                // two independent min3 chains per function: the fastest of 24
                // reduction shapes measured (tools/proto/uni_search.cu)
                const uint32_t a2 = C.a2[S * kGroup + r];
                const uint32_t t0 = min3u(a1[r] + a2 * xc.y, m[r], a1[r] + a2 * yc.x);
                const uint32_t t1 = min3u(a1[r] + a2 * xc.w, a1[r] + a2 * xc.z, a1[r] + a2 * yc.y);
                const uint32_t t2 = min3u(a1[r] + a2 * xc.x, a1[r] + a2 * yc.w, t0);
                m[r] = min3u(t2, t1, a1[r] + a2 * yc.z);
            }
        }
    }
}

template <int G>
__device__ __forceinline__ void hash_full(const UniformCoef& C, uint32_t g, const uint32_t* ids,
                                          uint32_t head, uint64_t nq, uint64_t nnz, uint32_t lane,
                                          uint32_t (&m)[kGroup]) {
    if (g == G) return group_hash<G, kGroup>(C, ids, head, nq, nnz, lane, m);
    if constexpr (G + 1 < kFullGroups) hash_full<G + 1>(C, g, ids, head, nq, nnz, lane, m);
}

__device__ __forceinline__ void hash_tail(const UniformCoef& C, uint32_t fc, const uint32_t* ids,
                                          uint32_t head, uint64_t nq, uint64_t nnz, uint32_t lane,
                                          uint32_t (&m)[kGroup]) {
    switch (fc) {
        case 4: return group_hash<kFullGroups, 4>(C, ids, head, nq, nnz, lane, m);
        case 8: return group_hash<kFullGroups, 8>(C, ids, head, nq, nnz, lane, m);
        case 12: return group_hash<kFullGroups, 12>(C, ids, head, nq, nnz, lane, m);
        case 16: return group_hash<kFullGroups, 16>(C, ids, head, nq, nnz, lane, m);
        case 20: return group_hash<kFullGroups, 20>(C, ids, head, nq, nnz, lane, m);
        case 24: return group_hash<kFullGroups, 24>(C, ids, head, nq, nnz, lane, m);
        case 28: return group_hash<kFullGroups, 28>(C, ids, head, nq, nnz, lane, m);
        default: return group_hash<kFullGroups, 32>(C, ids, head, nq, nnz, lane, m);
    }
}

// One item: document d, functions [32 g, 32 g + cnt).
__device__ __forceinline__ void uniform_item(const UniformCoef& C, const UniformArgs& A, uint32_t d,
                                             uint32_t g, uint32_t lane, uint32_t* s_t) {
    uint64_t beg = A.row_ptr[d], end = A.row_ptr[d + 1];
    if (end < beg) {
        if (lane == 0) atomicOr(A.err, 2);
        end = beg;
    }
    const uint32_t* ids = A.idx + (beg - A.base);
    const uint64_t nnz = end - beg;
    // head ids up to 16-byte alignment, whole quads, tail ids
    const uint64_t h16 = ((16 - ((uintptr_t)ids & 15)) & 15) >> 2;
    const uint32_t head = (uint32_t)(nnz < h16 ? nnz : h16);
    const uint64_t nq = (nnz - head) >> 2;

    uint32_t m[kGroup];
#pragma unroll
    for (int r = 0; r < kGroup; ++r) m[r] = 0xffffffffu;
    if (g < A.full)
        hash_full<0>(C, g, ids, head, nq, nnz, lane, m);
    else
        hash_tail(C, A.tail_fc, ids, head, nq, nnz, lane, m);

    // the rest, with the group's coefficients read by a runtime slot index
    // (the uniform kernel takes long rows, where this is a few percent of
    // the work): 4-id steps while they are mostly full (duplicated quads
    // leave the minimum unchanged), then single-id rounds over the remaining
    // quads' ids, the head ids and the tail ids (padded tail functions have
    // zero coefficients; their minima are dropped)
    const uint4* q4 = reinterpret_cast<const uint4*>(ids + head);
    const uint32_t slot = (g < A.full ? g : (uint32_t)kFullGroups) * kGroup;
    uint64_t s = nq & ~63ull;
    while (nq - s > 24) {
        const uint4 x = __ldg(q4 + min(s + lane, nq - 1));
#pragma unroll
        for (int r = 0; r < kGroup; ++r) {
            const uint32_t a1 = C.a1[slot + r], a2 = C.a2[slot + r];
            const uint32_t t0 = min3u(a1 + a2 * x.x, a1 + a2 * x.y, a1 + a2 * x.z);
            m[r] = min3u(m[r], t0, a1 + a2 * x.w);
        }
        s = min(s + 32, nq);
    }
    const uint64_t rest0 = head + 4 * s;  // first unprocessed id after the head
    const uint64_t e = head + (nnz - rest0);
    for (uint64_t i0 = 0; i0 < e; i0 += 32) {
        const uint64_t i = i0 + lane;
        const uint32_t t = __ldg(ids + (i >= e ? 0 : i < head ? i : rest0 + (i - head)));
#pragma unroll
        for (int r = 0; r < kGroup; ++r) m[r] = min(m[r], C.a1[slot + r] + C.a2[slot + r] * t);
    }

    // lane l ends with the warp's minimum of function l of the group: lane l
    // writes column l of a 32 x 32 tile, reads row l (8 conflict-free
    // LDS.128) and reduces it -- ~60 instructions against ~250 for a
    // shuffle transpose (+1.3% at C2, profiles/round2/uniform_variants_ab.jsonl)
#pragma unroll
    for (int r = 0; r < kGroup; ++r) s_t[r * kRow + lane] = m[r];
    __syncwarp();
    uint32_t mn;
    {
        const uint4* row = reinterpret_cast<const uint4*>(s_t + lane * kRow);
        uint32_t u[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint4 v0 = row[2 * c], v1 = row[2 * c + 1];
            u[c] = min3u(min3u(v0.x, v0.y, v0.z), min3u(v0.w, v1.x, v1.y), min(v1.z, v1.w));
        }
        mn = min(min3u(u[0], u[1], u[2]), u[3]);
    }
    __syncwarp();

    // ---- epilogue: minimum -> code -> packed bitstream (sketch.cpp:80-98) ----
    const uint32_t k = A.k, b = A.b;
    const uint32_t j0 = g * kGroup;
    const uint32_t cnt = min((uint32_t)kGroup, k - j0);
    const bool empty = nnz == 0;
    const uint32_t mask = b >= 32 ? 0xffffffffu : ((1u << b) - 1);
    mn >>= A.shift;
    const uint32_t code = empty ? mask : (mn & mask);
    if (A.minima && lane < cnt) A.minima[(uint64_t)d * k + j0 + lane] = empty ? ~0ull : (uint64_t)mn;
    const uint64_t cb = ((uint64_t)k * b + 7) >> 3;
    uint8_t* out = A.codes + (uint64_t)d * cb + (uint64_t)j0 * b / 8;  // j0 * b is a multiple of 8
    if (b == 8) {
        if (lane < cnt) out[lane] = (uint8_t)code;
    } else {
        uint32_t* s_code = s_t;  // the transpose tile is free again
        s_code[lane] = code;
        __syncwarp();
        const uint32_t nbytes = (cnt * b + 7) >> 3;
        for (uint32_t B = lane; B < nbytes; B += 32) {
            const uint32_t bit0 = B << 3;
            const uint32_t ja = bit0 / b;
            const uint32_t jb = min((bit0 + 7) / b, cnt - 1);
            uint32_t v = 0;
            for (uint32_t j = ja; j <= jb; ++j) {
                const uint64_t c = s_code[j];
                const int pos = (int)(j * b) - (int)bit0;
                v |= (uint32_t)(pos >= 0 ? (c << pos) : (c >> -pos));
            }
            out[B] = (uint8_t)v;
        }
        __syncwarp();
    }
    if (g == 0 && lane == 0 && A.flags) A.flags[d] = empty ? 1 : 0;
}

__global__ void __launch_bounds__(kTpb, 6) sketch_uniform_kernel(const __grid_constant__ UniformCoef C,
                                                              const __grid_constant__ UniformArgs A) {
    __shared__ __align__(16) uint32_t s_t[kTpb / 32][kGroup * kRow];
    if (A.min_nnz && A.row_ptr[A.n] - A.row_ptr[0] < (uint64_t)A.min_nnz * A.n)
        return;  // the persistent kernel launched beside this one takes the batch
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = kTpb / 32;
    const uint32_t items = A.n * A.groups;
    const uint32_t stride = gridDim.x * W;
    uint32_t sb_docs = A.sb_docs;
    if (!sb_docs) {
        const uint64_t bytes = (A.row_ptr[A.n] - A.row_ptr[0]) * 4 + 1;
        const uint64_t fit = kSbBytes * A.n / bytes;
        const uint64_t want = fit > kSbMinDocs ? fit : kSbMinDocs;
        sb_docs = (uint32_t)(want < A.n ? want : A.n);
    }
    const uint32_t sb_items = sb_docs * A.groups;
    // items after the first wave come from a ticket counter, one ticket ahead
    auto fetch_next = [&](uint32_t cur) -> uint32_t {
        if (!A.work) return cur + stride;
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(&A.work[0], 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        return t >= items ? items : (uint32_t)(stride + t);
    };
    uint32_t it = blockIdx.x * W + warp;
    // the next ticket is taken when the current item is done (not one item
    // ahead): the items in flight then span ~one ticket per warp, so fewer
    // groups share the instruction cache
    for (; it < items; it = fetch_next(it)) {
        // item -> (super-block, group, document): group-major inside a super-block
        const uint32_t sb = it / sb_items;
        const uint32_t rr = it - sb * sb_items;
        const uint32_t d0 = sb * sb_docs;
        const uint32_t nd = min(sb_docs, A.n - d0);
        const uint32_t g = rr / nd;
        const uint32_t d = d0 + (rr - g * nd);
        uniform_item(C, A, d, g, lane, s_t[warp]);
    }
    if (A.work && lane == 0) {  // the last warp out resets the counters
        __threadfence();
        if (atomicAdd(&A.work[1], 1ull) == (unsigned long long)stride - 1) {
            A.work[0] = 0;
            A.work[1] = 0;
        }
    }
}

}  // namespace

// Measured crossovers against the persistent kernel (profiles/round2/
// uniform_ab.jsonl, webspam-shaped rows of 40..3,728 ids): the uniform
// kernel's per-item cost (cross-lane transpose, epilogue, partial steps) is
// paid per (document, group), so it needs longer rows as k grows.
uint32_t uniform_min_nnz(const KernelFamily& F, uint64_t n) {
    const int64_t mode = opt(Opt::Uniform2U);  // 0 off, 1 by row length, 2 whenever it applies
    const uint32_t k = F.k;
    if (F.scheme != 1 || !F.host2u || mode == 0) return 0;
    if (k <= 16 || k > kUniformMaxK || n < kUniformMinDocs) return 0;
    // at k = 32 the lane-split kernel (all functions per lane) is as fast on
    // webspam rows and 6% faster on 12,000-id rows; at 16 < k < 32 it pays
    // for functions its lanes hold but the group width does not
    // (profiles/round2/uniform_smallk_ab.jsonl: k = 20 / 24 / 28 1.55 /
    // 1.32 / 1.16x at 3,728 ids)
    if (k == kGroup && mode < 2) return 0;
    const uint32_t groups = (k + kGroup - 1) / kGroup;
    if (n * groups >= (1ull << 32)) return 0;
    if (mode >= 2) return 1;
    // with the shared-memory transpose (profiles/round2/uniform_crossover.jsonl,
    // 1,500..12,000 ids per row): at k = 300/400 the uniform kernel is ahead
    // from 1,500 ids (+3/+5%), at k = 544 by 1.25x (the persistent kernel
    // pads 544 functions to 2 x 512 lanes); at 400 < k <= 512 the persistent
    // kernel's 16-function-wide threads keep up until ~3,700 ids (k = 500:
    // 0.99x at 2,600, 1.003x at 3,728, 1.02x at 12,000)
    return k < kGroup ? 1500 : k <= 64 ? 700 : k <= 128 ? 1000 : k <= 400 ? 1500 : k <= 512 ? 3600 : 1500;
}

void launch_uniform_2u(const KernelFamily& F, const uint64_t* row_ptr, uint64_t base,
                       const uint32_t* idx, uint64_t n, uint32_t b, uint8_t* codes,
                       uint64_t* minima, uint8_t* flags, int* err, cudaStream_t st,
                       uint32_t min_nnz) {
    const uint32_t k = F.k;
    const uint32_t full = std::min<uint32_t>(k / kGroup, kFullGroups);
    const uint32_t rem = k - full * kGroup;  // <= 32
    const uint32_t groups = full + (rem ? 1 : 0);

    UniformCoef C;
    std::memset(&C, 0, sizeof(C));  // padded tail functions hash to 0; their codes are dropped
    for (uint32_t j = 0; j < k; ++j) {
        const uint32_t slot = j < full * kGroup ? j : kFullGroups * kGroup + (j - full * kGroup);
        C.a1[slot] = F.host2u[2 * j];
        C.a2[slot] = F.host2u[2 * j + 1];
    }
    int dev = 0;
    cudaGetDevice(&dev);
    static std::mutex mu;
    static std::map<int, int> occ_cache;
    int occ = 0;
    {
        std::lock_guard lk(mu);
        auto it = occ_cache.find(dev);
        if (it == occ_cache.end()) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sketch_uniform_kernel, kTpb, 0);
            cudaGetLastError();
            it = occ_cache.emplace(dev, occ < 1 ? 1 : occ).first;
        }
        occ = it->second;
    }
    const int cap = (int)opt(Opt::CtasPerSm);
    if (cap > 0 && cap < occ) occ = cap;
    const uint64_t items = n * groups;
    uint64_t grid = (uint64_t)sm_count() * occ;
    const uint64_t need = (items + kTpb / 32 - 1) / (kTpb / 32);
    if (grid > need) grid = need;
    UniformArgs A{};
    uint64_t sb_override = 0;
    A.row_ptr = row_ptr;
    A.base = base;
    A.idx = idx;
    A.codes = codes;
    A.minima = minima;
    A.flags = flags;
    A.err = err;
    A.work = opt(Opt::DynamicDocs) ? ticket_slot(dev) : nullptr;
    A.n = (uint32_t)n;
    A.k = k;
    A.b = b;
    A.shift = F.shift2u;
    A.full = full;
    A.groups = groups;
    A.tail_fc = rem ? (rem + 3) & ~3u : 0;
    if (opt(Opt::UniformSbDocs) > 0) sb_override = (uint64_t)opt(Opt::UniformSbDocs);
    A.sb_docs = (uint32_t)std::min<uint64_t>(sb_override, n);  // 0: from the row lengths, on the device
    A.min_nnz = min_nnz;
    sketch_uniform_kernel<<<(unsigned)grid, kTpb, 0, st>>>(C, A);
    if (const cudaError_t e = cudaPeekAtLastError(); e != cudaSuccess)
        fprintf(stderr, "bbmh: uniform 2U launch failed (%s)\n", cudaGetErrorString(e));
    count_launches(1);
    count(Counter::UniformLaunches);
}

}  // namespace bbmh
