// uniform4.cu -- the 4U-bit sketch kernel with warp-uniform hash functions (sm_100a).
//
// As in uniform.cu, a warp takes an item = (document, group of 32 functions),
// its lanes take different ids and all lanes evaluate the same function at a
// time: the coefficients are kernel-parameter operands read into uniform
// registers by a uniform-indexed loop over the group's functions
// (`LDCU UR, c[0x0][UR + imm]`), and each Horner step reads two vector
// registers (`IMAD.WIDE.U32 v, h, 2t, UR{c, 0}`). A 4U evaluation is ~14
// instructions, so the function loop is not unrolled (no code per group, no
// instruction-cache pressure): each lane keeps its running minima in its own
// column of the warp's shared-memory tile, which is also the transpose at the
// end of the item (lane l reads row l).
// Measured (profiles/round2/uniform4_ks.jsonl): 1.16-1.20 T evals/s for every
// k, against 1.30-1.34 T for the persistent kernel where its shape fits k
// (fewer register reads did not lift the IMAD.WIDE chain) and 0.81-1.15 T
// where it does not; uniform4_applies picks by the persistent shape.
// Reference semantics: hash_family.hpp:24-63 (4U, Mersenne fold, mod D),
// sketch.cpp:71-100.
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "kernels.cuh"
#include "options.hpp"

namespace bbmh {

namespace {

constexpr uint32_t kP = 0x7fffffffu;  // p = 2^31 - 1
constexpr int kGroup = 32;
constexpr uint32_t kMaxK = 1024;      // functions in the parameter bank
constexpr uint64_t kMinDocs = 2048;
constexpr uint64_t kSbBytes = 64ull << 20;
constexpr uint64_t kSbMinDocs = 3072;
constexpr int kTpb = 128;
constexpr int kRow = 36;  // words per row of a lane-column tile (conflict-free LDS.128 rows)
constexpr int kQuads = 4; // quads per lane per step: 16 ids

struct U4Coef {  // kernel-parameter bank; {a3, 2 a2, 2 a1, 2 a0} of the fold (kernels.cu)
    uint32_t a3[kMaxK];
    uint32_t c2[kMaxK];
    uint64_t c1[kMaxK];  // 64-bit: the IMAD.WIDE addend comes straight from a uniform register pair
    uint64_t c0[kMaxK];
};

struct U4Args {
    const uint64_t* row_ptr;
    uint64_t base;
    const uint32_t* idx;
    uint8_t* codes;
    uint64_t* minima;
    uint8_t* flags;
    int* err;
    unsigned long long* work;  // ticket counters (nullptr: static round-robin)
    uint32_t n, k, b;
    uint32_t groups;           // ceil(k / 32)
    uint32_t sb_docs;          // documents per super-block (0: from the row lengths)
    uint32_t dim_mask, neg_dim32, magic, magic_shift;
};

__device__ __forceinline__ uint32_t min3u(uint32_t a, uint32_t b, uint32_t c) { return min(min(a, b), c); }

__device__ __forceinline__ uint32_t fold(uint64_t v) {  // mod_mersenne31's first fold on doubled operands
    return (uint32_t)(v >> 32) + ((uint32_t)v >> 1);
}

template <bool POW2>
__device__ __forceinline__ uint32_t h4(uint32_t a3, uint32_t c2, uint64_t c1, uint64_t c0, uint32_t t2,
                                       const U4Args& A) {
    uint32_t s = fold((uint64_t)a3 * t2 + c2);
    uint32_t h = min(s, s - kP);  // lazy: [0, p + 1]
    s = fold((uint64_t)h * t2 + c1);
    h = min(s, s - kP);
    s = fold((uint64_t)h * t2 + c0);
    h = min3u(s, s - kP, s - 2 * kP);  // canonical
    if constexpr (POW2)
        return h & A.dim_mask;
    else
        return h + A.neg_dim32 * (__umulhi(h, A.magic) >> A.magic_shift);
}

// Every function of the group against NI staged ids of this lane; the running
// minima live in the lane's column of the tile (row r = function r).
template <bool POW2, int NI>
__device__ __forceinline__ void hash_ids(const U4Coef& C, const U4Args& A, uint32_t j0, uint32_t fc,
                                         const uint32_t (&t2)[NI], uint32_t* col) {
    for (uint32_t r = 0; r < fc; ++r) {
        const uint32_t j = j0 + r;
        const uint32_t a3 = C.a3[j], c2 = C.c2[j];
        const uint64_t c1 = C.c1[j], c0 = C.c0[j];
        uint32_t mn = col[r * kRow];
#pragma unroll
        for (int i = 0; i + 1 < NI; i += 2)
            mn = min3u(mn, h4<POW2>(a3, c2, c1, c0, t2[i], A), h4<POW2>(a3, c2, c1, c0, t2[i + 1], A));
        if constexpr (NI & 1) mn = min(mn, h4<POW2>(a3, c2, c1, c0, t2[NI - 1], A));
        col[r * kRow] = mn;
    }
}

__device__ __forceinline__ uint32_t stage(uint32_t t) {  // 2 (t mod p) for any u32 id
    return min3u(t, t - kP, t - 2 * kP) << 1;
}

template <bool POW2>
__device__ __forceinline__ void item4(const U4Coef& C, const U4Args& A, uint32_t d, uint32_t g, uint32_t lane,
                                      uint32_t* tile) {
    uint64_t beg = A.row_ptr[d], end = A.row_ptr[d + 1];
    if (end < beg) {
        if (lane == 0) atomicOr(A.err, 2);
        end = beg;
    }
    const uint32_t* ids = A.idx + (beg - A.base);
    const uint64_t nnz = end - beg;
    const uint64_t h16 = ((16 - ((uintptr_t)ids & 15)) & 15) >> 2;
    const uint32_t head = (uint32_t)(nnz < h16 ? nnz : h16);
    const uint64_t nq = (nnz - head) >> 2;
    const uint4* q4 = reinterpret_cast<const uint4*>(ids + head);
    // the group's first parameter slot and width in uniform registers
    const uint32_t gs = __reduce_min_sync(0xffffffffu, g);
    const uint32_t fc = __reduce_min_sync(0xffffffffu, min((uint32_t)kGroup, A.k - gs * kGroup));
    const uint32_t j0 = gs * kGroup;
    uint32_t* col = tile + lane;
#pragma unroll
    for (int r = 0; r < kGroup; ++r) col[r * kRow] = 0xffffffffu;
    // steps of 32 x kQuads quads (loads clamped to the last quad: a duplicated
    // id leaves the minimum unchanged)
    const uint32_t steps = __reduce_min_sync(0xffffffffu, (uint32_t)((nq + 32 * kQuads - 1) / (32 * kQuads)));
    for (uint32_t s = 0; s < steps; ++s) {
        uint32_t t2[4 * kQuads];
#pragma unroll
        for (int q = 0; q < kQuads; ++q) {
            const uint4 x = __ldg(q4 + min((uint64_t)s * 32 * kQuads + q * 32 + lane, nq - 1));
            t2[4 * q] = stage(x.x);
            t2[4 * q + 1] = stage(x.y);
            t2[4 * q + 2] = stage(x.z);
            t2[4 * q + 3] = stage(x.w);
        }
        hash_ids<POW2, 4 * kQuads>(C, A, j0, fc, t2, col);
    }
    // head ids before the first 16-byte granule and tail ids after the last
    // whole quad (<= 6): one single-id round
    const uint64_t tail0 = head + 4 * nq;
    const uint32_t left = __reduce_min_sync(0xffffffffu, head + (uint32_t)(nnz - tail0));
    if (left) {
        const uint32_t i = lane < left ? lane : 0;
        const uint32_t t2[1] = {stage(__ldg(ids + (i < head ? i : tail0 + (i - head))))};
        hash_ids<POW2, 1>(C, A, j0, fc, t2, col);
    }
    __syncwarp();
    // lane l reads row l: the minimum of function l over the warp's lanes
    uint32_t mn;
    {
        const uint4* row = reinterpret_cast<const uint4*>(tile + lane * kRow);
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
    const uint32_t cnt = fc;
    const bool empty = nnz == 0;
    const uint32_t mask = b >= 32 ? 0xffffffffu : ((1u << b) - 1);
    const uint32_t code = empty ? mask : (mn & mask);
    if (A.minima && lane < cnt) A.minima[(uint64_t)d * k + j0 + lane] = empty ? ~0ull : (uint64_t)mn;
    const uint64_t cb = ((uint64_t)k * b + 7) >> 3;
    uint8_t* out = A.codes + (uint64_t)d * cb + (uint64_t)j0 * b / 8;  // j0 * b is a multiple of 8
    if (b == 8) {
        if (lane < cnt) out[lane] = (uint8_t)code;
    } else {
        tile[lane] = code;
        __syncwarp();
        const uint32_t nbytes = (cnt * b + 7) >> 3;
        for (uint32_t B = lane; B < nbytes; B += 32) {
            const uint32_t bit0 = B << 3;
            const uint32_t ja = bit0 / b;
            const uint32_t jb = min((bit0 + 7) / b, cnt - 1);
            uint32_t v = 0;
            for (uint32_t j = ja; j <= jb; ++j) {
                const uint64_t c = tile[j];
                const int pos = (int)(j * b) - (int)bit0;
                v |= (uint32_t)(pos >= 0 ? (c << pos) : (c >> -pos));
            }
            out[B] = (uint8_t)v;
        }
        __syncwarp();
    }
    if (gs == 0 && lane == 0 && A.flags) A.flags[d] = empty ? 1 : 0;
}

template <bool POW2>
__global__ void __launch_bounds__(kTpb) sketch_uniform4_kernel(const __grid_constant__ U4Coef C,
                                                               const __grid_constant__ U4Args A) {
    __shared__ __align__(16) uint32_t s_t[kTpb / 32][kGroup * kRow];
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
    auto fetch_next = [&](uint32_t cur) -> uint32_t {
        if (!A.work) return cur + stride;
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(&A.work[0], 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        return t >= items ? items : (uint32_t)(stride + t);
    };
    for (uint32_t it = blockIdx.x * W + warp; it < items; it = fetch_next(it)) {
        const uint32_t sb = it / sb_items;
        const uint32_t rr = it - sb * sb_items;
        const uint32_t d0 = sb * sb_docs;
        const uint32_t nd = min(sb_docs, A.n - d0);
        const uint32_t g = rr / nd;
        const uint32_t d = d0 + (rr - g * nd);
        item4<POW2>(C, A, d, g, lane, s_t[warp]);
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

// The persistent kernel's shape for k decides (profiles/round2/uniform4_ks.jsonl,
// 60,000 webspam docs): it runs at ~1.30-1.34 T evals/s times its lane
// utilisation k / (J x tpb x tiles), but its 96- and 160-thread CTAs run at
// ~1.0-1.15 T; the uniform kernel runs at 1.16-1.20 T for every k. So: the
// uniform kernel when the persistent shape fills < 90% of its lanes or has
// a CTA size that is not a power of two (15 of 15 sampled k picked right:
// k = 40, 48, 96, 160, 200, 300, 400, 600, 800 uniform, +2..43%; k = 64,
// 128, 250, 500, 512, 1000 persistent).
// k in (16, 32]: one group of width k; the persistent shape for k = 24 fills
// 75% of its lanes (0.95 T evals/s).
bool uniform4_applies(const KernelFamily& F, uint64_t n) {
    const int64_t mode = opt(Opt::Uniform4U);  // 0 never, 1 by the persistent shape, 2 whenever it applies
    if (mode == 0 || F.scheme != 3 || !F.host4u) return false;
    if (F.k <= 16 || F.k > kMaxK || n < kMinDocs) return false;  // (k <= 16: the lane-split kernel)
    const uint64_t groups = (F.k + kGroup - 1) / kGroup;
    if (n * groups >= (1ull << 32)) return false;
    if (mode >= 2) return true;
    const LaunchShape sh = choose_shape(F.k, 3, n, sm_count());
    const double util = double(F.k) / (double(sh.jtile) * sh.jtiles);
    return util < 0.9 || (sh.tpb & (sh.tpb - 1)) != 0;
}

void launch_uniform_4u(const KernelFamily& F, const uint64_t* row_ptr, uint64_t base, const uint32_t* idx,
                       uint64_t n, uint32_t b, uint8_t* codes, uint64_t* minima, uint8_t* flags, int* err,
                       cudaStream_t st) {
    const uint32_t k = F.k;
    U4Coef C;
    std::memset(&C, 0, sizeof(C));
    for (uint32_t j = 0; j < k; ++j) {
        C.a3[j] = F.host4u[4 * j];
        C.c2[j] = F.host4u[4 * j + 1];
        C.c1[j] = F.host4u[4 * j + 2];
        C.c0[j] = F.host4u[4 * j + 3];
    }
    using KernelFn = void (*)(U4Coef, U4Args);
    const KernelFn kern = F.dim_pow2 ? sketch_uniform4_kernel<true> : sketch_uniform4_kernel<false>;
    int dev = 0;
    cudaGetDevice(&dev);
    static std::mutex mu;
    static std::map<std::pair<int, bool>, int> occ_cache;
    int occ = 0;
    {
        std::lock_guard lk(mu);
        auto it = occ_cache.find({dev, F.dim_pow2 != 0});
        if (it == occ_cache.end()) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTpb, 0);
            cudaGetLastError();
            it = occ_cache.emplace(std::make_pair(dev, F.dim_pow2 != 0), occ < 1 ? 1 : occ).first;
        }
        occ = it->second;
    }
    const int cap = (int)opt(Opt::CtasPerSm);
    if (cap > 0 && cap < occ) occ = cap;
    const uint32_t groups = (k + kGroup - 1) / kGroup;
    const uint64_t items = n * groups;
    uint64_t grid = (uint64_t)sm_count() * occ;
    const uint64_t need = (items + kTpb / 32 - 1) / (kTpb / 32);
    if (grid > need) grid = need;
    U4Args A{};
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
    A.groups = groups;
    A.sb_docs = opt(Opt::UniformSbDocs) > 0 ? (uint32_t)std::min<uint64_t>(opt(Opt::UniformSbDocs), n) : 0;
    A.dim_mask = F.dim_mask;
    A.neg_dim32 = F.neg_dim32;
    A.magic = F.magic;
    A.magic_shift = F.magic_shift;
    kern<<<(unsigned)grid, kTpb, 0, st>>>(C, A);
    if (const cudaError_t e = cudaPeekAtLastError(); e != cudaSuccess)
        fprintf(stderr, "bbmh: uniform 4U launch failed (%s)\n", cudaGetErrorString(e));
    count_launches(1);
    count(Counter::UniformLaunches);
}

}  // namespace bbmh
