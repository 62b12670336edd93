// kernels.cu -- sm_100a minwise-hashing kernels (the hot path).
//
// One CTA sketches one document (or one tile of `jtile` hash functions of
// it, for very large k). Layout and roofline reasoning are in DESIGN.md; the
// short version:
//   * the document's feature ids are staged once into shared memory (and
//     pre-transformed per scheme: t mod p, doubled for the Mersenne trick),
//     padded to a multiple of 4 with a duplicate id (min is unaffected);
//   * each thread owns J hash functions (coefficients and running minima in
//     registers) and streams the staged ids with broadcast 128-bit shared
//     loads, so one LDS.128 feeds 4*J hash evaluations;
//   * 2U is one IMAD per evaluation plus half a 3-input min (VIMNMX3); the
//     2U top-s-bit shift is applied once to the minimum (shifting is
//     monotone, so min(h >> c) == min(h) >> c);
//   * 4U over GF(2^31-1) folds every Horner step with a single
//     IMAD.WIDE.U32 on doubled operands: 2v = h*(2t) + 2a puts v >> 31 in the
//     high word and (v & p) << 1 in the low word, so the fold is hi + (lo>>1);
//     intermediate steps are reduced lazily to [0, p+1] with one min, the
//     last one canonically with a 3-input min;
//   * `% D` for non-power-of-two D is a multiply-high by a host-computed
//     magic number; 4U-mod (any prime p) uses a 64-bit Barrett reduction;
//   * the epilogue turns minima into b-bit codes and packs them into the
//     reference's little-endian bitstream (sketch.cpp:64-69) through shared
//     memory, writing bytes coalesced.
// Reference semantics: sketch.cpp:71-100, hash_family.hpp:24-63,77-109.
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <cstdio>
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "options.hpp"

namespace bbmh {

namespace {

constexpr uint32_t kDefaultTile = 4096;  // feature ids staged per pipeline item (16 KB)
constexpr uint32_t kP31 = 0x7fffffffu;

std::atomic<uint64_t> g_launches{0};

// SM count of the current device, cached (attribute queries cost microseconds)
int device_sms() {
    static std::atomic<int> cache[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    int v = cache[dev].load(std::memory_order_relaxed);
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
        cache[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

enum : int { S_PERM = 0, S_2U = 1, S_4UMOD = 2, S_4UBIT = 3 };

__device__ __forceinline__ uint32_t min3u(uint32_t a, uint32_t b, uint32_t c) {
    return min(min(a, b), c);
}

// 2*(h*t + a) with t2 = 2t, c = 2a; returns ((h*t+a) >> 31) + ((h*t+a) & p),
// which is < 2^32 whenever h*t + a < 2^62 (mod_mersenne31's first fold,
// hash_family.hpp:27).
__device__ __forceinline__ uint32_t m31_fold(uint32_t h, uint32_t t2, uint32_t c) {
    const uint64_t v = (uint64_t)h * t2 + c;
    return (uint32_t)(v >> 32) + ((uint32_t)v >> 1);
}

// x mod p for x < 2^62, 3 <= p < 2^31 (and p = 2), barrett = floor((2^64-1)/p)
__device__ __forceinline__ uint32_t mod_barrett(uint64_t x, uint32_t p, uint64_t barrett) {
    const uint64_t q = __umul64hi(x, barrett);
    const uint32_t r = (uint32_t)x + (uint32_t)q * (0u - p);  // x - q*p; true r in [0, 2p)
    return min(r, r - p);
}

template <bool POW2>
__device__ __forceinline__ uint32_t reduce_dim(const KernelFamily& F, uint32_t h) {
    if constexpr (POW2) {
        return h & F.dim_mask;
    } else {
        // h - D*q as h + q*(2^32 - D): one IMAD, no negation (IMAD.MOV) on the fma pipe
        return h + F.neg_dim32 * (__umulhi(h, F.magic) >> F.magic_shift);
    }
}

template <int SCHEME>
__device__ __forceinline__ uint32_t stage_transform(const KernelFamily& F, uint32_t t, int* err) {
    if constexpr (SCHEME == S_4UBIT) {
        const uint32_t r = min3u(t, t - kP31, t - 2 * kP31);  // t mod p for any u32 t
        return r << 1;
    } else if constexpr (SCHEME == S_4UMOD) {
        return mod_barrett(t, F.p, F.barrett);
    } else if constexpr (SCHEME == S_PERM) {
        if ((uint64_t)t >= F.dim) {  // the reference reads out of bounds here (UB)
            atomicOr(err, 1);
            return 0;
        }
        return t;
    } else {
        return t;
    }
}

template <int SCHEME>
struct Coef;

template <>
struct Coef<S_2U> {
    uint32_t a1, a2;
    __device__ void load(const KernelFamily& F, uint32_t j) {
        const uint2 c = reinterpret_cast<const uint2*>(F.coef)[j];
        a1 = c.x;
        a2 = c.y;
    }
};

template <>
struct Coef<S_4UBIT> {
    uint32_t a3, c2, c1, c0;
    __device__ void load(const KernelFamily& F, uint32_t j) {
        const uint4 c = reinterpret_cast<const uint4*>(F.coef)[j];
        a3 = c.x;
        c2 = c.y;
        c1 = c.z;
        c0 = c.w;
    }
};

template <>
struct Coef<S_4UMOD> {
    uint32_t a3, a2, a1, a0;
    __device__ void load(const KernelFamily& F, uint32_t j) {
        const uint4 c = reinterpret_cast<const uint4*>(F.coef)[j];
        a3 = c.x;
        a2 = c.y;
        a1 = c.z;
        a0 = c.w;
    }
};

template <>
struct Coef<S_PERM> {
    const uint32_t* tab;
    __device__ void load(const KernelFamily& F, uint32_t j) { tab = F.perm + (uint64_t)j * F.dim; }
};

// One hash evaluation h_j(t) on the staged (transformed) id.
template <int SCHEME, bool POW2>
__device__ __forceinline__ uint32_t hash1(const KernelFamily& F, const Coef<SCHEME>& c,
                                          uint32_t t) {
    if constexpr (SCHEME == S_2U) {
        return c.a1 + c.a2 * t;  // natural 32-bit wrap; shift deferred to the minimum
    } else if constexpr (SCHEME == S_4UBIT) {
        uint32_t s = m31_fold(c.a3, t, c.c2);
        uint32_t h = min(s, s - kP31);  // lazy: h in [0, p+1]
        s = m31_fold(h, t, c.c1);
        h = min(s, s - kP31);
        s = m31_fold(h, t, c.c0);
        h = min3u(s, s - kP31, s - 2 * kP31);  // canonical in [0, p)
        return reduce_dim<POW2>(F, h);
    } else if constexpr (SCHEME == S_4UMOD) {
        uint32_t h = mod_barrett((uint64_t)c.a3 * t + c.a2, F.p, F.barrett);
        h = mod_barrett((uint64_t)h * t + c.a1, F.p, F.barrett);
        h = mod_barrett((uint64_t)h * t + c.a0, F.p, F.barrett);
        return reduce_dim<POW2>(F, h);
    } else {
        return __ldg(c.tab + t);
    }
}

// ---- TMA bulk copy + mbarrier helpers (sm_90+ PTX; SASS: UBLKCP / SYNCS) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// One unit of pipelined work: up to `tile` ids of one document.
struct Item {
    uint64_t doc;
    uint32_t cnt;    // ids in this tile (0 for an empty document)
    uint32_t head;   // garbage ids before the first one (16-byte alignment of the copy)
    uint32_t first;  // first tile of the document
    uint32_t last;   // last tile (run the epilogue)
    uint32_t empty;  // document has no ids
    uint32_t valid;  // 0 = no more work for this CTA
};

// each buffer holds tile + 8 ids: room for the 16-byte head/tail slack.
// The bulk copy spans whole 16-byte granules, so it may read up to 12 bytes
// past an item's last id (inside the same granule, never across a page); the
// values land in the slack and are overwritten by the padding. Every id
// buffer the library allocates has that slack (engine.cu kIdsSlack); callers
// of the device API are told so in bbmh_ext.h. (Splitting the tail off the
// copy cost 1.5-2% of 2U throughput through register allocation in the hash
// loop, profiles/r10/README.md.)

// Persistent sketch kernel. Each CTA walks documents blockIdx.x,
// blockIdx.x + gridDim.x, ... for hash-function tile blockIdx.y. Thread 0 is
// the producer: it issues one TMA bulk copy per item into one of two shared
// buffers (completion signalled on an mbarrier) one item ahead, so the next
// document's ids land while the current one is hashed.
// TRACE (tools/residency_probe.cu only): thread 0 of every CTA records its
// SM, start and end times (%globaltimer, ns) and the documents it finished.
template <int SCHEME, bool POW2, int J, bool TRACE = false>
__global__ void __launch_bounds__(256) sketch_kernel(KernelFamily F, const uint64_t* __restrict__ row_ptr,
                                                     uint64_t index_base,
                                                     const uint32_t* __restrict__ indices,
                                                     uint64_t n_docs, uint32_t b, uint32_t jtile,
                                                     uint32_t tile,
                                                     uint8_t* __restrict__ codes,
                                                     uint64_t* __restrict__ minima,
                                                     uint8_t* __restrict__ flags, int* err,
                                                     unsigned long long* cta_trace = nullptr) {
    extern __shared__ __align__(128) uint32_t smem[];
    const uint32_t kBuf = tile + 8;
    uint32_t* s_code = smem + 2 * kBuf;  // jtile codes
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ Item desc[2];

    if (F.yield_nnz && row_ptr[n_docs] - row_ptr[0] >= (uint64_t)F.yield_nnz * n_docs)
        return;  // the uniform kernel launched beside this one takes the batch
    const uint32_t tid = threadIdx.x;
    const uint32_t tpb = blockDim.x;
    const uint32_t k = F.k;
    const uint32_t j0 = blockIdx.y * jtile;
    [[maybe_unused]] unsigned long long trace_t0 = 0;
    [[maybe_unused]] uint32_t trace_docs = 0;
    if constexpr (TRACE) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(trace_t0));
    const uint32_t jcnt = min(jtile, k - j0);

    // ---- producer state (thread 0 only) ----
    // Documents go round-robin: CTA x takes x, x + gridDim.x, ... Under the
    // warp scheduler's priorities the CTAs sharing an SM drift apart (the
    // first finishes after a fifth of the kernel, tools/residency_probe.cu),
    // but the SM's pipes stay as busy with fewer resident CTAs: handing out
    // documents from an atomic ticket counter kept every CTA resident to the
    // end and gained 1.8%, yet its code cost the item loop its uniform control
    // flow (ptxas moved the loop bounds and LDS addresses from uniform to
    // vector registers: +4 IMAD per iteration), a net loss of 3%
    // (profiles/round2/dynamic_tickets_ab.jsonl).
    uint64_t p_doc = blockIdx.x, p_off = 0, p_beg = 0, p_end = 0;
    auto load_bounds = [&]() {
        if (p_doc < n_docs) {
            p_beg = row_ptr[p_doc];
            p_end = row_ptr[p_doc + 1];
            if (p_end < p_beg) {
                atomicOr(err, 2);
                p_end = p_beg;
            }
        }
    };
    auto issue = [&](int bi) {
        Item it{};
        if (p_doc >= n_docs) {
            it.valid = 0;
            desc[bi] = it;
            return;
        }
        const uint64_t nnz = p_end - p_beg;
        const uint64_t rem = nnz - p_off;
        it.valid = 1;
        it.doc = p_doc;
        it.first = p_off == 0;
        it.empty = nnz == 0;
        it.cnt = (uint32_t)(rem < tile ? rem : tile);
        it.last = p_off + it.cnt >= nnz;
        if (it.cnt) {
            const uint32_t* src = indices + (p_beg - index_base) + p_off;
            const uintptr_t a0 = (uintptr_t)src & ~(uintptr_t)15;
            it.head = (uint32_t)(((uintptr_t)src - a0) >> 2);
            const uint32_t bytes = ((it.head + it.cnt) * 4 + 15) & ~15u;
            // order earlier generic-proxy writes to this buffer before the async-proxy copy
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&mbar[bi], bytes);
            tma_bulk_g2s(smem + bi * kBuf, reinterpret_cast<const void*>(a0), bytes, &mbar[bi]);
        }
        desc[bi] = it;
        if (it.last) {
            p_doc += gridDim.x;
            p_off = 0;
            load_bounds();
        } else {
            p_off += it.cnt;
        }
    };

    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        load_bounds();
        issue(0);
    }
    __syncthreads();

    Coef<SCHEME> c[J];
    uint32_t m[J];
#pragma unroll
    for (int r = 0; r < J; ++r) {
        const uint32_t j = min(j0 + tid + r * tpb, k - 1);  // spare lanes recompute j = k-1
        c[r].load(F, j);
        m[r] = 0xffffffffu;
    }
    const uint32_t mask = b >= 32 ? 0xffffffffu : ((1u << b) - 1);
    const uint64_t cb = ((uint64_t)k * b + 7) >> 3;
    uint32_t phase = 0;  // bit i = parity of the next completion of mbar[i]

    for (uint32_t itn = 0;; ++itn) {
        const int bi = itn & 1;
        const Item d = desc[bi];
        if (!d.valid) break;
        if (tid == 0) issue(bi ^ 1);  // prefetch the next item into the other buffer
        if (d.first) {
#pragma unroll
            for (int r = 0; r < J; ++r) m[r] = 0xffffffffu;
        }
        if (d.cnt) {
            uint32_t* buf = smem + bi * kBuf;
            mbar_wait(&mbar[bi], (phase >> bi) & 1);
            phase ^= 1u << bi;
            const uint32_t lo = d.head, hi = d.head + d.cnt;
            const uint32_t n4 = (hi + 3) >> 2;
            constexpr bool kTransform = SCHEME != S_2U;
            if (kTransform || lo != 0 || (hi & 3) != 0) {
                // pad the alignment slack with a duplicate id (min unaffected) and
                // pre-transform ids in place (t mod p, doubled for 4U-bit)
                const uint32_t first = buf[lo];
                if (kTransform) __syncthreads();  // everyone read `first` before rewriting
                for (uint32_t i = tid; i < 4 * n4; i += tpb) {
                    const uint32_t t = (i < lo || i >= hi) ? first : buf[i];
                    if (kTransform || i < lo || i >= hi) buf[i] = stage_transform<SCHEME>(F, t, err);
                }
                __syncthreads();
            }
            const uint4* b4 = reinterpret_cast<const uint4*>(buf);
            // 2U: software-pipelined, the next quad loads under this one's IMADs (the
            // LDS latency was the top short-scoreboard stall); the 4U schemes have
            // enough arithmetic per quad to hide it and run slower with it
            constexpr bool kPrefetch = SCHEME == S_2U;
            uint4 tn = kPrefetch ? b4[0] : make_uint4(0, 0, 0, 0);
#pragma unroll(J >= 8 ? 2 : 4)
            for (uint32_t q = 0; q < n4; ++q) {
                uint4 t4;
                if constexpr (kPrefetch) {
                    t4 = tn;
                    tn = b4[min(q + 1, n4 - 1)];
                } else {
                    t4 = b4[q];
                }
#pragma unroll
                for (int r = 0; r < J; ++r) {
                    const uint32_t h0 = hash1<SCHEME, POW2>(F, c[r], t4.x);
                    const uint32_t h1 = hash1<SCHEME, POW2>(F, c[r], t4.y);
                    const uint32_t h2 = hash1<SCHEME, POW2>(F, c[r], t4.z);
                    const uint32_t h3 = hash1<SCHEME, POW2>(F, c[r], t4.w);
                    m[r] = min3u(m[r], h0, h1);
                    m[r] = min3u(m[r], h2, h3);
                }
            }
        }
        if (d.last) {
            // ---- epilogue: minima -> codes -> packed bitstream (sketch.cpp:80-98) ----
            if constexpr (TRACE) ++trace_docs;
            const uint64_t doc = d.doc;
            const bool empty = d.empty;
#pragma unroll
            for (int r = 0; r < J; ++r) {
                const uint32_t jl = tid + r * tpb;
                if (jl < jcnt) {
                    uint32_t mn = m[r];
                    if constexpr (SCHEME == S_2U) mn >>= F.shift2u;
                    s_code[jl] = empty ? mask : (mn & mask);
                    if (minima) minima[doc * k + j0 + jl] = empty ? ~0ull : (uint64_t)mn;
                }
            }
            if (flags && blockIdx.y == 0 && tid == 0) flags[doc] = empty ? 1 : 0;
            __syncthreads();
            const uint64_t byte0 = ((uint64_t)j0 * b) >> 3;  // j0*b is a multiple of 8
            const uint64_t byte1e = ((uint64_t)(j0 + jcnt) * b + 7) >> 3;
            const uint64_t byte1 = byte1e < cb ? byte1e : cb;
            uint8_t* out = codes + doc * cb;
            for (uint64_t B = byte0 + tid; B < byte1; B += tpb) {
                const uint64_t bit0 = B << 3;
                const uint32_t ja = (uint32_t)(bit0 / b);
                const uint64_t jb0 = (bit0 + 7) / b, jlast = (uint64_t)j0 + jcnt - 1;
                const uint32_t jb = (uint32_t)(jb0 < jlast ? jb0 : jlast);
                uint32_t v = 0;
                for (uint32_t j = ja; j <= jb; ++j) {
                    const uint64_t code = s_code[j - j0];
                    const int64_t pos = (int64_t)j * b - (int64_t)bit0;
                    v |= (uint32_t)(pos >= 0 ? (code << pos) : (code >> -pos));
                }
                out[B] = (uint8_t)v;
            }
        }
        __syncthreads();  // buffer bi and s_code free; desc[bi ^ 1] visible
    }
    if constexpr (TRACE) {
        if (tid == 0) {
            unsigned long long t1;
            uint32_t smid;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            unsigned long long* o = cta_trace + 4 * ((uint64_t)blockIdx.y * gridDim.x + blockIdx.x);
            o[0] = smid;
            o[1] = trace_t0;
            o[2] = t1;
            o[3] = trace_docs;
        }
    }
}

// ---- small k (<= 32 for 2U, <= 16 for 4U): split the ids across lanes --------
// With k < 32 the layout above leaves 32 - k lanes of each warp idle and every
// busy lane walks all ids of the document alone (latency-bound: 2U at k = 1..32
// ran at 19% of HBM, 4U-bit at 2%). Here every lane holds all k <= J hash
// functions and takes every 32nd quad of the document's ids, read straight
// from global memory with 16-byte loads (each id read once, coalesced across
// the warp); the 32 partial minima per function are merged with shuffles.
// Each warp sketches its own documents. Same arithmetic and epilogue as
// sketch_kernel.
template <int SCHEME, bool POW2, int J>
__global__ void __launch_bounds__(128) sketch_split_kernel(KernelFamily Fm,
                                                           const uint64_t* __restrict__ row_ptr,
                                                           uint64_t index_base,
                                                           const uint32_t* __restrict__ indices,
                                                           uint64_t n_docs, uint32_t b,
                                                           uint8_t* __restrict__ codes,
                                                           uint64_t* __restrict__ minima,
                                                           uint8_t* __restrict__ flags, int* err,
                                                           unsigned long long* work) {
    __shared__ uint32_t s_code[4][J];
    if (Fm.yield_nnz && row_ptr[n_docs] - row_ptr[0] >= (uint64_t)Fm.yield_nnz * n_docs)
        return;  // the uniform kernel launched beside this one takes the batch
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
    const uint32_t k = Fm.k;
    Coef<SCHEME> c[J];
#pragma unroll
    for (int r = 0; r < J; ++r) c[r].load(Fm, (uint32_t)r < k ? r : k - 1);
    const uint32_t mask = b >= 32 ? 0xffffffffu : ((1u << b) - 1);
    const uint64_t cb = ((uint64_t)k * b + 7) >> 3;
    // kQ quads per lane per step, the next step's loaded under this one's
    // hashing, and the next document's first step under this one's merge and
    // epilogue (with one step's loads in flight per warp the k = 8 launch
    // reached 68% of HBM)
    constexpr int kQ = SCHEME == S_2U && J <= 8 ? 4 : 2;  // quads per lane per step
    const uint64_t stride = (uint64_t)gridDim.x * W;
    const uint32_t* ids = nullptr;
    uint64_t nnz = 0, head = 0, nq = 0;
    const uint4* q4 = nullptr;
    uint4 nx[kQ];
    auto describe = [&](uint64_t d) {  // document d's id ranges and first step
        uint64_t beg = row_ptr[d], end = row_ptr[d + 1];
        if (end < beg) {
            if (lane == 0) atomicOr(err, 2);
            end = beg;
        }
        ids = indices + (beg - index_base);
        nnz = end - beg;
        // head ids up to 16-byte alignment, whole quads, tail ids
        const uint64_t h = ((16 - ((uintptr_t)ids & 15)) & 15) / 4;
        head = nnz < h ? nnz : h;
        nq = (nnz - head) / 4;
        q4 = reinterpret_cast<const uint4*>(ids + head);
#pragma unroll
        for (int i = 0; i < kQ; ++i)
            nx[i] = lane + 32 * i < nq ? __ldg(q4 + lane + 32 * i) : make_uint4(0, 0, 0, 0);
    };
    // documents after the first wave come from a ticket counter, one ticket
    // ahead; round-robin without `work`
    auto fetch_next = [&](uint64_t cur) -> uint64_t {
        if (!work) return cur + stride;
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(&work[0], 1ull);
        return stride + __shfl_sync(0xffffffffu, t, 0);
    };
    uint64_t doc = (uint64_t)blockIdx.x * W + warp;
    uint64_t nxt = doc < n_docs ? fetch_next(doc) : n_docs;
    if (doc < n_docs) describe(doc);
    for (; doc < n_docs; doc = nxt, nxt = doc < n_docs ? fetch_next(doc) : n_docs) {
        uint32_t m[J];
#pragma unroll
        for (int r = 0; r < J; ++r) m[r] = 0xffffffffu;
        auto eval = [&](uint32_t t) {
            const uint32_t tt = stage_transform<SCHEME>(Fm, t, err);
#pragma unroll
            for (int r = 0; r < J; ++r) m[r] = min(m[r], hash1<SCHEME, POW2>(Fm, c[r], tt));
        };
        if (lane < head) eval(__ldg(ids + lane));
        for (uint64_t q = lane; q < nq; q += 32 * kQ) {
            uint4 cx[kQ];
#pragma unroll
            for (int i = 0; i < kQ; ++i) {
                cx[i] = nx[i];
                if (q + 32 * (kQ + i) < nq) nx[i] = __ldg(q4 + q + 32 * (kQ + i));
            }
#pragma unroll
            for (int i = 0; i < kQ; ++i) {
                if (i == 0 || q + 32 * i < nq) {
                    eval(cx[i].x);
                    eval(cx[i].y);
                    eval(cx[i].z);
                    eval(cx[i].w);
                }
            }
        }
        const uint64_t t0 = head + 4 * nq;
        if (t0 + lane < nnz) eval(__ldg(ids + t0 + lane));
        const bool empty = nnz == 0;
        if (nxt < n_docs) describe(nxt);  // loads in flight during the merge
        // merge the 32 lanes' minima, function by function
#pragma unroll
        for (int r = 0; r < J; ++r) {
#pragma unroll
            for (uint32_t off = 1; off < 32; off <<= 1)
                m[r] = min(m[r], __shfl_xor_sync(0xffffffffu, m[r], off));
            if constexpr (SCHEME == S_2U) m[r] >>= Fm.shift2u;
        }
        if (lane == 0) {
#pragma unroll
            for (int r = 0; r < J; ++r)
                if ((uint32_t)r < k) s_code[warp][r] = empty ? mask : (m[r] & mask);
            if (flags) flags[doc] = empty ? 1 : 0;
        }
        if (minima) {
#pragma unroll
            for (int r = 0; r < J; ++r)
                if (lane == (uint32_t)r && (uint32_t)r < k)
                    minima[doc * k + r] = empty ? ~0ull : (uint64_t)m[r];
        }
        __syncwarp();
        uint8_t* out = codes + doc * cb;
        for (uint64_t B = lane; B < cb; B += 32) {
            const uint64_t bit0 = B << 3;
            const uint32_t ja = (uint32_t)(bit0 / b);
            const uint64_t jb0 = (bit0 + 7) / b;
            const uint32_t jb = (uint32_t)(jb0 < k - 1 ? jb0 : k - 1);
            uint32_t v = 0;
            for (uint32_t j = ja; j <= jb; ++j) {
                const uint64_t code = s_code[warp][j];
                const int64_t pos = (int64_t)j * b - (int64_t)bit0;
                v |= (uint32_t)(pos >= 0 ? (code << pos) : (code >> -pos));
            }
            out[B] = (uint8_t)v;
        }
        __syncwarp();
    }
    if (work && lane == 0) {  // the last warp out resets the counters
        __threadfence();
        if (atomicAdd(&work[1], 1ull) == stride - 1) {
            work[0] = 0;
            work[1] = 0;
        }
    }
}

// Ticket counters of the small-k kernel (see sketch_split_kernel): a pool
// of zeroed {ticket, exit} pairs per device, taken round-robin per launch;
// each launch leaves its pair zeroed, and a pair is reused only 1,023
// launches later.
unsigned long long* work_slot(int dev, int pairs = 1) {
    constexpr int kSlots = 1024;
    static std::mutex mu;
    static std::map<int, unsigned long long*> pools;
    static std::atomic<uint64_t> seq{0};
    unsigned long long* pool = nullptr;
    {
        std::lock_guard lk(mu);
        auto it = pools.find(dev);
        if (it == pools.end()) {
            if (cudaMalloc(&pool, kSlots * 2 * sizeof(unsigned long long)) != cudaSuccess ||
                cudaMemset(pool, 0, kSlots * 2 * sizeof(unsigned long long)) != cudaSuccess) {
                cudaGetLastError();
                if (pool) cudaFree(pool);
                return nullptr;  // static assignment
            }
            it = pools.emplace(dev, pool).first;
        }
        pool = it->second;
    }
    // `pairs` consecutive pairs, not wrapping past the end of the pool
    uint64_t at = seq.fetch_add(pairs, std::memory_order_relaxed) % kSlots;
    if (at + pairs > kSlots) at = 0;
    return pool + 2 * at;
}

template <int SCHEME, bool POW2, int J, bool TRACE = false>
void launch_one(const KernelFamily& F, const LaunchShape& sh, const uint64_t* row_ptr,
                uint64_t base, const uint32_t* idx, uint64_t n, uint32_t b, uint8_t* codes,
                uint64_t* minima, uint8_t* flags, int* err, cudaStream_t st,
                unsigned long long* cta_trace = nullptr) {
    auto kern = sketch_kernel<SCHEME, POW2, J, TRACE>;
    // 1,024-id tiles for 2U and for 4U below 256 threads per CTA: 4U CTAs of one
    // or two warps with 4,096-id tiles are held to ~7 per SM by shared memory
    // (k = 32: 0.91 -> 1.25 T evals/s, k = 64: 0.95 -> 1.31; tools/grid_4u_tiles.json)
    const bool small_tile = SCHEME == S_2U || ((SCHEME == S_4UBIT || SCHEME == S_4UMOD) && sh.tpb < 256);
    int tile = (int)opt(Opt::Tile);
    if (tile <= 0) tile = small_tile ? 1024 : (int)kDefaultTile;
    tile = tile < 64 ? 64 : tile > 16384 ? 16384 : tile & ~3;
    const size_t smem = (2 * (tile + 8) + sh.jtile) * sizeof(uint32_t);
    int dev = 0;
    cudaGetDevice(&dev);
    // occupancy/attribute queries cost several microseconds each: do them once
    // per (kernel instance, device, block shape, smem)
    static std::mutex mu;
    static std::map<std::tuple<int, int, size_t, int>, std::pair<int, int>> cache;  // -> (sms, occ)
    int sms = 148, occ = 1;
    const int carveout = (int)opt(Opt::Carveout);
    {
        std::lock_guard lk(mu);
        auto key = std::make_tuple(dev, sh.tpb, smem, carveout);
        auto it = cache.find(key);
        if (it == cache.end()) {
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            // the attribute is a per-function ceiling: set it to the device's
            // opt-in maximum, not to this shape's smem, or a later launch of a
            // larger shape of the same kernel would fail with invalid argument
            // (opt-in block limit minus the kernel's static shared memory)
            int optin = 0;
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, kern);
            const int dyn_max = optin - (int)fa.sharedSizeBytes;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 dyn_max > (int)smem ? dyn_max : (int)smem);
            // The persistent grid is sized to the occupancy limit, so the
            // shared-memory carveout the driver picks at launch must admit
            // that many CTAs; -1 leaves the choice to the driver.
            cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 carveout >= 0 && carveout <= 100 ? carveout : -1);
            cudaGetLastError();
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, sh.tpb, smem);
            occ = occ < 1 ? 1 : occ;
            it = cache.emplace(key, std::make_pair(sms, occ)).first;
        }
        sms = it->second.first;
        occ = it->second.second;
    }
    // One-warp CTAs of the wide-J 2U shapes (k = 200: J = 7; k = 256: J = 8)
    // run 8% faster at 20 CTAs per SM than at the 24 shared memory allows;
    // the thin-J ones (k <= 128) run 8% slower with that cap
    // (tools/grid_2u_cap.json, profiles/r11/ksweep_cap.txt).
    if (SCHEME == S_2U && J >= 7 && sh.tpb == 32 && opt(Opt::SmemCap))
        occ = std::min(occ, 20);
    const int ctas_cap = (int)opt(Opt::CtasPerSm);
    if (ctas_cap > 0 && ctas_cap < occ) occ = ctas_cap;
    // persistent: one wave of CTAs per j-tile, each looping over documents
    uint64_t gx = (uint64_t)sms * occ / sh.jtiles;
    if (gx < 1) gx = 1;
    if (gx > n) gx = n;
    dim3 grid((unsigned)gx, sh.jtiles);
    const cudaError_t pre = cudaPeekAtLastError();
    kern<<<grid, sh.tpb, smem, st>>>(F, row_ptr, base, idx, n, b, sh.jtile, (uint32_t)tile, codes,
                                     minima, flags, err, cta_trace);
    if (const cudaError_t e = cudaPeekAtLastError(); e != cudaSuccess)
        fprintf(stderr, "bbmh: sketch launch failed (%s; before launch: %s) grid %u x %u tpb %d smem %zu\n",
                cudaGetErrorString(e), cudaGetErrorString(pre), grid.x, grid.y, sh.tpb, smem);
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

template <int SCHEME, bool POW2>
void dispatch_j(const KernelFamily& F, const LaunchShape& sh, const uint64_t* row_ptr,
                uint64_t base, const uint32_t* idx, uint64_t n, uint32_t b, uint8_t* codes,
                uint64_t* minima, uint8_t* flags, int* err, cudaStream_t st) {
    switch (sh.J) {
        case 1: return launch_one<SCHEME, POW2, 1>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
        case 2: return launch_one<SCHEME, POW2, 2>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
        case 4: return launch_one<SCHEME, POW2, 4>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
        case 8: return launch_one<SCHEME, POW2, 8>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
        case 7:
            if constexpr (SCHEME != S_PERM)
                return launch_one<SCHEME, POW2, 7>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
            return launch_one<SCHEME, POW2, 8>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
        case 5:
            if constexpr (SCHEME == S_2U)
                return launch_one<SCHEME, POW2, 5>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
            return launch_one<SCHEME, POW2, 8>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
        case 6:
            if constexpr (SCHEME == S_2U)
                return launch_one<SCHEME, POW2, 6>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
            return launch_one<SCHEME, POW2, 8>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
        default: return launch_one<SCHEME, POW2, 16>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
    }
}


template <int SCHEME, bool POW2, int FF>
void launch_split(const KernelFamily& F, const uint64_t* row_ptr, uint64_t base,
                  const uint32_t* idx, uint64_t n, uint32_t b, uint8_t* codes, uint64_t* minima,
                  uint8_t* flags, int* err, cudaStream_t st) {
    constexpr int kTpb = 128;  // 4 warps, each on its own documents
    static std::atomic<int> occ_cache{0};
    int occ = occ_cache.load(std::memory_order_relaxed);
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sketch_split_kernel<SCHEME, POW2, FF>,
                                                      kTpb, 0);
        occ = occ < 1 ? 1 : occ;
        occ_cache.store(occ, std::memory_order_relaxed);
    }
    uint64_t grid = (uint64_t)device_sms() * occ;
    const uint64_t need = (n + 3) / 4;
    if (grid > need) grid = need;
    int dev = 0;
    cudaGetDevice(&dev);
    // Tickets: +7-17% for 2U at k = 8..32 and 4U at k = 1..16 (the warps
    // sharing an SM drift apart under round-robin assignment), but at 2U
    // k <= 2 a document is so short that the single counter serialises the
    // warps (k = 1: 1.73 -> 1.11 T evals/s): those stay round-robin
    // (profiles/round2/dynamic_tickets_smallk_ab.jsonl).
    const bool tickets = opt(Opt::DynamicDocs) && !(SCHEME == S_2U && FF <= 2);
    unsigned long long* work = tickets ? work_slot(dev) : nullptr;
    sketch_split_kernel<SCHEME, POW2, FF><<<(unsigned)grid, kTpb, 0, st>>>(
        F, row_ptr, base, idx, n, b, codes, minima, flags, err, work);
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

template <int SCHEME, bool POW2>
void dispatch_split(const KernelFamily& F, const uint64_t* row_ptr, uint64_t base,
                    const uint32_t* idx, uint64_t n, uint32_t b, uint8_t* codes, uint64_t* minima,
                    uint8_t* flags, int* err, cudaStream_t st) {
    const uint32_t k = F.k;
    if (k <= 1) return launch_split<SCHEME, POW2, 1>(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
    if (k <= 2) return launch_split<SCHEME, POW2, 2>(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
    if (k <= 4) return launch_split<SCHEME, POW2, 4>(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
    if (k <= 8) return launch_split<SCHEME, POW2, 8>(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
    if constexpr (SCHEME == S_2U)
        if (k > 16) return launch_split<SCHEME, POW2, 32>(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
    return launch_split<SCHEME, POW2, 16>(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
}

}  // namespace

int sm_count() { return device_sms(); }
unsigned long long* ticket_slot(int dev) { return work_slot(dev); }
unsigned long long* ticket_block(int dev, int pairs) { return work_slot(dev, pairs); }

LaunchShape choose_shape(uint32_t k, int scheme, uint64_t n, int sms) {
    // Each thread owns J hash functions and streams every staged id, so its
    // serial work is ~J * eff per id, where eff is the measured relative
    // inefficiency of small J (one LDS.128 feeds 4*J evaluations;
    // tools/tune.py, profiles/r02): 2U is issue-bound so J = 1 costs ~35% and
    // J = 8 is best; 4U is arithmetic-bound and flat in J. An SM saturates at
    // about kSatThreads threads; below that, time is the per-thread serial
    // work. Model: time ~ J * eff * max(1, threads / (sms * kSatThreads)),
    // with threads = n * tiles * tpb. For large batches this is the lane-slot
    // cost (idle j >= k lanes included); for small online batches it prefers
    // more, thinner j-tiles so the batch still fills the GPU. Ties prefer
    // fewer CTAs per document.
    // 4U's fold chains need more resident threads before an SM saturates:
    // with 384 the model kept small online batches (a few hundred documents
    // per chunk) on one 512-lane tile per document and half the SMs idle
    // (C5 4U-bit, 1,024 docs: 1.92 -> 1.62 ms with two 256-lane tiles,
    // profiles/round2/c5_4u_shapes.jsonl). Large batches fill every SM under
    // either figure, so their shapes do not change.
    const double kSatThreads = (scheme == S_4UBIT || scheme == S_4UMOD) ? 1024 : 384;
    const double docs = n ? (double)n : 1e12;
    LaunchShape best;
    double best_cost = 1e300;
    // J = 7: 7 x 32 = 224 lanes fit k = 200 (config 1) with 11% idle instead of
    // 22% at 256 (4U at k = 200: 1.02 -> 1.19 T evals/s against J = 1 x 224,
    // tools/grid_4u_k200b.json)
    // J = 5, 6 (2U): 5 x 64 = 320 lanes fit k = 300 (9.2 -> 12.8 T evals/s), and
    // 5 x 32 = 160 fit k = 160 (9.0 -> 12.9; tools/grid_2u_k300.json). The 2U
    // costs of thin J are measured (k = 64 with J = 2: 1.28; k = 300 with J = 2
    // x 160 threads: ~1.5).
    const int Js[7] = {8, 7, 6, 5, 4, 2, 1};
    for (int J : Js) {
        if (J == 7 && scheme == S_PERM) continue;
        if ((J == 5 || J == 6) && scheme != S_2U) continue;
        const double eff = scheme == S_2U ? (J == 8 ? 1.0 : J == 7 ? 1.02 : J == 6 ? 1.03 : J == 5 ? 1.08
                                             : J == 4 ? 1.10 : J == 2 ? 1.3 : 1.35)
                                          : (J == 2 || J == 7 ? 1.0 : J == 4 ? 1.01 : J == 8 ? 1.02 : 1.02);
        for (int tpb = 32; tpb <= 256; tpb += 32) {
            const uint64_t jtile = (uint64_t)tpb * J;
            const uint64_t tiles = (k + jtile - 1) / jtile;
            if (tiles > 65535) continue;
            const double threads = docs * (double)tiles * tpb;
            const double fill = threads / ((double)sms * kSatThreads);
            const double cost = J * eff * (fill > 1.0 ? fill : 1.0) * (1.0 + 0.01 * (double)tiles);
            if (cost < best_cost * (1.0 - 1e-9)) {
                best_cost = cost;
                best.J = J;
                best.tpb = tpb;
                best.jtile = (uint32_t)jtile;
                best.jtiles = (uint32_t)tiles;
            }
        }
    }
    // tuning switches (bbmh_ext_set_option "shape_j" / "shape_tpb")
    const int J = (int)opt(Opt::ShapeJ), tpb = (int)opt(Opt::ShapeTpb);
    if ((J == 1 || J == 2 || J == 4 || J == 8 || (J == 7 && scheme != S_PERM) ||
         ((J == 5 || J == 6) && scheme == S_2U)) && tpb >= 32 &&
        tpb <= 256 && tpb % 32 == 0) {
        best.J = J;
        best.tpb = tpb;
        best.jtile = (uint32_t)(J * tpb);
        best.jtiles = (k + best.jtile - 1) / best.jtile;
    }
    return best;
}

void launch_sketch(const KernelFamily& F, const uint64_t* row_ptr, uint64_t base,
                   const uint32_t* idx, uint64_t n, uint32_t b, uint8_t* codes, uint64_t* minima,
                   uint8_t* flags, int* err, cudaStream_t st, double avg_nnz) {
    if (n == 0) return;
    const uint32_t split_max = F.scheme == S_2U ? 32u : 16u;  // functions a lane holds in registers
    // 2U at 16 < k < 32: the coefficient-uniform kernel when the rows are
    // long enough (uniform.cu), the lane-split kernel otherwise; with device
    // row_ptr both are launched and the batch's mean row length on the
    // device decides which one returns at once
    const uint32_t need_small = F.scheme == S_2U && F.k <= split_max ? uniform_min_nnz(F, n) : 0;
    const bool uniform_small = need_small && avg_nnz >= need_small;
    if (F.k <= split_max && F.scheme != S_PERM && opt(Opt::SplitSmallK) && !uniform_small) {
        switch (F.scheme) {
            case S_2U:
                if (need_small && avg_nnz < 0) {
                    launch_uniform_2u(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st, need_small);
                    KernelFamily Fy = F;
                    Fy.yield_nnz = need_small;
                    return dispatch_split<S_2U, true>(Fy, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
                }
                return dispatch_split<S_2U, true>(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
            case S_4UBIT:
                if (F.dim_pow2)
                    return dispatch_split<S_4UBIT, true>(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
                return dispatch_split<S_4UBIT, false>(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
            default:
                if (F.dim_pow2)
                    return dispatch_split<S_4UMOD, true>(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
                return dispatch_split<S_4UMOD, false>(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
        }
    }
    const LaunchShape sh = choose_shape(F.k, F.scheme, n, device_sms());
    switch (F.scheme) {
        case S_2U: {
            const uint32_t need = uniform_min_nnz(F, n);
            if (!need) return dispatch_j<S_2U, true>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
            if (avg_nnz >= 0) {
                if (avg_nnz >= need)
                    return launch_uniform_2u(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st, 0);
                return dispatch_j<S_2U, true>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
            }
            // row lengths unknown on the host: both kernels, one returns at once
            launch_uniform_2u(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st, need);
            KernelFamily Fy = F;
            Fy.yield_nnz = need;
            return dispatch_j<S_2U, true>(Fy, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
        }
        case S_4UBIT:
            if (uniform4_applies(F, n))
                return launch_uniform_4u(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
            if (F.dim_pow2)
                return dispatch_j<S_4UBIT, true>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
            return dispatch_j<S_4UBIT, false>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
        case S_4UMOD:
            if (F.dim_pow2)
                return dispatch_j<S_4UMOD, true>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
            return dispatch_j<S_4UMOD, false>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
        default:
            // L2-resident table-outer schedule (perm.cu)
            if (perm_tablewise_applies(F, n) &&
                launch_perm_tablewise(F, row_ptr, base, idx, n, b, codes, minima, flags, err, st))
                return;
            return dispatch_j<S_PERM, true>(F, sh, row_ptr, base, idx, n, b, codes, minima, flags, err, st);
    }
}

uint64_t kernel_launch_count() { return g_launches.load(); }

void count_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {
std::atomic<uint64_t> g_h2d{0}, g_d2h{0};
}  // namespace

void count_transfer(uint64_t h2d, uint64_t d2h) {
    g_h2d.fetch_add(h2d, std::memory_order_relaxed);
    g_d2h.fetch_add(d2h, std::memory_order_relaxed);
}

void transfer_counts(uint64_t& h2d, uint64_t& d2h) {
    h2d = g_h2d.load();
    d2h = g_d2h.load();
}

namespace {
std::atomic<uint64_t> g_counters[int(Counter::kCount)];
constexpr const char* kCounterNames[] = {"peer_copy_bytes", "zero_copy_calls", "delta16_chunks",
                                         "raw_chunks", "range_shards", "device_id_batches",
                                         "uniform_launches"};
static_assert(sizeof(kCounterNames) / sizeof(kCounterNames[0]) == size_t(Counter::kCount));
}  // namespace

void count(Counter c, uint64_t n) { g_counters[int(c)].fetch_add(n, std::memory_order_relaxed); }

bool counter_value(const char* name, uint64_t* out) {
    if (!name) return false;
    const std::string s = name;
    uint64_t v = 0;
    if (s == "kernel_launches") {
        v = g_launches.load();
    } else if (s == "h2d_bytes") {
        v = g_h2d.load();
    } else if (s == "d2h_bytes") {
        v = g_d2h.load();
    } else {
        int i = 0;
        while (i < int(Counter::kCount) && s != kCounterNames[i]) ++i;
        if (i == int(Counter::kCount)) return false;
        v = g_counters[i].load();
    }
    if (out) *out = v;
    return true;
}

}  // namespace bbmh
