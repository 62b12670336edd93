// vw.cu -- VW signed random-bin projection on the GPU.
//
// Reference: VwProjector (vw.cpp:11-59) and vw_project_file (vw.cpp:61-77):
//   bin(t)  = eval_2u over `bins` (power of two) with coefficients
//             keyed_u64(seed, 7, 0, {0,1}) (a2 forced odd);
//   sign(t) = +1 if the 4U polynomial mod 2^31-1 (coefficients drawn from
//             keyed_u64(seed, 8, attempt, i) >> 33 below p) is odd, else -1;
//   a row becomes the ascending list of bins whose signed counts are non-zero,
//   written as LibSVM text "%+d" + " %u:%g" (bin + 1, count) per entry.
// GPU path per batch of rows (vw_row_kernel): one CTA per row hashes its ids
// into keys bin << 1 | (sign > 0), sorts them with a bitonic network in shared
// memory (rows longer than the shared buffer use a global scratch of the same
// layout), and sums the signs of each run of equal bins; the non-zero runs are
// written in bin order at the row's offset. Signed counts are exact integers,
// so the summation order does not matter. The host formats the rows in order.
#include <cuda_runtime.h>

#include <bit>
#include <cmath>
#include <cstring>
#include <algorithm>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "engine.hpp"
#include "io.hpp"
#include "pipeline.hpp"

namespace bbmh {

namespace {

constexpr uint32_t kP31 = 0x7fffffffu;

struct VwCoef {
    uint32_t a1, a2, shift;        // bin hash (2U)
    uint32_t s3, s2x2, s1x2, s0x2;  // sign hash (4U): a3 and doubled a2, a1, a0
};

__device__ __forceinline__ uint32_t fold31(uint32_t h, uint32_t t2, uint32_t c) {
    const uint64_t v = (uint64_t)h * t2 + c;  // 2(h t + a): (v >> 31) hi, (v & p) << 1 lo
    return (uint32_t)(v >> 32) + ((uint32_t)v >> 1);
}

constexpr uint32_t kVwThreads = 256;
constexpr uint32_t kVwSmemKeys = 8192;  // rows up to this many ids sort in shared memory

// bin << 1 | (sign > 0). A bin has up to 32 bits: with bins = 1 the 2U hash is
// shifted by 32, which the reference's x86 build executes as a shift by 0.
__device__ __forceinline__ unsigned long long vw_key(const VwCoef& c, uint32_t t) {
    const uint32_t h2 = c.a1 + c.a2 * t;
    const uint32_t bin = c.shift ? h2 >> c.shift : h2;
    const uint32_t t2 = t << 1;
    uint32_t s = fold31(c.s3, t2, c.s2x2);
    uint32_t h = min(s, s - kP31);
    s = fold31(h, t2, c.s1x2);
    h = min(s, s - kP31);
    s = fold31(h, t2, c.s0x2);
    h = min(min(s, s - kP31), s - 2 * kP31);
    return (unsigned long long)bin << 1 | (h & 1);
}

// One CTA per row (grid-stride): keys -> bitonic sort -> signed run sums ->
// the row's non-zero (bin, count) entries in bin order at out[row_ptr[r]..],
// their number in counts[r]. `scratch` (row_ptr-indexed, 2x the ids) holds
// the keys of rows longer than the shared buffer.
__global__ void __launch_bounds__(kVwThreads) vw_row_kernel(const uint64_t* __restrict__ row_ptr,
                                                            uint64_t n, const uint32_t* __restrict__ ids,
                                                            VwCoef c, unsigned long long* __restrict__ scratch,
                                                            uint32_t* __restrict__ out_bins,
                                                            int* __restrict__ out_sums,
                                                            uint32_t* __restrict__ counts, int* err) {
    extern __shared__ unsigned long long s_keys[];  // kVwSmemKeys
    __shared__ uint32_t s_cnt[kVwThreads];
    const uint32_t tid = threadIdx.x;
    for (uint64_t r = blockIdx.x; r < n; r += gridDim.x) {
        const uint64_t beg = row_ptr[r], end = row_ptr[r + 1];
        const uint32_t len = (uint32_t)(end - beg);
        uint32_t P = 1;
        while (P < len) P <<= 1;
        unsigned long long* keys = P <= kVwSmemKeys ? s_keys : scratch + 2 * beg;
        for (uint32_t i = tid; i < P; i += kVwThreads) {
            unsigned long long k = ~0ull;  // padding sorts last (above any bin << 1 | sign)
            if (i < len) {
                uint32_t t = ids[beg + i];
                if (t >= kP31) {  // the reference fails here (vw.cpp:38-40); the host stops at this row
                    atomicOr(err, 1);
                    t = 0;
                }
                k = vw_key(c, t);
            }
            keys[i] = k;
        }
        __syncthreads();
        // bitonic sort, ascending
        for (uint32_t kk = 2; kk <= P; kk <<= 1) {
            for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
                for (uint32_t i = tid; i < P; i += kVwThreads) {
                    const uint32_t ixj = i ^ j;
                    if (ixj > i) {
                        const unsigned long long a = keys[i], b = keys[ixj];
                        const bool up = (i & kk) == 0;
                        if ((a > b) == up) {
                            keys[i] = b;
                            keys[ixj] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
        // each thread takes a contiguous chunk of positions; a run belongs to
        // the chunk holding its first key and is summed by walking it
        const uint32_t chunk = (len + kVwThreads - 1) / kVwThreads;
        const uint32_t p0 = min(len, tid * chunk), p1 = min(len, p0 + chunk);
        auto run_sum = [&](uint32_t i, uint32_t& next) {
            const unsigned long long bin = keys[i] >> 1;
            int sum = 0;
            uint32_t q = i;
            for (; q < len && (keys[q] >> 1) == bin; ++q) sum += (keys[q] & 1) ? 1 : -1;
            next = q;
            return sum;
        };
        uint32_t mine = 0;
        for (uint32_t i = p0; i < p1;) {
            if (i > 0 && (keys[i] >> 1) == (keys[i - 1] >> 1)) {
                ++i;
                continue;
            }
            uint32_t nx;
            mine += run_sum(i, nx) != 0;
            i = nx;
        }
        s_cnt[tid] = mine;
        __syncthreads();
        // exclusive scan of the per-thread counts (256: one warp per step)
        if (tid < 32) {
            uint32_t v[kVwThreads / 32], acc = 0;
#pragma unroll
            for (int w = 0; w < (int)(kVwThreads / 32); ++w) {
                v[w] = s_cnt[tid * (kVwThreads / 32) + w];
                acc += v[w];
            }
            uint32_t incl = acc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= (uint32_t)o) incl += y;
            }
            uint32_t run = incl - acc;
#pragma unroll
            for (int w = 0; w < (int)(kVwThreads / 32); ++w) {
                const uint32_t x = v[w];
                s_cnt[tid * (kVwThreads / 32) + w] = run;
                run += x;
            }
            if (tid == 31) counts[r] = incl;
        }
        __syncthreads();
        uint32_t pos = s_cnt[tid];
        for (uint32_t i = p0; i < p1;) {
            if (i > 0 && (keys[i] >> 1) == (keys[i - 1] >> 1)) {
                ++i;
                continue;
            }
            uint32_t nx;
            const int sum = run_sum(i, nx);
            if (sum != 0) {
                out_bins[beg + pos] = uint32_t(keys[i] >> 1);
                out_sums[beg + pos] = sum;
                ++pos;
            }
            i = nx;
        }
        __syncthreads();  // keys / s_cnt are reused by the next row
    }
}

// page-locked host array (D2H at full PCIe rate, no zero-fill of a std::vector)
template <typename T>
struct HostBuf {
    T* p = nullptr;
    size_t cap = 0;
    void reserve(size_t n) {
        if (n <= cap) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = std::max<size_t>(n, cap + cap / 2);
        BBMH_CUDA(cudaMallocHost(&p, cap * sizeof(T)));
    }
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
    T& operator[](size_t i) { return p[i]; }
    const T& operator[](size_t i) const { return p[i]; }
};

template <typename T>
struct Buf {
    T* p = nullptr;
    size_t cap = 0;
    void reserve(size_t n) {
        if (n <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        cap = std::max<size_t>(n, cap + cap / 2);
        BBMH_CUDA(cudaMalloc(&p, cap * sizeof(T)));
    }
    ~Buf() {
        if (p) cudaFree(p);
    }
};

// VwProjector ctor (vw.cpp:11-26)
VwCoef make_coef(uint32_t bins, uint64_t seed) {
    if (bins < 1 || (bins & (bins - 1)) != 0)
        fail(Errc::UnsupportedUniverse, "bin count must be a power of two");
    const uint32_t s = uint32_t(std::countr_zero(bins));
    VwCoef c{};
    c.a1 = uint32_t(keyed_u64(seed, 7, 0, 0));
    c.a2 = uint32_t(keyed_u64(seed, 7, 0, 1)) | 1u;
    c.shift = (32 - s) & 31;  // eval_2u's h >> (32 - s); s = 0 shifts by 32 (see Family::map)
    uint64_t a[4];
    for (uint64_t i = 0; i < 4; ++i) {
        uint64_t v, attempt = 0;
        do {
            v = keyed_u64(seed, 8, attempt++, i) >> 33;
        } while (v >= kMersenne31);
        a[i] = v;
    }
    c.s3 = uint32_t(a[3]);
    c.s2x2 = uint32_t(2 * a[2]);
    c.s1x2 = uint32_t(2 * a[1]);
    c.s0x2 = uint32_t(2 * a[0]);
    return c;
}

inline char* put_uint(char* p, uint64_t v) {
    char tmp[24];
    int n = 0;
    do {
        tmp[n++] = char('0' + v % 10);
        v /= 10;
    } while (v);
    while (n) *p++ = tmp[--n];
    return p;
}

}  // namespace

uint64_t vw_project_file(const std::string& corpus_path, const std::string& out_path,
                         uint32_t bins, uint64_t seed) {
    const VwCoef coef = make_coef(bins, seed);
    auto reader = open_corpus(corpus_path, 8);
    FILE* out = std::fopen(out_path.c_str(), "wb");
    if (!out) fail(Errc::Io, out_path + ": cannot open for writing");
    struct Closer {
        FILE* f;
        ~Closer() { std::fclose(f); }
    } guard{out};

    cudaStream_t st;
    BBMH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct SG {
        cudaStream_t s;
        ~SG() { cudaStreamDestroy(s); }
    } sg{st};
    // device work buffers are kept across calls too (per device; the
    // function-level lock below serialises their use)
    struct DevBufs {
        Buf<uint64_t> d_rp;
        Buf<uint32_t> d_ids;
        Buf<unsigned long long> d_keys, d_keys2, d_ukeys, d_okeys;
        Buf<int> d_vals, d_vals2, d_sums, d_osums, d_nrun, d_nsel, d_err;
        Buf<unsigned char> d_flags, d_tmp;
    };
    // buffers live for the call (the library keeps no device or page-locked
    // memory between VW calls)
    Buf<uint64_t> d_rp;
    Buf<uint32_t> d_ids, d_bins, d_counts;
    Buf<unsigned long long> d_scratch;
    Buf<int> d_sums, d_err;
    d_err.reserve(1);
    HostBuf<uint32_t> bins_h, counts_h;
    HostBuf<int> sums;
    Batch batch;
    uint64_t rows_written = 0;
    int dev = 0, sms = 148;
    BBMH_CUDA(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    for (;;) {
        batch.clear();
        batch.reserve_ids((1u << 24) + (1u << 22));
        trace("vw: fill");
        if (!reader->fill(batch, 1u << 16, 1u << 24)) break;
        trace("vw: filled");
        const uint64_t n = batch.n, nid = batch.nids();
        uint64_t n_ok = n;  // rows to write (those before a failing one)
        counts_h.reserve(n + 1);
        if (nid) {
            d_rp.reserve(n + 1);
            d_ids.reserve(nid);
            d_bins.reserve(nid);
            d_sums.reserve(nid);
            d_counts.reserve(n);
            // rows longer than the shared buffer sort in a scratch of 2x their ids
            uint64_t longest = 0;
            for (uint64_t r = 0; r < n; ++r) longest = std::max(longest, batch.row_ptr[r + 1] - batch.row_ptr[r]);
            if (longest > kVwSmemKeys) d_scratch.reserve(2 * nid + 2);
            BBMH_CUDA(cudaMemcpyAsync(d_rp.p, batch.row_ptr.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
            BBMH_CUDA(cudaMemcpyAsync(d_ids.p, batch.ids, nid * 4, cudaMemcpyHostToDevice, st));
            BBMH_CUDA(cudaMemsetAsync(d_err.p, 0, sizeof(int), st));
            const unsigned grid = (unsigned)std::min<uint64_t>(n, uint64_t(sms) * 8);
            static const bool smem_ok = [] {
                return cudaFuncSetAttribute(vw_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            int(kVwSmemKeys * sizeof(unsigned long long))) == cudaSuccess;
            }();
            if (!smem_ok) fail(Errc::Cuda, "cannot give the VW row kernel its shared sort buffer");
            vw_row_kernel<<<grid, kVwThreads, kVwSmemKeys * sizeof(unsigned long long), st>>>(d_rp.p, n, d_ids.p, coef, d_scratch.p, d_bins.p,
                                                      d_sums.p, d_counts.p, d_err.p);
            BBMH_CUDA(cudaGetLastError());
            count_launches(1);
            int err = 0;
            bins_h.reserve(nid);
            sums.reserve(nid);
            BBMH_CUDA(cudaMemcpyAsync(counts_h.p, d_counts.p, n * 4, cudaMemcpyDeviceToHost, st));
            BBMH_CUDA(cudaMemcpyAsync(bins_h.p, d_bins.p, nid * 4ull, cudaMemcpyDeviceToHost, st));
            BBMH_CUDA(cudaMemcpyAsync(sums.p, d_sums.p, nid * 4ull, cudaMemcpyDeviceToHost, st));
            BBMH_CUDA(cudaMemcpyAsync(&err, d_err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
            BBMH_CUDA(cudaStreamSynchronize(st));
            if (err) {
                // the reference writes every row before the first offending
                // one, then fails (vw.cpp:61-77): keep only those rows
                uint64_t bad_row = 0;
                for (uint64_t i = 0; i < nid; ++i)
                    if (batch.ids[i] >= 0x7fffffffu) {
                        bad_row = uint64_t(std::upper_bound(batch.row_ptr.begin(), batch.row_ptr.end(), i) -
                                           batch.row_ptr.begin()) - 1;
                        break;
                    }
                n_ok = bad_row;
            }
        } else {
            std::memset(counts_h.p, 0, n * 4);
        }
        trace("vw: device done");
        // write_libsvm (dataio.cpp:115-125): "%+d" then " %u:%g" per entry.
        // Rows are formatted in parallel ranges (the text is ~12 bytes per
        // entry: this was the single-threaded bottleneck) and written in order.
        const unsigned T = n_ok < 512 ? 1u : std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        // entry <= 22 chars (" 4294967296:-999999"), row head <= 3 + newline
        std::vector<std::vector<char>> parts(T);
        std::vector<size_t> used(T, 0);
        auto fmt = [&](unsigned w) {
            const uint64_t r0 = n_ok * w / T, r1 = n_ok * (w + 1) / T;
            uint64_t entries = 0;
            for (uint64_t r = r0; r < r1; ++r) entries += counts_h.p[r];
            std::vector<char>& buf = parts[w];
            buf.resize(entries * 24 + (r1 - r0) * 8 + 64);
            char* p = buf.data();
            for (uint64_t r = r0; r < r1; ++r) {
                const int lab = batch.labels[r];
                *p++ = lab < 0 ? '-' : '+';
                p = put_uint(p, uint64_t(lab < 0 ? -lab : lab));
                const uint64_t e0 = batch.row_ptr[r], e1 = e0 + counts_h.p[r];
                for (uint64_t e = e0; e < e1; ++e) {
                    const uint32_t bin = bins_h.p[e];
                    const int v = sums.p[e];
                    *p++ = ' ';
                    p = put_uint(p, uint32_t(bin + 1u));  // "%u" of the u32 index + 1
                    *p++ = ':';
                    if (v > -1000000 && v < 1000000) {  // %g of an integer below 1e6 prints digits
                        if (v < 0) *p++ = '-';
                        p = put_uint(p, uint64_t(v < 0 ? -int64_t(v) : v));
                    } else {
                        p += std::snprintf(p, 32, "%g", double(float(v)));
                    }
                }
                *p++ = '\n';
            }
            used[w] = size_t(p - buf.data());
        };
        if (T == 1) {
            fmt(0);
        } else {
            std::vector<std::thread> ts;
            for (unsigned w = 1; w < T; ++w) ts.emplace_back(fmt, w);
            fmt(0);
            for (auto& t : ts) t.join();
        }
        trace("vw: formatted");
        for (unsigned w = 0; w < T; ++w) write_all(out, parts[w].data(), used[w]);
        trace("vw: written");
        rows_written += n_ok;
        if (n_ok < n) fail(Errc::UnsupportedUniverse, "feature id must be < 2^31-1 for the sign hash");
    }
    return rows_written;
}

}  // namespace bbmh
