// vw.cu -- VW signed random-bin projection on the GPU.
//
// Reference: VwProjector (vw.cpp:11-59) and vw_project_file (vw.cpp:61-77):
//   bin(t)  = eval_2u over `bins` (power of two) with coefficients
//             keyed_u64(seed, 7, 0, {0,1}) (a2 forced odd);
//   sign(t) = +1 if the 4U polynomial mod 2^31-1 (coefficients drawn from
//             keyed_u64(seed, 8, attempt, i) >> 33 below p) is odd, else -1;
//   a row becomes the ascending list of bins whose signed counts are non-zero,
//   written as LibSVM text "%+d" + " %u:%g" (bin + 1, count) per entry.
// GPU path per batch of rows: one thread per id computes the 64-bit key
// (row << 32 | bin) and its sign; a CUB radix sort orders the keys (only the
// bits in use), CUB reduce-by-key sums the signs per (row, bin), and the
// non-zero entries are compacted on the device. Signed counts are exact
// integers, so the summation order does not matter. The host formats the
// rows in order.
#include <cuda_runtime.h>

#include <bit>
#include <cmath>
#include <cstring>
#include <cub/cub.cuh>
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

__global__ void vw_keys_kernel(const uint64_t* __restrict__ row_ptr, uint64_t n,
                               const uint32_t* __restrict__ ids, VwCoef c,
                               unsigned long long* __restrict__ keys, int* __restrict__ vals,
                               int* err) {
    // one thread per row id range would serialise long rows; map threads to ids
    // and find the row by binary search over row_ptr
    const uint64_t total = row_ptr[n];
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = n;  // row r with row_ptr[r] <= i < row_ptr[r+1]
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (row_ptr[mid] <= i) lo = mid;
            else hi = mid;
        }
        uint32_t t = ids[i];
        if (t >= kP31) {
            atomicOr(err, 1);
            t = 0;
        }
        const uint32_t h2 = c.a1 + c.a2 * t;
        const uint32_t bin = c.shift ? h2 >> c.shift : h2;
        const uint32_t t2 = t << 1;
        uint32_t s = fold31(c.s3, t2, c.s2x2);
        uint32_t h = min(s, s - kP31);
        s = fold31(h, t2, c.s1x2);
        h = min(s, s - kP31);
        s = fold31(h, t2, c.s0x2);
        h = min(min(s, s - kP31), s - 2 * kP31);
        keys[i] = (unsigned long long)lo << 32 | bin;
        vals[i] = (h & 1) ? 1 : -1;
    }
}

__global__ void vw_flag_kernel(const int* __restrict__ sums, const int* __restrict__ nrun,
                               unsigned char* __restrict__ flags) {
    const int n = *nrun;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        flags[i] = sums[i] != 0;
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
    DevBufs D;
    auto& d_rp = D.d_rp;
    auto& d_ids = D.d_ids;
    auto& d_keys = D.d_keys;
    auto& d_keys2 = D.d_keys2;
    auto& d_ukeys = D.d_ukeys;
    auto& d_okeys = D.d_okeys;
    auto& d_vals = D.d_vals;
    auto& d_vals2 = D.d_vals2;
    auto& d_sums = D.d_sums;
    auto& d_osums = D.d_osums;
    auto& d_nrun = D.d_nrun;
    auto& d_nsel = D.d_nsel;
    auto& d_err = D.d_err;
    auto& d_flags = D.d_flags;
    auto& d_tmp = D.d_tmp;
    d_nrun.reserve(1);
    d_nsel.reserve(1);
    d_err.reserve(1);
    {
        // one allocation round for the largest batch (growing buffers batch by
        // batch re-allocates, and cudaFree stalls)
        const size_t cap = (1u << 24) + (1u << 22);
        d_ids.reserve(cap);
        d_keys.reserve(cap);
        d_keys2.reserve(cap);
        d_vals.reserve(cap);
        d_vals2.reserve(cap);
        d_ukeys.reserve(cap);
        d_sums.reserve(cap);
        d_okeys.reserve(cap);
        d_osums.reserve(cap);
        d_flags.reserve(cap);
        d_rp.reserve((1u << 16) + 1);
    }
    HostBuf<unsigned long long> keys;
    HostBuf<int> sums;
    Batch batch;
    uint64_t rows_written = 0;
    int dev = 0, sms = 148;
    BBMH_CUDA(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int row_bits = 17, bin_bits = 32;  // rows per batch < 2^17
    for (;;) {
        batch.clear();
        batch.reserve_ids((1u << 24) + (1u << 22));
        trace("vw: fill");
        if (!reader->fill(batch, 1u << 16, 1u << 24)) break;
        trace("vw: filled");
        const uint64_t n = batch.n, nid = batch.nids();
        uint64_t n_ok = n;  // rows to write (those before a failing one)
        int nsel = 0;
        if (nid) {
            d_rp.reserve(n + 1);
            d_ids.reserve(nid);
            d_keys.reserve(nid);
            d_keys2.reserve(nid);
            d_vals.reserve(nid);
            d_vals2.reserve(nid);
            d_ukeys.reserve(nid);
            d_sums.reserve(nid);
            d_okeys.reserve(nid);
            d_osums.reserve(nid);
            d_flags.reserve(nid);
            BBMH_CUDA(cudaMemcpyAsync(d_rp.p, batch.row_ptr.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
            BBMH_CUDA(cudaMemcpyAsync(d_ids.p, batch.ids, nid * 4, cudaMemcpyHostToDevice, st));
            BBMH_CUDA(cudaMemsetAsync(d_err.p, 0, sizeof(int), st));
            const unsigned grid = (unsigned)std::min<uint64_t>((nid + 255) / 256, uint64_t(sms) * 32);
            vw_keys_kernel<<<grid, 256, 0, st>>>(d_rp.p, n, d_ids.p, coef, d_keys.p, d_vals.p, d_err.p);
            BBMH_CUDA(cudaGetLastError());
            count_launches(1);
            const int end_bit = bin_bits + row_bits;
            size_t need = 0, n2 = 0, n3 = 0;
            BBMH_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need, d_keys.p, d_keys2.p, d_vals.p,
                                                      d_vals2.p, (int)nid, 0, end_bit, st));
            BBMH_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, n2, d_keys2.p, d_ukeys.p, d_vals2.p,
                                                     d_sums.p, d_nrun.p, cuda::std::plus<int>(),
                                                     (int)nid, st));
            BBMH_CUDA(cub::DeviceSelect::Flagged(nullptr, n3, d_ukeys.p, d_flags.p, d_okeys.p,
                                                 d_nsel.p, (int)nid, st));
            d_tmp.reserve(std::max({need, n2, n3, size_t(1)}));
            size_t tb = d_tmp.cap;
            BBMH_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp.p, tb, d_keys.p, d_keys2.p, d_vals.p,
                                                      d_vals2.p, (int)nid, 0, end_bit, st));
            tb = d_tmp.cap;
            BBMH_CUDA(cub::DeviceReduce::ReduceByKey(d_tmp.p, tb, d_keys2.p, d_ukeys.p, d_vals2.p,
                                                     d_sums.p, d_nrun.p, cuda::std::plus<int>(),
                                                     (int)nid, st));
            vw_flag_kernel<<<grid, 256, 0, st>>>(d_sums.p, d_nrun.p, d_flags.p);
            count_launches(1);
            // runs beyond *d_nrun carry stale flags: select over nid only after zeroing them
            int nrun = 0;
            BBMH_CUDA(cudaMemcpyAsync(&nrun, d_nrun.p, sizeof(int), cudaMemcpyDeviceToHost, st));
            BBMH_CUDA(cudaStreamSynchronize(st));
            tb = d_tmp.cap;
            BBMH_CUDA(cub::DeviceSelect::Flagged(d_tmp.p, tb, d_ukeys.p, d_flags.p, d_okeys.p,
                                                 d_nsel.p, nrun, st));
            tb = d_tmp.cap;
            BBMH_CUDA(cub::DeviceSelect::Flagged(d_tmp.p, tb, d_sums.p, d_flags.p, d_osums.p,
                                                 d_nsel.p, nrun, st));
            int err = 0;
            BBMH_CUDA(cudaMemcpyAsync(&nsel, d_nsel.p, sizeof(int), cudaMemcpyDeviceToHost, st));
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
            keys.reserve(size_t(nsel) + 1);
            sums.reserve(size_t(nsel) + 1);
            if (nsel) {
                BBMH_CUDA(cudaMemcpyAsync(keys.p, d_okeys.p, nsel * 8ull, cudaMemcpyDeviceToHost, st));
                BBMH_CUDA(cudaMemcpyAsync(sums.p, d_osums.p, nsel * 4ull, cudaMemcpyDeviceToHost, st));
                BBMH_CUDA(cudaStreamSynchronize(st));
            }
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
            // first entry of row r0: keys are sorted by (row << 32 | bin)
            uint64_t e = std::lower_bound(keys.p, keys.p + nsel, (unsigned long long)r0 << 32) - keys.p;
            uint64_t e_end = std::lower_bound(keys.p, keys.p + nsel, (unsigned long long)r1 << 32) - keys.p;
            std::vector<char>& buf = parts[w];
            buf.resize((e_end - e) * 24 + (r1 - r0) * 8 + 64);
            char* p = buf.data();
            for (uint64_t r = r0; r < r1; ++r) {
                const int lab = batch.labels[r];
                *p++ = lab < 0 ? '-' : '+';
                p = put_uint(p, uint64_t(lab < 0 ? -lab : lab));
                for (; e < e_end && (keys[e] >> 32) == r; ++e) {
                    const uint32_t bin = uint32_t(keys[e]);
                    const int v = sums[e];
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
