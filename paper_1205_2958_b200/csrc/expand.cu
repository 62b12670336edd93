// expand.cu -- bbmh_expand_file: BBMH sketch -> k*2^b one-hot rows.
//
// Reference: expand_stream (expansion.cpp:47-90) decodes each record with
// get_code (sketch.cpp:55-62), forms ones[j] = j*2^b + code_j
// (expansion.cpp:17-27) and writes a BBCV row (dataio.cpp:139-145) or a
// LibSVM line "%+d" + " %u:1"*k + "\n" with 1-based ids (dataio.cpp:115-125);
// flagged empty records become empty rows (expansion.cpp:61-66,78-83).
//
// Here the rows of a batch of records are produced on the GPU:
//   BBCV  : one CTA per record writes label, count and the k ids at a
//           host-computed byte offset (row sizes depend only on the flags);
//   LibSVM: a length pass (per-record byte count, digits of every id), an
//           exclusive scan over records, and a write pass in which each
//           thread formats a contiguous run of ids at its block-scanned
//           offset (device-side integer -> decimal).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "engine.hpp"
#include "io.hpp"
#include "pipeline.hpp"

namespace bbmh {

namespace {

constexpr int kExpandThreads = 256;

__device__ __forceinline__ uint32_t get_code_dev(const uint8_t* codes, uint32_t j, uint32_t b) {
    const uint64_t bit = (uint64_t)j * b;
    const uint8_t* p = codes + (bit >> 3);
    const uint32_t sh = (uint32_t)(bit & 7);
    const uint32_t nbytes = (sh + b + 7) >> 3;  // <= 5
    uint64_t v = 0;
    for (uint32_t i = 0; i < nbytes; ++i) v |= (uint64_t)p[i] << (8 * i);
    v >>= sh;
    return b >= 32 ? (uint32_t)v : (uint32_t)(v & ((1ull << b) - 1));
}

// ones[j] = uint32(2^b * j + code_j) (expansion.cpp:25-26, 32-bit truncation)
__device__ __forceinline__ uint32_t one_index(const uint8_t* codes, uint32_t j, uint32_t b) {
    const uint64_t v = ((uint64_t)j << b) + get_code_dev(codes, j, b);
    return (uint32_t)v;
}

__device__ __forceinline__ uint32_t ndigits(uint32_t v) {
    uint32_t d = 1;
    while (v >= 10) {
        v /= 10;
        ++d;
    }
    return d;
}

__device__ __forceinline__ uint32_t write_u32(uint8_t* out, uint32_t v, uint32_t nd) {
    for (uint32_t i = nd; i > 0; --i) {
        out[i - 1] = (uint8_t)('0' + v % 10);
        v /= 10;
    }
    return nd;
}

__device__ __forceinline__ uint32_t label_len(int8_t l) {
    const int a = l < 0 ? -(int)l : (int)l;
    return 1 + ndigits((uint32_t)a);
}

__global__ void expand_bbcv_kernel(const uint8_t* __restrict__ recs, size_t rec_bytes,
                                   const uint64_t* __restrict__ offs, uint32_t k, uint32_t b,
                                   uint8_t* __restrict__ out) {
    const uint64_t r = blockIdx.x;
    const uint8_t* rec = recs + r * rec_bytes;
    const bool empty = rec[1] & 1;
    uint8_t* dst = out + offs[r];
    if (threadIdx.x == 0) {
        dst[0] = rec[0];
        const uint32_t cnt = empty ? 0 : k;
        for (int i = 0; i < 4; ++i) dst[1 + i] = (uint8_t)(cnt >> (8 * i));
    }
    if (empty) return;
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) {
        const uint32_t v = one_index(rec + 2, j, b);
        uint8_t* p = dst + 5 + 4ull * j;
        p[0] = (uint8_t)v;
        p[1] = (uint8_t)(v >> 8);
        p[2] = (uint8_t)(v >> 16);
        p[3] = (uint8_t)(v >> 24);
    }
}

// per-record byte count of the LibSVM line
__global__ void expand_text_len_kernel(const uint8_t* __restrict__ recs, size_t rec_bytes,
                                       uint32_t k, uint32_t b, uint64_t* __restrict__ lens) {
    __shared__ uint64_t part[kExpandThreads];
    const uint64_t r = blockIdx.x;
    const uint8_t* rec = recs + r * rec_bytes;
    const bool empty = rec[1] & 1;
    uint64_t acc = 0;
    if (!empty)
        for (uint32_t j = threadIdx.x; j < k; j += blockDim.x)
            acc += 3 + ndigits(one_index(rec + 2, j, b) + 1u);  // " %u:1", 1-based, u32 wrap
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) part[threadIdx.x] += part[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) lens[r] = part[0] + label_len((int8_t)rec[0]) + 1;
}

__global__ void expand_text_write_kernel(const uint8_t* __restrict__ recs, size_t rec_bytes,
                                         const uint64_t* __restrict__ offs, uint32_t k,
                                         uint32_t b, uint8_t* __restrict__ out) {
    __shared__ uint64_t scan[kExpandThreads];
    const uint64_t r = blockIdx.x;
    const uint8_t* rec = recs + r * rec_bytes;
    const bool empty = rec[1] & 1;
    uint8_t* dst = out + offs[r];
    const int8_t label = (int8_t)rec[0];
    const uint32_t ll = label_len(label);
    // contiguous run of ids per thread
    const uint32_t per = empty ? 0 : (k + blockDim.x - 1) / blockDim.x;
    const uint32_t j0 = min(k, threadIdx.x * per), j1 = min(k, j0 + per);
    uint64_t mine = 0;
    for (uint32_t j = j0; j < j1; ++j) mine += 3 + ndigits(one_index(rec + 2, j, b) + 1u);
    scan[threadIdx.x] = mine;
    __syncthreads();
    for (int s = 1; s < blockDim.x; s <<= 1) {  // inclusive Hillis-Steele scan
        const uint64_t v = threadIdx.x >= s ? scan[threadIdx.x - s] : 0;
        __syncthreads();
        scan[threadIdx.x] += v;
        __syncthreads();
    }
    uint64_t pos = ll + scan[threadIdx.x] - mine;
    for (uint32_t j = j0; j < j1; ++j) {
        const uint32_t v = one_index(rec + 2, j, b) + 1u;
        const uint32_t nd = ndigits(v);
        dst[pos] = ' ';
        write_u32(dst + pos + 1, v, nd);
        dst[pos + 1 + nd] = ':';
        dst[pos + 2 + nd] = '1';
        pos += 3 + nd;
    }
    if (threadIdx.x == blockDim.x - 1) {
        dst[0] = label < 0 ? '-' : '+';
        const int a = label < 0 ? -(int)label : (int)label;
        write_u32(dst + 1, (uint32_t)a, ll - 1);
        dst[pos] = '\n';
    }
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;
    void reserve(size_t n) {
        if (n <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        cap = std::max(n, cap + cap / 2);
        BBMH_CUDA(cudaMalloc(&p, cap * sizeof(T)));
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

template <typename T>
struct HostBuf {
    T* p = nullptr;
    size_t cap = 0;
    void reserve(size_t n) {
        if (n <= cap) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = std::max(n, cap + cap / 2);
        BBMH_CUDA(cudaMallocHost(&p, cap * sizeof(T)));
    }
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
};

void read_exact(FILE* f, void* p, size_t n) {
    if (n && std::fread(p, 1, n, f) != n) fail(Errc::Io, "short read");
}

}  // namespace

uint64_t expand_file(const std::string& sketch_path, const std::string& out_path, bool binary) {
    // SketchReader ctor (sketch.cpp:143-163)
    FILE* in = open_or_fail(sketch_path, "rb");
    struct Closer {
        FILE* f;
        ~Closer() {
            if (f) std::fclose(f);
        }
    } in_guard{in};
    uint8_t h[36];
    read_exact(in, h, 4);
    if (std::memcmp(h, "BBMH", 4) != 0)
        fail(Errc::MalformedLine, sketch_path + ": not a BBMH sketch file");
    read_exact(in, h + 4, 4);
    if (h[4] != 1) fail(Errc::MalformedLine, sketch_path + ": unknown version");
    if (h[5] > 3) fail(Errc::MalformedLine, sketch_path + ": unknown scheme tag");
    read_exact(in, h + 8, 28);
    const uint32_t b = h[6];
    const uint32_t k = get_u32(h + 8);
    const uint64_t count = get_u64(h + 28);
    // expanded_dim (expansion.cpp:9-15)
    if (b < 1 || b > 32) fail(Errc::InvalidArgument, "b must be in 1..32");
    const uint64_t edim = (uint64_t(1) << b) * k;
    if (edim > (uint64_t(1) << 32))
        fail(Errc::DimensionExceeded, "2^b * k exceeds 32-bit row indices");

    FILE* out = nullptr;
    if (binary) {
        out = open_or_fail(out_path, "wb");
    } else {
        out = std::fopen(out_path.c_str(), "wb");
        if (!out) fail(Errc::Io, out_path + ": cannot open for writing");
    }
    struct OutCloser {
        FILE* f;
        bool binary;
        uint64_t n = 0;
        ~OutCloser() {  // CorpusWriter::close patches the count (dataio.cpp:147-153)
            if (!f) return;
            if (binary) {
                uint8_t c[8];
                put_u64(c, n);
                if (std::fseek(f, 13, SEEK_SET) == 0) std::fwrite(c, 1, 8, f);
            }
            std::fclose(f);
        }
    } og{out, binary};
    if (binary) {
        uint8_t ch[21];
        std::memcpy(ch, "BBCV", 4);
        ch[4] = 1;
        put_u64(ch + 5, edim);
        put_u64(ch + 13, 0);
        write_all(out, ch, sizeof ch);
    }

    const size_t cb = packed_code_bytes(k, b);
    const size_t rec_bytes = 2 + cb;
    const uint64_t batch = std::max<uint64_t>(1, std::min<uint64_t>(65536, (64ull << 20) / rec_bytes));
    cudaStream_t st;
    BBMH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    HostBuf<uint8_t> h_recs, h_out;
    HostBuf<uint64_t> h_offs;
    DevBuf<uint8_t> d_recs, d_out;
    DevBuf<uint64_t> d_offs;
    std::vector<uint64_t> lens;

    for (uint64_t done = 0; done < count;) {
        const uint64_t n = std::min(batch, count - done);
        h_recs.reserve(n * rec_bytes);
        // the reference reads record by record and fails at the first short one
        const size_t got = std::fread(h_recs.p, 1, n * rec_bytes, in);
        const uint64_t whole = got / rec_bytes;
        const uint64_t nn = whole;
        h_offs.reserve(nn + 1);
        d_recs.reserve(std::max<uint64_t>(nn * rec_bytes, 1));
        d_offs.reserve(nn + 1);
        if (nn) {
            BBMH_CUDA(cudaMemcpyAsync(d_recs.p, h_recs.p, nn * rec_bytes, cudaMemcpyHostToDevice, st));
            if (binary) {
                h_offs.p[0] = 0;
                for (uint64_t i = 0; i < nn; ++i)
                    h_offs.p[i + 1] = h_offs.p[i] + 5 + ((h_recs.p[i * rec_bytes + 1] & 1) ? 0 : 4ull * k);
            } else {
                DevBuf<uint64_t>& d_lens = d_offs;
                expand_text_len_kernel<<<(unsigned)nn, kExpandThreads, 0, st>>>(d_recs.p, rec_bytes, k, b,
                                                                                d_lens.p);
                BBMH_CUDA(cudaGetLastError());
                count_launches(1);
                BBMH_CUDA(cudaMemcpyAsync(h_offs.p + 1, d_lens.p, nn * 8, cudaMemcpyDeviceToHost, st));
                BBMH_CUDA(cudaStreamSynchronize(st));
                h_offs.p[0] = 0;
                for (uint64_t i = 0; i < nn; ++i) h_offs.p[i + 1] += h_offs.p[i];
            }
            const uint64_t total = h_offs.p[nn];
            BBMH_CUDA(cudaMemcpyAsync(d_offs.p, h_offs.p, (nn + 1) * 8, cudaMemcpyHostToDevice, st));
            d_out.reserve(total);
            h_out.reserve(total);
            if (binary)
                expand_bbcv_kernel<<<(unsigned)nn, kExpandThreads, 0, st>>>(d_recs.p, rec_bytes, d_offs.p,
                                                                            k, b, d_out.p);
            else
                expand_text_write_kernel<<<(unsigned)nn, kExpandThreads, 0, st>>>(d_recs.p, rec_bytes,
                                                                                  d_offs.p, k, b, d_out.p);
            BBMH_CUDA(cudaGetLastError());
            count_launches(1);
            BBMH_CUDA(cudaMemcpyAsync(h_out.p, d_out.p, total, cudaMemcpyDeviceToHost, st));
            BBMH_CUDA(cudaStreamSynchronize(st));
            write_all(out, h_out.p, total);
            og.n += nn;
        }
        done += nn;
        if (nn < n) fail(Errc::Io, "short read");
    }
    return og.n;
}

}  // namespace bbmh
