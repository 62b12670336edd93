// replay.cu -- epoch replay of a corpus on the GPU: the consumer side of the
// sketch files.
//
// The reference's learner reads its training data once per epoch through a
// RowSource (open_rows, learner.cpp:301-312): a BBMH sketch is expanded at
// run time, record by record (SketchRowSource, learner.cpp:271-297, reading
// through SketchReader, sketch.cpp:143-207: ones[j] = j*2^b + code_j, flagged
// empty records as empty rows), and the original data is parsed again every
// epoch (LibsvmRowSource / BinaryRowSource, learner.cpp:215-269). Paper
// Table 4 is the loading-time ratio of the two.
//
// Here a Replay streams batches of rows as device CSR: for a BBMH file the
// raw record blocks are read with parallel pread into page-locked memory (the
// next block while the caller consumes the current one), copied to the GPU
// and expanded there by one kernel; for LibSVM / BBCV the corpus loader
// (GPU LibSVM parser, ids left on the device) fills the batch. reset()
// starts the next epoch.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <thread>
#include <vector>

#include "engine.hpp"
#include "hostpool.hpp"
#include "io.hpp"
#include "replay.hpp"

namespace bbmh {

namespace {

// one CTA per row: indices[row_ptr[r] + j] = j*2^b + code_j for unflagged rows
// (expand, expansion.cpp:17-27, with the 32-bit truncation of ones[j])
__global__ void replay_expand_kernel(const uint8_t* __restrict__ recs, size_t rec_bytes,
                                     const uint64_t* __restrict__ row_ptr, uint32_t k, uint32_t b,
                                     uint32_t* __restrict__ out) {
    const uint64_t r = blockIdx.x;
    const uint8_t* rec = recs + r * rec_bytes;
    if (rec[1] & 1) return;  // flagged empty set: empty row
    const uint8_t* codes = rec + 2;
    uint32_t* dst = out + row_ptr[r];
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) {
        const uint64_t bit = (uint64_t)j * b;
        const uint8_t* p = codes + (bit >> 3);
        const uint32_t sh = (uint32_t)(bit & 7);
        const uint32_t nbytes = (sh + b + 7) >> 3;
        uint64_t v = 0;
        for (uint32_t i = 0; i < nbytes; ++i) v |= (uint64_t)p[i] << (8 * i);
        v >>= sh;
        const uint32_t code = b >= 32 ? (uint32_t)v : (uint32_t)(v & ((1ull << b) - 1));
        dst[j] = (uint32_t)(((uint64_t)j << b) + code);
    }
}

template <typename T>
struct Pinned {
    T* p = nullptr;
    uint64_t cap = 0;
    void reserve(uint64_t n) {
        if (n <= cap) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        BBMH_CUDA(cudaMallocHost(&p, std::max<uint64_t>(n, 1) * sizeof(T)));
        cap = n;
    }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

template <typename T>
struct Dev {
    T* p = nullptr;
    uint64_t cap = 0;
    int dev = -1;
    void reserve(uint64_t n) {
        if (n <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        BBMH_CUDA(cudaMalloc(&p, std::max<uint64_t>(n, 1) * sizeof(T)));
        cap = n;
    }
    ~Dev() {
        if (p) cudaFree(p);
    }
};

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

struct Replay::Impl {
    int device = 0;
    uint64_t max_rows = 0;
    ReplayInfo info;
    cudaStream_t st = nullptr;
    // BBMH mode
    int fd = -1;
    size_t rec_bytes = 0;
    uint64_t next_rec = 0;     // first record of the block the read-ahead fetches / fetched
    bool short_seen = false;
    Pinned<uint8_t> blk[2];    // record blocks: the current one and the read-ahead
    uint64_t blk_rows[2] = {0, 0};
    bool blk_short[2] = {false, false};
    int cur = 0;
    std::thread ahead;
    std::exception_ptr ahead_err;
    Dev<uint8_t> d_recs;
    // raw-corpus mode
    std::string path;
    unsigned threads = 1;
    std::unique_ptr<CorpusReader> corpus;
    Batch batch;
    // outputs of the last batch
    Pinned<uint64_t> h_rp;
    Dev<uint64_t> d_rp;
    Dev<uint32_t> d_idx;
    std::vector<int8_t> labels;
    ReplayStats stats;
    std::atomic<uint64_t> io_ns{0};  // written by the read-ahead thread

    ~Impl() {
        if (ahead.joinable()) ahead.join();
        if (fd >= 0) ::close(fd);
        if (st) cudaStreamDestroy(st);
    }

    // pread of records [r0, r0 + n) into blk[i] (parallel for large blocks)
    void read_block(int i, uint64_t r0) {
        const uint64_t n = std::min(max_rows, info.count > r0 ? info.count - r0 : 0);
        blk_rows[i] = 0;
        blk_short[i] = false;
        if (n == 0) return;
        const size_t bytes = n * rec_bytes;
        blk[i].reserve(bytes);
        const auto t0 = std::chrono::steady_clock::now();
        const unsigned T = bytes >= (size_t(16) << 20) ? std::min(16u, host_threads()) : 1u;
        std::vector<size_t> got(T, 0);
        std::vector<int> err(T, 0);
        const off_t base = off_t(36 + r0 * rec_bytes);
        host_parallel(T, [&](unsigned w) {
            const size_t lo = bytes * w / T, hi = bytes * (w + 1) / T;
            size_t done = 0;
            while (lo + done < hi) {
                const ssize_t r = ::pread(fd, blk[i].p + lo + done, hi - lo - done, base + off_t(lo + done));
                if (r < 0) {
                    if (errno == EINTR) continue;
                    err[w] = errno;
                    break;
                }
                if (r == 0) break;
                done += size_t(r);
            }
            got[w] = done;
        });
        size_t total = 0;
        for (unsigned w = 0; w < T; ++w) {
            if (err[w]) fail(Errc::Io, path + ": read error");
            total += got[w];
            if (got[w] < bytes * (w + 1) / T - bytes * w / T) break;
        }
        blk_rows[i] = total / rec_bytes;
        blk_short[i] = blk_rows[i] < n;  // the reference fails at the first short record
        io_ns += uint64_t(seconds_since(t0) * 1e9);
    }

    void start_ahead(uint64_t r0) {
        ahead_err = nullptr;
        const int i = cur ^ 1;
        ahead = std::thread([this, i, r0] {
            try {
                read_block(i, r0);
            } catch (...) {
                ahead_err = std::current_exception();
            }
        });
    }

    uint64_t next_bbmh() {
        if (short_seen) fail(Errc::Io, "short read");
        if (ahead.joinable()) ahead.join();
        if (ahead_err) std::rethrow_exception(ahead_err);
        cur ^= 1;
        const uint64_t n = blk_rows[cur];
        const bool was_short = blk_short[cur];
        if (n == 0) {
            if (was_short) fail(Errc::Io, "short read");
            return 0;
        }
        next_rec += n;
        // read the block after this one while the caller works on this one
        if (!was_short && next_rec < info.count) start_ahead(next_rec);
        else blk_rows[cur ^ 1] = 0, blk_short[cur ^ 1] = false;
        const auto t0 = std::chrono::steady_clock::now();
        const uint8_t* recs = blk[cur].p;
        h_rp.reserve(n + 1);
        labels.resize(n);
        h_rp.p[0] = 0;
        for (uint64_t r = 0; r < n; ++r) {
            labels[r] = int8_t(recs[r * rec_bytes]);
            h_rp.p[r + 1] = h_rp.p[r] + ((recs[r * rec_bytes + 1] & 1) ? 0 : info.k);
        }
        const uint64_t nnz = h_rp.p[n];
        d_recs.reserve(n * rec_bytes);
        d_rp.reserve(n + 1);
        d_idx.reserve(nnz + 4);
        BBMH_CUDA(cudaMemcpyAsync(d_recs.p, recs, n * rec_bytes, cudaMemcpyHostToDevice, st));
        BBMH_CUDA(cudaMemcpyAsync(d_rp.p, h_rp.p, (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
        replay_expand_kernel<<<(unsigned)n, 128, 0, st>>>(d_recs.p, rec_bytes, d_rp.p, info.k, info.b,
                                                          d_idx.p);
        BBMH_CUDA(cudaGetLastError());
        count_launches(1);
        BBMH_CUDA(cudaStreamSynchronize(st));
        stats.expand_seconds += seconds_since(t0);
        if (was_short) short_seen = true;  // the next call reports it
        return n;
    }

    uint64_t next_corpus() {
        const auto t0 = std::chrono::steady_clock::now();
        batch.clear();
        batch.want_device_ids = corpus->parser_device() == device;
        if (!batch.want_device_ids) batch.reserve_ids(std::max<uint64_t>(1 << 20, batch.cap_ids));
        if (!corpus->fill(batch, max_rows, 1ull << 24)) return 0;
        const uint64_t n = batch.n, nnz = batch.nids();
        const uint32_t* d_ids = nullptr;
        if (batch.want_device_ids && batch.d_dev == device && batch.d_valid == nnz) {
            d_ids = batch.d_ids;
        } else {
            d_idx.reserve(nnz + 4);
            if (nnz)
                BBMH_CUDA(cudaMemcpyAsync(d_idx.p, batch.ids, nnz * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            d_ids = d_idx.p;
        }
        h_rp.reserve(n + 1);
        std::memcpy(h_rp.p, batch.row_ptr.data(), (n + 1) * sizeof(uint64_t));
        d_rp.reserve(n + 1);
        BBMH_CUDA(cudaMemcpyAsync(d_rp.p, h_rp.p, (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
        BBMH_CUDA(cudaStreamSynchronize(st));
        labels.assign(batch.labels.begin(), batch.labels.end());
        raw_ids = d_ids;
        stats.io_seconds = corpus->io_seconds();
        stats.parse_seconds = corpus->parse_seconds();
        stats.expand_seconds += seconds_since(t0);
        return n;
    }
    const uint32_t* raw_ids = nullptr;

    void open_corpus_reader() {
        BBMH_CUDA(cudaSetDevice(device));
        corpus = open_corpus(path, threads);
    }
};

Replay::Replay(const std::string& path, int device, uint64_t max_rows, unsigned threads)
    : p_(std::make_unique<Impl>()) {
    Impl& m = *p_;
    m.device = device;
    m.path = path;
    m.threads = std::max(1u, threads);
    m.max_rows = std::max<uint64_t>(1, max_rows);
    BBMH_CUDA(cudaSetDevice(device));
    BBMH_CUDA(cudaStreamCreateWithFlags(&m.st, cudaStreamNonBlocking));
    FILE* f = open_or_fail(path, "rb");
    uint8_t h[36] = {};
    const size_t got = std::fread(h, 1, 36, f);
    std::fclose(f);
    if (got >= 4 && std::memcmp(h, "BBMH", 4) == 0) {
        // SketchReader's header checks and messages (sketch.cpp:143-163)
        if (got < 8) fail(Errc::Io, "short read");
        if (h[4] != 1) fail(Errc::MalformedLine, path + ": unknown version");
        if (h[5] > 3) fail(Errc::MalformedLine, path + ": unknown scheme tag");
        if (got < 36) fail(Errc::Io, "short read");
        m.info.sketch = true;
        m.info.scheme = h[5];
        m.info.b = h[6];
        m.info.k = get_u32(h + 8);
        m.info.dim = get_u64(h + 12);
        m.info.seed = get_u64(h + 20);
        m.info.count = get_u64(h + 28);
        // expanded_dim (expansion.cpp:9-15)
        if (m.info.b < 1 || m.info.b > 32) fail(Errc::InvalidArgument, "b must be in 1..32");
        m.info.expanded_dim = (uint64_t(1) << m.info.b) * m.info.k;
        if (m.info.expanded_dim > (uint64_t(1) << 32))
            fail(Errc::DimensionExceeded, "2^b * k exceeds 32-bit row indices");
        m.rec_bytes = 2 + packed_code_bytes(m.info.k, m.info.b);
        m.fd = ::open(path.c_str(), O_RDONLY);
        if (m.fd < 0) fail(Errc::Io, path + ": " + std::strerror(errno));
    } else {
        m.info.sketch = false;
    }
    reset();
}

Replay::~Replay() = default;

const ReplayInfo& Replay::info() const { return p_->info; }
ReplayStats Replay::stats() const {
    ReplayStats s = p_->stats;
    if (p_->info.sketch) s.io_seconds = double(p_->io_ns.load()) * 1e-9;
    return s;
}

void Replay::reset() {
    Impl& m = *p_;
    m.stats.epochs += 1;
    if (m.info.sketch) {
        if (m.ahead.joinable()) m.ahead.join();
        m.next_rec = 0;
        m.short_seen = false;
        m.cur = 1;  // the read-ahead fills blk[0], which next() makes current
        m.start_ahead(0);
    } else {
        m.open_corpus_reader();
    }
}

uint64_t Replay::next(const uint64_t** d_row_ptr, const uint32_t** d_indices, const int8_t** labels,
                      const uint64_t** h_row_ptr) {
    Impl& m = *p_;
    BBMH_CUDA(cudaSetDevice(m.device));
    const uint64_t n = m.info.sketch ? m.next_bbmh() : m.next_corpus();
    m.stats.rows += n;
    if (d_row_ptr) *d_row_ptr = n ? m.d_rp.p : nullptr;
    if (d_indices) *d_indices = n ? (m.info.sketch ? m.d_idx.p : m.raw_ids) : nullptr;
    if (labels) *labels = n ? m.labels.data() : nullptr;
    if (h_row_ptr) *h_row_ptr = n ? m.h_rp.p : nullptr;
    if (n) m.stats.nnz += m.h_rp.p[n];
    return n;
}

}  // namespace bbmh
