// io.cpp -- corpus readers feeding the GPU pipeline.
//
// The reference reads one record at a time on one thread (fgetc per
// character for LibSVM, dataio.cpp:166-175; fread per u32 for BBCV,
// dataio.cpp:217-221) -- 36 MB/s and 132 MB/s measured (SURVEY.md finding 7).
// Here:
//   * BBCV rows are fread straight into page-locked batch memory, validated
//     (label +-1, strictly ascending ids) in place;
//   * LibSVM text is read in large blocks, split at line boundaries and the
//     lines of a block are parsed by `parse_threads` threads into per-thread
//     CSR fragments that are concatenated in order. The first error in file
//     order wins, with the reference's line numbering and messages. Common
//     tokens take a fast path ("idx:1"); anything unusual falls back to the
//     same strtod/strtoll calls the reference makes, so accepted inputs,
//     values and error texts are identical.
#include "io.hpp"
#include "parse.hpp"
#include "hostpool.hpp"
#include "options.hpp"

#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>

namespace bbmh {

FILE* open_or_fail(const std::string& path, const char* mode) {
    FILE* f = std::fopen(path.c_str(), mode);
    if (!f) fail(Errc::Io, path + ": " + std::strerror(errno));
    return f;
}

void write_all(FILE* f, const void* data, size_t n) {
    if (n && std::fwrite(data, 1, n, f) != n) fail(Errc::Io, "short write");
}

Batch::~Batch() {
    if (ids) cudaFreeHost(ids);
    if (d_ids) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(d_dev);
        cudaFree(d_ids);
        cudaSetDevice(cur);
    }
}

void Batch::reserve_ids(uint64_t cap) {
    if (cap <= cap_ids) return;
    cap = std::max<uint64_t>(cap, cap_ids + cap_ids / 2);
    uint32_t* p = nullptr;
    if (cudaMallocHost(&p, std::max<uint64_t>(cap, 1) * sizeof(uint32_t)) != cudaSuccess)
        fail(Errc::Cuda, "cudaMallocHost failed for a loader batch");
    if (ids) {
        // (with device-resident ids the host array may be shorter than nids())
        std::memcpy(p, ids, std::min(nids(), cap_ids) * sizeof(uint32_t));
        cudaFreeHost(ids);
    }
    ids = p;
    cap_ids = cap;
}

uint32_t* Batch::reserve_device_ids(int dev, uint64_t cap) {
    constexpr uint64_t kSlack = 16;  // the sketch kernel's bulk copies read whole 16-byte granules
    if (d_ids && d_dev == dev && cap + kSlack <= d_cap) return d_ids;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    const uint64_t ncap = std::max<uint64_t>(cap + kSlack, d_dev == dev ? d_cap + d_cap / 2 : 0);
    uint32_t* p = nullptr;
    if (cudaMalloc(&p, ncap * sizeof(uint32_t)) != cudaSuccess) {
        cudaGetLastError();
        cudaSetDevice(cur);
        fail(Errc::Cuda, "cudaMalloc failed for a loader batch");
    }
    if (d_ids && d_dev == dev && d_valid) cudaMemcpy(p, d_ids, d_valid * sizeof(uint32_t), cudaMemcpyDeviceToDevice);
    if (d_ids) {
        cudaSetDevice(d_dev);
        cudaFree(d_ids);
        cudaSetDevice(dev);
    }
    if (d_dev != dev) d_valid = 0;
    d_ids = p;
    d_cap = ncap;
    d_dev = dev;
    cudaSetDevice(cur);
    return d_ids;
}

namespace {

void read_exact(FILE* f, void* p, size_t n) {
    if (n && std::fread(p, 1, n, f) != n) fail(Errc::Io, "short read");
}

// ---- BBCV ------------------------------------------------------------------
// The file is mapped read-only. fill() walks record headers sequentially
// (label check, bounds) -- cheap, one touch per record -- then copies and
// validates the id runs of the batch in parallel straight into the batch's
// page-locked buffer. The first failing record (lowest index) wins, with the
// reference's messages (dataio.cpp:211-230).
class BinaryReader : public CorpusReader {
    std::atomic<uint32_t> sink_{0};

public:
    BinaryReader(const std::string& path, unsigned threads)
        : path_(path), threads_(std::max(1u, std::min(threads, 64u))) {
        FILE* f = open_or_fail(path, "rb");
        uint8_t head[21];
        read_exact(f, head, 4);
        if (std::memcmp(head, "BBCV", 4) != 0) {
            std::fclose(f);
            fail(Errc::MalformedLine, path_ + ": not a BBCV corpus");
        }
        try {
            read_exact(f, head + 4, 1);
            if (head[4] != 1) fail(Errc::MalformedLine, path_ + ": unknown BBCV version");
            read_exact(f, head + 5, 16);
        } catch (...) {
            std::fclose(f);
            throw;
        }
        std::fseek(f, 0, SEEK_END);
        size_ = uint64_t(std::ftell(f));
        std::fclose(f);
        dim_ = get_u64(head + 5);
        count_ = get_u64(head + 13);
        pos_ = 21;
        fd_ = ::open(path.c_str(), O_RDONLY);
        if (fd_ < 0) fail(Errc::Io, path_ + ": " + std::strerror(errno));
        if (size_ > 0) {
            void* m = ::mmap(nullptr, size_, PROT_READ, MAP_PRIVATE, fd_, 0);
            if (m == MAP_FAILED) fail(Errc::Io, path_ + ": mmap failed");
            map_ = static_cast<const uint8_t*>(m);
            ::madvise(m, size_, MADV_SEQUENTIAL);
        }
    }
    ~BinaryReader() override {
        if (map_) ::munmap(const_cast<uint8_t*>(map_), size_);
        if (fd_ >= 0) ::close(fd_);
    }

    // Maps the pages of [off, off + n) on all pool threads. A batch's header
    // walk otherwise takes one page fault per few records on one thread
    // (~1.7 ms per 67 MB batch, as long as copying it).
    void prefault(uint64_t off, uint64_t n) {
        if (!map_ || n < (uint64_t(4) << 20)) return;
        const unsigned T = std::min(16u, host_threads());
        host_parallel(T, [&](unsigned w) {
            const uint64_t lo = off + n * w / T, hi = off + n * (w + 1) / T;
            uint32_t acc = 0;
            for (uint64_t p = lo; p < hi; p += 4096) acc += map_[p];
            sink_.fetch_add(acc, std::memory_order_relaxed);  // keep the reads
        });
    }

    bool fill(Batch& b, uint64_t max_docs, uint64_t max_ids) override {
        // 1. sequential header walk
        struct Rec {
            uint64_t src;  // byte offset of the first id
            uint64_t dst;  // id offset in the batch
            uint32_t n;
        };
        std::vector<Rec> recs;
        Errc pend_code = Errc::Io;
        std::string pend_msg;
        bool pending = false;
        uint64_t nid = b.nids();
        const uint64_t first = read_;
        prefault(pos_, std::min<uint64_t>(size_ - pos_, (max_ids + max_ids / 4) * 4 + 5 * max_docs));
        while (read_ < count_ && b.n + recs.size() < max_docs && (nid < max_ids || recs.empty())) {
            if (pos_ + 1 > size_) {
                pending = true, pend_code = Errc::Io, pend_msg = "short read";
                break;
            }
            const int8_t label = int8_t(map_[pos_]);
            if (label != 1 && label != -1) {
                pending = true, pend_code = Errc::NonBinaryLabel;
                pend_msg = "record " + std::to_string(read_) + ": bad label";
                break;
            }
            if (pos_ + 5 > size_) {
                pending = true, pend_code = Errc::Io, pend_msg = "short read";
                break;
            }
            const uint32_t n = get_u32(map_ + pos_ + 1);
            if (pos_ + 5 + uint64_t(n) * 4 > size_) {
                pending = true, pend_code = Errc::Io, pend_msg = "short read";
                break;
            }
            recs.push_back({pos_ + 5, nid, n});
            b.labels.push_back(label);
            nid += n;
            pos_ += 5 + uint64_t(n) * 4;
            ++read_;
        }
        if (recs.empty() && !pending) return false;
        trace("bbcv: headers walked");
        if (nid > b.cap_ids) b.reserve_ids(std::max<uint64_t>(nid, max_ids + max_ids / 4));
        // 2. parallel copy + strictly-ascending check
        const size_t nr = recs.size();
        const unsigned W = nr < 256 ? 1u : threads_;
        std::vector<uint64_t> bad(W, UINT64_MAX);
        auto work = [&](unsigned w) {
            const size_t lo = nr * w / W, hi = nr * (w + 1) / W;
            for (size_t r = lo; r < hi; ++r) {
                const Rec& rc = recs[r];
                uint32_t* dst = b.ids + rc.dst;
                std::memcpy(dst, map_ + rc.src, size_t(rc.n) * 4);
                uint32_t nonasc = 0;
                for (uint32_t i = 1; i < rc.n; ++i) nonasc |= dst[i] <= dst[i - 1];
                if (nonasc) {
                    bad[w] = r;
                    return;
                }
            }
        };
        host_parallel(W, work);
        trace("bbcv: ids copied");
        for (unsigned w = 0; w < W; ++w)
            if (bad[w] != UINT64_MAX)
                fail(Errc::NonAscendingIndex, "record " + std::to_string(first + bad[w]));
        if (pending) fail(pend_code, pend_msg);
        for (const Rec& rc : recs) b.row_ptr.push_back(rc.dst + rc.n);
        b.n += nr;
        return true;
    }

private:
    std::string path_;
    unsigned threads_;
    int fd_ = -1;
    const uint8_t* map_ = nullptr;
    uint64_t size_ = 0, pos_ = 0;
    uint64_t dim_ = 0, count_ = 0, read_ = 0;
};

// ---- LibSVM ----------------------------------------------------------------
struct LineErr {
    Errc code = Errc::Io;
    uint64_t line = 0;
    std::string detail;
    bool set = false;
};

inline bool is_value_end(char c) {
    return c == ' ' || c == '\t' || c == '\0' || c == '\r' || c == '#';
}

// parse_libsvm (dataio.cpp:60-106) with 0/1 labels accepted. Binary mode
// (vals == nullptr, the sketch loader) rejects values != 1; value mode (the
// prediction loader, learner.cpp:254) keeps float(val) per id.
// `line` is NUL-terminated. Appends ids; returns false with `err` set.
bool parse_line(const char* line, uint64_t line_no, std::vector<uint32_t>& ids, int8_t& label,
                LineErr& err, std::vector<float>* vals = nullptr) {
    auto bad = [&](Errc c, const std::string& what) {
        err.code = c;
        err.line = line_no;
        err.detail = what;
        err.set = true;
        return false;
    };
    const char* p = line;
    char* end = nullptr;
    double lv;
    if ((p[0] == '+' || p[0] == '-') && p[1] == '1' && (p[2] == ' ' || p[2] == '\t' || p[2] == '\0')) {
        lv = p[0] == '+' ? 1.0 : -1.0;
        end = const_cast<char*>(p + 2);
    } else {
        lv = std::strtod(p, &end);
        if (end == p) return bad(Errc::MalformedLine, "missing label");
    }
    if (lv == 1 || lv == -1) label = int8_t(lv);
    else if (lv == 0) label = -1;
    else return bad(Errc::MalformedLine, "label must be +-1 (or 0/1)");
    p = end;
    int64_t prev = -1;
    for (;;) {
        while (*p == ' ' || *p == '\t') ++p;
        const char c = *p;
        if (c == '\0' || c == '\n' || c == '\r' || c == '#') break;
        long long idx;
        if (c >= '0' && c <= '9') {  // fast path: plain decimal digits
            uint64_t v = 0;
            const char* q = p;
            int nd = 0;
            while (*q >= '0' && *q <= '9' && nd < 19) {
                v = v * 10 + uint64_t(*q - '0');
                ++q;
                ++nd;
            }
            if (*q >= '0' && *q <= '9') {  // too long for the fast path
                idx = std::strtoll(p, &end, 10);
            } else {
                idx = (long long)v;
                end = const_cast<char*>(q);
            }
        } else {
            idx = std::strtoll(p, &end, 10);
        }
        if (end == p || *end != ':') return bad(Errc::MalformedLine, "expected idx:val");
        if (idx < 1 || idx > (long long)UINT32_MAX)
            return bad(Errc::MalformedLine, "index out of range (1-based u32)");
        if (idx - 1 <= prev) return bad(Errc::NonAscendingIndex, "indices must be strictly ascending");
        prev = idx - 1;
        p = end + 1;
        double val;
        if (p[0] == '1' && is_value_end(p[1])) {
            val = 1.0;
            end = const_cast<char*>(p + 1);
        } else {
            val = std::strtod(p, &end);
            if (end == p) return bad(Errc::MalformedLine, "missing value");
        }
        p = end;
        if (vals)
            vals->push_back(float(val));
        else if (val != 1.0)
            return bad(Errc::NonBinaryValue, "value " + std::to_string(val) + " in binary mode");
        ids.push_back(uint32_t(idx - 1));
    }
    return true;
}

// Text buffer: page-locked when the GPU parser is used (so blocks DMA straight
// to the device), plain heap memory otherwise. resize() keeps the contents.
class TextBuf {
public:
    ~TextBuf() { release(); }
    void set_pinned(bool on) { pinned_ = on; }
    char* data() { return p_; }
    size_t size() const { return n_; }
    char& operator[](size_t i) { return p_[i]; }
    void resize(size_t n) {
        if (n <= n_) return;
        char* q = nullptr;
        if (pinned_) {
            if (cudaMallocHost(&q, n) != cudaSuccess) {
                cudaGetLastError();
                fail(Errc::Cuda, "cudaMallocHost failed for the text buffer");
            }
        } else {
            q = static_cast<char*>(std::malloc(n));
            if (!q) fail(Errc::Io, "out of memory");
        }
        if (p_) std::memcpy(q, p_, n_);
        release();
        p_ = q;
        n_ = n;
    }

private:
    void release() {
        if (!p_) return;
        if (pinned_) cudaFreeHost(p_);
        else std::free(p_);
        p_ = nullptr;
        n_ = 0;
    }
    char* p_ = nullptr;
    size_t n_ = 0;
    bool pinned_ = false;
};

// Reader resources are pooled process-wide: a 128 MB page-locked text buffer
// and the device parser's buffers cost tens of milliseconds to allocate, more
// than parsing a small corpus takes.
struct TextRes {
    int device = -1;  // -1: CPU parsing only (plain heap buffer)
    TextBuf buf, alt;  // alt: the device parser's second window (GPU mode only)
    std::unique_ptr<GpuLibsvmParser> gpu;
};
std::mutex g_text_mu;
std::vector<std::unique_ptr<TextRes>> g_text_pool;

std::unique_ptr<TextRes> lease_text_res(int device) {
    {
        std::lock_guard lk(g_text_mu);
        for (size_t i = 0; i < g_text_pool.size(); ++i)
            if (g_text_pool[i]->device == device) {
                auto r = std::move(g_text_pool[i]);
                g_text_pool.erase(g_text_pool.begin() + long(i));
                return r;
            }
    }
    auto r = std::make_unique<TextRes>();
    if (device >= 0) {
        try {
            r->gpu = std::make_unique<GpuLibsvmParser>(device);
            r->device = device;
        } catch (...) {
            r->gpu.reset();
        }
        cudaGetLastError();
    }
    r->buf.set_pinned(r->gpu != nullptr);
    r->alt.set_pinned(r->gpu != nullptr);
    return r;
}

void return_text_res(std::unique_ptr<TextRes> r) {
    if (!r) return;
    std::lock_guard lk(g_text_mu);
    g_text_pool.push_back(std::move(r));
}

class LibsvmReader : public CorpusReader {
public:
    LibsvmReader(const std::string& path, unsigned threads, bool binary, uint64_t begin = 0,
                 uint64_t end = UINT64_MAX)
        : path_(path), threads_(std::max(1u, std::min(threads, 64u))), binary_(binary), end_off_(end) {
        f_ = open_or_fail(path, "rb");
        buf_off_ = file_off_ = begin;
        // the device parser takes binary-mode corpora (the sketch loader)
        int dev = -1;
        if (binary_ && gpu_parse_enabled()) {
            if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
            cudaGetLastError();
        }
        res_ = lease_text_res(dev);
        buf_ = &res_->buf;
        gpu_ = res_->gpu.get();
        gpu_block_ = gpu_parse_block_bytes(kGpuBlock);
        // GPU mode: two windows, each with room for the block being parsed,
        // the next one, the read-ahead block and a few more (4 blocks: 7% slower; 8: no faster)
        // (a block size set through the test knob sizes the windows alone, so
        // small corpora exercise the window switch)
        const size_t win = gpu_block_ == kGpuBlock ? std::max(2 * kBlock, 6 * gpu_block_) : 6 * gpu_block_;
        win_ = gpu_ ? win : 2 * kBlock;
        buf_->resize(win_ + 1);
        if (gpu_) {
            alt_ = &res_->alt;
            alt_->resize(win_ + 1);
        }
    }
    ~LibsvmReader() override {
        if (f_) std::fclose(f_);
        if (gpu_) {
            try {
                gpu_->cancel_prefetch();
            } catch (...) {
            }
        }
        return_text_res(std::move(res_));
    }

    int parser_device() const override { return gpu_ ? gpu_->device() : -1; }
    uint64_t lines_consumed() const override { return line_no_; }
    double io_seconds() const override { return double(io_ns_.load()) * 1e-9; }
    double parse_seconds() const override { return double(parse_ns_.load()) * 1e-9; }

    bool fill(Batch& b, uint64_t max_docs, uint64_t max_ids) override {
        if (!gpu_) b.want_device_ids = false;
        const bool any = fill_rows(b, max_docs, max_ids);
        if (b.want_device_ids) upload_host_ids(b);  // every id on the device
        return any;
    }

private:
    // The CPU parser's rows [d_valid, nids()) of a device-resident batch, up.
    void upload_host_ids(Batch& b) {
        if (b.d_valid >= b.nids()) return;
        const int dev = gpu_->device();
        b.reserve_device_ids(dev, b.nids());
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(dev);
        const cudaError_t e = cudaMemcpy(b.d_ids + b.d_valid, b.ids + b.d_valid,
                                         (b.nids() - b.d_valid) * sizeof(uint32_t), cudaMemcpyHostToDevice);
        cudaSetDevice(cur);
        if (e != cudaSuccess) {
            cudaGetLastError();
            fail(Errc::Cuda, std::string("upload of a loader batch failed: ") + cudaGetErrorString(e));
        }
        b.d_valid = b.nids();
    }

    bool fill_rows(Batch& b, uint64_t max_docs, uint64_t max_ids) {
        bool any = false;
        while (b.n < max_docs && (b.nids() < max_ids || b.n == 0)) {
            if (gpu_ && pos_ >= cpu_until_) {
                const uint64_t n0 = b.n;
                const int g = gpu_block(b, max_docs, max_ids);
                if (g == 1) {
                    any |= b.n > n0;
                    continue;
                }
                if (g == 0 || g == 2) {  // end of input / batch full (this block may have added rows)
                    any |= b.n > n0;
                    break;
                }
                // g < 0: the block is parsed by the CPU path below
            }
            // gather complete lines (as NUL-terminated spans) for this round
            std::vector<std::pair<size_t, size_t>> lines;  // [begin, end) in buf_
            const uint64_t byte_budget = std::max<uint64_t>(1, (max_ids - std::min(max_ids, b.nids())) * 4);
            uint64_t bytes = 0;
            while (lines.size() < max_docs - b.n && bytes < byte_budget) {
                if (!next_line(lines)) break;
                bytes += lines.back().second - lines.back().first + 1;
            }
            if (lines.empty()) break;
            any |= parse_lines(lines, b);
            compact_if_needed();
        }
        return any;
    }

    static constexpr size_t kBlock = size_t(64) << 20;
    static constexpr size_t kGpuBlock = size_t(32) << 20;

    // Where a GPU block starting at `start` ends: 1 with [start, cut) set, 0 at
    // the end of input, 2 if the batch is full, 3 if more input must be read
    // first (only when !may_refill; refilling needs start == pos_). The block
    // is sized from the bytes per line / per id seen so far to what the batch
    // still takes, plus a little: the parser keeps the prefix that fits.
    int plan_block(uint64_t rows_left, uint64_t ids_left, bool batch_empty, size_t start, size_t& cut,
                   bool& at_eof, bool may_refill) {
        size_t target = gpu_block_;
        if (lines_seen_) {
            const double per_line = double(bytes_seen_) / double(lines_seen_);
            const double per_id = ids_seen_ ? double(bytes_seen_) / double(ids_seen_) : 4.0;
            double fit = per_line * double(rows_left);
            if (!batch_empty) fit = std::min(fit, per_id * double(ids_left));
            if (!batch_empty && fit < 0.5 * per_line) return 2;
            fit = 1.05 * fit + 2 * per_line;
            if (fit < double(target)) target = std::max<size_t>(4096, size_t(fit));
        }
        for (;;) {
            const bool final = sealed_ || eof_;  // the window's data ends at a line end / the file's end
            if (len_ - start < target && !final) {
                if (!may_refill) return 3;
                trace("reader: refill");
                refill();
                trace("reader: refilled");
                continue;
            }
            if (start >= len_) {
                if (!sealed_) return 0;
                if (!may_refill) return 3;
                unseal();  // the window is drained: go on in the next one
                continue;
            }
            const size_t end = std::min(len_, start + target);
            cut = 0;
            if (end == len_ && final) {
                cut = len_;
            } else {
                const void* nl = memrchr(buf_->data() + start, '\n', end - start);
                if (nl) cut = size_t(static_cast<const char*>(nl) - buf_->data()) + 1;
            }
            if (!cut) {  // one line longer than the block: widen it
                if (final && end == len_) return 0;
                target *= 2;
                continue;
            }
            at_eof = cut == len_ && eof_ && !sealed_;
            return 1;
        }
    }

    // The current window is used up; its successor (holding the line the
    // window's data stopped in the middle of, and what was read after it)
    // becomes current.
    void unseal() {
        if (gpu_) gpu_->cancel_prefetch();  // the old window is about to be overwritten
        std::swap(buf_, alt_);
        buf_off_ = alt_off_;
        len_ = alt_len_;
        pos_ = 0;
        cpu_until_ = 0;
        alt_len_ = 0;
        sealed_ = false;
    }

    uint64_t file_pos(size_t buf_pos) const { return buf_off_ + buf_pos; }

    // One block of complete lines through the GPU parser. Returns 1 if the
    // block was consumed, 0 at the end of input, 2 if the batch is full (the
    // rest starts the next one), -1 if it must go through the CPU parser (set
    // up via cpu_until_).
    //
    // While the GPU parses [pos_, cut), a host thread reads the next block
    // into the free tail of the window. When the tail is full the window is
    // sealed at its last line end: the partial line after it starts the other
    // window, reading goes on there, and the GPU drains this one first. Blocks
    // never straddle windows and only a partial line is ever copied. The copy
    // of the block after this one to the device starts as soon as this
    // block's kernels are queued.
    int gpu_block(Batch& b, uint64_t max_docs, uint64_t max_ids) {
        const uint64_t rows_left = max_docs - b.n;
        const uint64_t ids_left = max_ids - std::min(max_ids, b.nids());
        const bool empty = b.n == 0;
        size_t cut = 0;
        bool at_eof = false;
        const int plan = plan_block(rows_left, ids_left, empty, pos_, cut, at_eof, true);
        if (plan != 1) return plan;
        const uint64_t key = file_pos(pos_);
        // the next block as planned now (the batch state moves on, so it may
        // be planned differently when it comes: that only wastes the copy)
        size_t ncut = 0;
        bool neof = false;
        const bool next = cut < len_ && plan_block(rows_left, ids_left, empty, cut, ncut, neof, false) == 1;
        const uint64_t nkey = file_pos(cut);

        enum { kNone, kTail, kSeal, kAltTail } mode = kNone;
        size_t seal_at = 0;
        if (!eof_) {
            if (!sealed_) {
                if (win_ - len_ >= gpu_block_) {
                    mode = kTail;
                } else {
                    // seal after the last line end (the blocks planned so far end before it)
                    const void* nl = memrchr(buf_->data() + cut, '\n', len_ - cut);
                    seal_at = nl ? size_t(static_cast<const char*>(nl) - buf_->data()) + 1 : cut;
                    if (win_ >= len_ - seal_at + gpu_block_) mode = kSeal;
                }
            } else if (win_ - alt_len_ >= gpu_block_) {
                mode = kAltTail;
            }
        }
        std::thread ahead;
        size_t ahead_got = 0;
        std::exception_ptr ahead_err;
        if (mode != kNone) {
            ahead = std::thread([&] {
                try {
                    if (mode == kTail) {
                        ahead_got = read_at(buf_->data() + len_, gpu_block_);
                    } else if (mode == kSeal) {
                        std::memcpy(alt_->data(), buf_->data() + seal_at, len_ - seal_at);
                        ahead_got = read_at(alt_->data() + (len_ - seal_at), gpu_block_);
                    } else {
                        ahead_got = read_at(alt_->data() + alt_len_, gpu_block_);
                    }
                    trace("ahead: read");
                } catch (...) {
                    ahead_err = std::current_exception();
                }
            });
        }
        auto reserve = [&](uint64_t need) {
            if (need > b.cap_ids) b.reserve_ids(need + (1u << 20));
            return b.ids;
        };
        // device-resident ids: the rows the CPU parser took go up first, so
        // the device holds a prefix [0, d_valid) and this block extends it
        const bool dev = b.want_device_ids;
        DeviceIdsOut dout;
        if (dev) {
            upload_host_ids(b);
            dout.reserve = [&](uint64_t need) { return b.reserve_device_ids(gpu_->device(), need); };
            dout.base = b.nids();
        }
        GpuParseResult r;
        const auto parse0 = std::chrono::steady_clock::now();
        try {
            r = gpu_->parse(buf_->data() + pos_, cut - pos_, at_eof, b.nids(), rows_left,
                            empty ? UINT64_MAX : ids_left, reserve, b.row_ptr, b.labels, key,
                            next ? buf_->data() + cut : nullptr, next ? ncut - cut : 0, nkey,
                            dev ? &dout : nullptr);
        } catch (...) {
            if (ahead.joinable()) ahead.join();
            throw;
        }
        parse_ns_ += uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                  std::chrono::steady_clock::now() - parse0).count());
        const bool whole = r.ok && r.bytes == cut - pos_;
        if (ahead.joinable()) {
            ahead.join();
            if (ahead_err) std::rethrow_exception(ahead_err);
            if (ahead_got < gpu_block_) eof_ = true;
            if (mode == kTail) {
                len_ += ahead_got;
            } else if (mode == kSeal) {
                alt_off_ = buf_off_ + seal_at;
                alt_len_ = len_ - seal_at + ahead_got;
                len_ = seal_at;
                sealed_ = true;
            } else {
                alt_len_ += ahead_got;
            }
        }
        if (!r.ok) {
            if (r.over_budget && b.n > 0) {
                trace("reader: batch full");
                return 2;  // this block starts the next batch
            }
            trace("reader: gpu block declined");
            cpu_until_ = cut;
            return -1;
        }
        if (trace_on()) {
            char msg[96];
            std::snprintf(msg, sizeof msg, "reader: gpu block parsed (%zu bytes, %llu rows)",
                          size_t(r.bytes), (unsigned long long)r.rows);
            trace(msg);
        }
        b.n += r.rows;
        if (dev) b.d_valid = b.nids();
        line_no_ += r.lines;
        lines_seen_ += r.lines;
        bytes_seen_ += r.bytes;
        ids_seen_ += r.ids;
        pos_ += r.bytes;
        gpu_blocks_ += 1;
        if (sealed_ && pos_ == len_) unseal();  // so the next window's first block can be prefetched
        // the next block's copy, if the one started above was planned otherwise
        // (a full batch: the next one starts empty)
        size_t cut2 = 0;
        bool eof2 = false;
        const bool full = !whole;
        int plan2 = plan_block(full ? max_docs : max_docs - b.n, full ? max_ids : max_ids - std::min(max_ids, b.nids()),
                               full || b.n == 0, pos_, cut2, eof2, false);
        if (plan2 == 2)  // this batch takes no more: the block opens the next one
            plan2 = plan_block(max_docs, max_ids, true, pos_, cut2, eof2, false);
        if (plan2 == 1 && !gpu_->prefetched(file_pos(pos_), cut2 - pos_))
            gpu_->prefetch(buf_->data() + pos_, cut2 - pos_, file_pos(pos_));
        if (full) return 2;
        return pos_ < len_ || sealed_ || !eof_ || r.rows ? 1 : 0;
    }

    // Finds the next line starting at pos_; reads more input as needed.
    bool next_line(std::vector<std::pair<size_t, size_t>>& lines) {
        for (;;) {
            void* nl = pos_ < len_ ? std::memchr(buf_->data() + pos_, '\n', len_ - pos_) : nullptr;
            if (nl) {
                const size_t e = size_t(static_cast<char*>(nl) - buf_->data());
                (*buf_)[e] = '\0';
                lines.emplace_back(pos_, e);
                pos_ = e + 1;
                return true;
            }
            if (eof_ && !sealed_) {
                if (pos_ < len_) {  // last line without a newline
                    (*buf_)[len_] = '\0';
                    lines.emplace_back(pos_, len_);
                    pos_ = len_;
                    return true;
                }
                return false;
            }
            if (!lines.empty()) return false;  // parse what we have before moving data
            refill();
        }
    }

    void refill() {
        if (gpu_) gpu_->cancel_prefetch();  // its host bytes are about to move
        if (sealed_) {
            // (the window ends at a line end, so it is drained by now; keep any
            // rest anyway, in front of the next window's data)
            const size_t rest = len_ - pos_;
            if (rest) {
                if (alt_len_ + rest > win_) grow_windows(alt_len_ + rest);
                std::memmove(alt_->data() + rest, alt_->data(), alt_len_);
                std::memcpy(alt_->data(), buf_->data() + pos_, rest);
                alt_off_ -= rest;
                alt_len_ += rest;
                pos_ = len_;
            }
            unseal();
            return;
        }
        if (pos_ > 0) {
            std::memmove(buf_->data(), buf_->data() + pos_, len_ - pos_);
            len_ -= pos_;
            buf_off_ += pos_;
            cpu_until_ = cpu_until_ > pos_ ? cpu_until_ - pos_ : 0;
            pos_ = 0;
        }
        const size_t room = gpu_ ? gpu_block_ : kBlock / 2;
        if (len_ + room > win_) grow_windows(len_ + 2 * room);
        size_t want = win_ - len_;
        if (gpu_) want = std::min(want, std::max(2 * gpu_block_, size_t(1) << 20));  // rest: read-ahead
        const size_t got = read_at(buf_->data() + len_, want);
        if (got < want) eof_ = true;
        len_ += got;
    }

    void grow_windows(size_t need) {
        win_ = std::max(win_ * 2, need);
        buf_->resize(win_ + 1);
        if (alt_) alt_->resize(win_ + 1);
    }

    void compact_if_needed() {}

    // pread of [file_off_, file_off_ + n) into p, split over up to 16 threads
    // (one thread copies ~10 GB/s out of the page cache); returns bytes read.
    size_t read_at(char* p, size_t n) {
        const int fd = fileno(f_);
        if (end_off_ != UINT64_MAX) n = size_t(std::min<uint64_t>(n, end_off_ > file_off_ ? end_off_ - file_off_ : 0));
        if (n == 0) return 0;
        const auto io0 = std::chrono::steady_clock::now();
        struct IoTimer {
            std::atomic<uint64_t>& acc;
            std::chrono::steady_clock::time_point t0;
            ~IoTimer() {
                acc += uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                    std::chrono::steady_clock::now() - t0).count());
            }
        } io_timer{io_ns_, io0};
        // 8 -> 16 threads: 15.7 -> 17.5 GB/s of text
        const unsigned kReadThreads = unsigned(std::max<int64_t>(1, opt(Opt::ReadThreads)));
        const unsigned T = n >= (size_t(16) << 20) ? std::min(kReadThreads, threads_) : 1u;
        std::vector<size_t> got(T, 0);
        std::vector<int> err(T, 0);
        auto work = [&](unsigned w) {
            const size_t lo = n * w / T, hi = n * (w + 1) / T;
            size_t done = 0;
            while (lo + done < hi) {
                const ssize_t r = ::pread(fd, p + lo + done, hi - lo - done, off_t(file_off_ + lo + done));
                if (r < 0) {
                    if (errno == EINTR) continue;
                    err[w] = errno;
                    break;
                }
                if (r == 0) break;
                done += size_t(r);
            }
            got[w] = done;
        };
        host_parallel(T, work);  // pooled threads: spawning 15 per block cost ~0.3 ms
        size_t total = 0;
        for (unsigned w = 0; w < T; ++w) {
            if (err[w]) fail(Errc::Io, path_ + ": read error");
            total += got[w];
            if (got[w] < n * (w + 1) / T - n * w / T) break;  // end of file inside slice w
        }
        file_off_ += total;
        return total;
    }

    struct Frag {
        std::vector<uint32_t> ids;
        std::vector<float> vals;
        std::vector<uint64_t> lens;
        std::vector<int8_t> labels;
        size_t err_line = SIZE_MAX;  // index into the round's lines
        LineErr err;
    };

    // Parses `lines` (in order) into b; throws the first error in file order.
    bool parse_lines(const std::vector<std::pair<size_t, size_t>>& lines, Batch& b) {
        const auto t0 = std::chrono::steady_clock::now();
        struct Timer {
            std::atomic<uint64_t>& acc;
            std::chrono::steady_clock::time_point t0;
            ~Timer() {
                acc += uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                    std::chrono::steady_clock::now() - t0).count());
            }
        } timer{parse_ns_, t0};
        const size_t nl = lines.size();
        const unsigned W = nl < 64 ? 1u : threads_;
        std::vector<Frag> frags(W);
        const uint64_t line0 = line_no_;
        auto work = [&](unsigned w) {
            Frag& fr = frags[w];
            const size_t lo = nl * w / W, hi = nl * (w + 1) / W;
            for (size_t i = lo; i < hi; ++i) {
                const auto [s, e] = lines[i];
                if (s == e) continue;  // blank line: skipped, but numbered
                int8_t label = 1;
                const size_t before = fr.ids.size();
                if (!parse_line(buf_->data() + s, line0 + i + 1, fr.ids, label, fr.err,
                                binary_ ? nullptr : &fr.vals)) {
                    fr.err_line = i;
                    fr.ids.resize(before);
                    if (!binary_) fr.vals.resize(before);
                    return;
                }
                fr.lens.push_back(fr.ids.size() - before);
                fr.labels.push_back(label);
            }
        };
        host_parallel(W, work);
        line_no_ += nl;
        bool any = false;
        for (Frag& fr : frags) {
            const uint64_t base = b.nids();
            if (base + fr.ids.size() > b.cap_ids) b.reserve_ids(base + fr.ids.size() + (1u << 20));
            std::memcpy(b.ids + base, fr.ids.data(), fr.ids.size() * sizeof(uint32_t));
            if (!binary_) b.vals.insert(b.vals.end(), fr.vals.begin(), fr.vals.end());
            uint64_t acc = base;
            for (size_t r = 0; r < fr.lens.size(); ++r) {
                acc += fr.lens[r];
                b.row_ptr.push_back(acc);
                b.labels.push_back(fr.labels[r]);
                ++b.n;
                any = true;
            }
            if (fr.err.set) throw LineError(fr.err.code, fr.err.line, fr.err.detail);
        }
        return any;
    }

    std::string path_;
    unsigned threads_;
    bool binary_;
    FILE* f_ = nullptr;
    std::unique_ptr<TextRes> res_;  // pooled: pinned text buffer + device parser
    TextBuf* buf_ = nullptr;
    TextBuf* alt_ = nullptr;  // GPU mode: the other window (see gpu_block)
    size_t win_ = 0;          // window size in use (both buffers hold at least win_ + 1)
    bool sealed_ = false;     // buf_ ends at len_; the data after it is in alt_ (see gpu_block)
    size_t alt_len_ = 0;      // bytes in alt_ while sealed_
    uint64_t buf_off_ = 0, alt_off_ = 0;  // file offsets of buf_[0], alt_[0]
    uint64_t file_off_ = 0;  // bytes of the file consumed by read_at
    size_t pos_ = 0, len_ = 0;
    bool eof_ = false;
    uint64_t line_no_ = 0;
    GpuLibsvmParser* gpu_ = nullptr;
    size_t cpu_until_ = 0;  // buffer offset up to which lines go through the CPU parser
    uint64_t lines_seen_ = 0, bytes_seen_ = 0, ids_seen_ = 0, gpu_blocks_ = 0;
    size_t gpu_block_ = kGpuBlock;
    uint64_t end_off_ = UINT64_MAX;  // range end (exclusive file offset)
    std::atomic<uint64_t> io_ns_{0}, parse_ns_{0};
};

}  // namespace

SketchFileReader::SketchFileReader(const std::string& path) {
    f_ = open_or_fail(path, "rb");
    try {
        uint8_t h[36];
        read_exact(f_, h, 4);
        if (std::memcmp(h, "BBMH", 4) != 0)
            fail(Errc::MalformedLine, path + ": not a BBMH sketch file");
        read_exact(f_, h + 4, 4);
        if (h[4] != 1) fail(Errc::MalformedLine, path + ": unknown version");
        if (h[5] > 3) fail(Errc::MalformedLine, path + ": unknown scheme tag");
        read_exact(f_, h + 8, 28);
        scheme_ = h[5];
        b_ = h[6];
        k_ = get_u32(h + 8);
        dim_ = get_u64(h + 12);
        seed_ = get_u64(h + 20);
        count_ = get_u64(h + 28);
    } catch (...) {
        std::fclose(f_);
        f_ = nullptr;
        throw;
    }
}

SketchFileReader::~SketchFileReader() {
    if (f_) std::fclose(f_);
}

void SketchFileReader::seek(uint64_t i) {
    const uint64_t rec = 2 + packed_code_bytes(k_, b_);
    if (std::fseek(f_, long(36 + i * rec), SEEK_SET) != 0) fail(Errc::Io, "seek failed");
    done_ = i;
    short_ = false;
}

uint64_t SketchFileReader::read(uint64_t max_rows, std::vector<uint8_t>& codes,
                                std::vector<uint8_t>& flags, std::vector<int8_t>& labels) {
    if (short_) fail(Errc::Io, "short read");
    const uint64_t want = std::min(max_rows, count_ - done_);
    if (want == 0) return 0;
    const size_t cb = packed_code_bytes(k_, b_);
    const size_t rec = 2 + cb;
    buf_.resize(want * rec);
    const size_t got = std::fread(buf_.data(), 1, want * rec, f_);
    const uint64_t n = got / rec;
    if (n < want) short_ = true;
    if (n == 0) fail(Errc::Io, "short read");
    codes.resize(n * cb);
    flags.resize(n);
    labels.resize(n);
    for (uint64_t i = 0; i < n; ++i) {
        labels[i] = int8_t(buf_[i * rec]);
        flags[i] = buf_[i * rec + 1];
        std::memcpy(codes.data() + i * cb, buf_.data() + i * rec + 2, cb);
    }
    done_ += n;
    return n;
}

bool is_libsvm_text(const std::string& path) {
    FILE* f = open_or_fail(path, "rb");
    char magic[4] = {0, 0, 0, 0};
    const size_t got = std::fread(magic, 1, 4, f);
    std::fclose(f);
    return !(got == 4 && std::memcmp(magic, "BBCV", 4) == 0);
}

uint64_t file_size(const std::string& path) {
    struct stat st {};
    if (::stat(path.c_str(), &st) != 0) fail(Errc::Io, path + ": " + std::strerror(errno));
    return uint64_t(st.st_size);
}

uint64_t line_start_at_or_after(const std::string& path, uint64_t off) {
    if (off == 0) return 0;
    const uint64_t size = file_size(path);
    if (off >= size) return size;
    const int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) fail(Errc::Io, path + ": " + std::strerror(errno));
    std::vector<char> buf(size_t(1) << 20);
    uint64_t pos = off - 1;  // a line starts at off if the byte before it is '\n'
    uint64_t found = size;
    while (pos < size) {
        const ssize_t r = ::pread(fd, buf.data(), buf.size(), off_t(pos));
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) break;
        const void* nl = std::memchr(buf.data(), '\n', size_t(r));
        if (nl) {
            found = pos + uint64_t(static_cast<const char*>(nl) - buf.data()) + 1;
            break;
        }
        pos += uint64_t(r);
    }
    ::close(fd);
    return found;
}

std::unique_ptr<CorpusReader> open_libsvm_range(const std::string& path, unsigned parse_threads,
                                                uint64_t begin, uint64_t end) {
    return std::make_unique<LibsvmReader>(path, parse_threads, true, begin, end);
}

std::unique_ptr<CorpusReader> open_corpus(const std::string& path, unsigned parse_threads,
                                          bool libsvm_values) {
    FILE* f = open_or_fail(path, "rb");
    char magic[4] = {0, 0, 0, 0};
    const size_t got = std::fread(magic, 1, 4, f);
    std::fclose(f);
    if (got == 4 && std::memcmp(magic, "BBCV", 4) == 0)
        return std::make_unique<BinaryReader>(path, parse_threads);
    return std::make_unique<LibsvmReader>(path, parse_threads, !libsvm_values);
}

}  // namespace bbmh
