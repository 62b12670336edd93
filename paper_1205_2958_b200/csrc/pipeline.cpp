// pipeline.cpp -- bbmh_sketch_file: loader -> pinned CSR batches -> GPU
// lanes (H2D / sketch kernel / D2H) -> order-restoring writer.
//
// Same three roles as the reference's sketch_stream (pipeline.cpp:123-213):
// one reader, a pool of compute workers (here: one host thread per GPU, each
// keeping three chunks in flight), and the calling thread as the in-order
// writer. Output bytes are identical for any (chunk_size, workers, devices).
// First error wins; files are left exactly as the reference's SketchWriter
// destructor leaves them (header with the count of records written).
#include "pipeline.hpp"

#include <chrono>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <atomic>
#include <deque>
#include <exception>
#include <map>
#include <utility>
#include <mutex>
#include <thread>

#include "engine.hpp"
#include "io.hpp"
#include "options.hpp"

namespace bbmh {

namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) {
    return std::chrono::duration<double>(Clock::now() - t0).count();
}

constexpr uint64_t kBatchIds = 1ull << 24;  // ids per loader batch (64 MiB pinned)

thread_local PipelineProfile t_profile;

template <typename T>
class BlockingQueue {
public:
    void push(T v) {
        std::lock_guard lk(m_);
        q_.push_back(std::move(v));
        cv_.notify_one();
    }
    bool pop(T& out) {
        std::unique_lock lk(m_);
        cv_.wait(lk, [&] { return !q_.empty() || closed_ || aborted_; });
        if (aborted_ || q_.empty()) return false;
        out = std::move(q_.front());
        q_.pop_front();
        return true;
    }
    void close() {
        std::lock_guard lk(m_);
        closed_ = true;
        cv_.notify_all();
    }
    void abort() {
        std::lock_guard lk(m_);
        aborted_ = true;
        cv_.notify_all();
    }

private:
    std::mutex m_;
    std::condition_variable cv_;
    std::deque<T> q_;
    bool closed_ = false, aborted_ = false;
};

struct OutBatch {
    uint64_t n = 0;
    std::vector<uint8_t> recs;     // n * (2 + cb): label, flags, codes
    std::vector<uint64_t> minima;  // n * k (optional)
    std::vector<double> scores;    // n (scoring pipeline only)
};

// order-restoring buffer (pipeline.cpp:77-119)
class Reorder {
public:
    void put(uint64_t seq, OutBatch&& b) {
        std::lock_guard lk(m_);
        done_[seq] = std::move(b);
        cv_.notify_all();
    }
    bool take(uint64_t seq, OutBatch& out) {
        std::unique_lock lk(m_);
        cv_.wait(lk, [&] { return done_.count(seq) || (total_known_ && seq >= total_) || aborted_; });
        if (aborted_) return false;
        auto it = done_.find(seq);
        if (it == done_.end()) return false;
        out = std::move(it->second);
        done_.erase(it);
        return true;
    }
    void set_total(uint64_t t) {
        std::lock_guard lk(m_);
        total_ = t;
        total_known_ = true;
        cv_.notify_all();
    }
    void abort() {
        std::lock_guard lk(m_);
        aborted_ = true;
        cv_.notify_all();
    }

private:
    std::mutex m_;
    std::condition_variable cv_;
    std::map<uint64_t, OutBatch> done_;
    uint64_t total_ = 0;
    bool total_known_ = false, aborted_ = false;
};

// Page-locked batch buffers are expensive to allocate (cudaMallocHost of
// ~80 MB each), so they are pooled process-wide and leased per call.
std::mutex g_batch_mu;
std::vector<std::unique_ptr<Batch>> g_batch_pool;

struct BatchLease {
    std::vector<Batch*> batches;
    std::vector<std::unique_ptr<Batch>> owned;
    explicit BatchLease(size_t n) {
        std::lock_guard lk(g_batch_mu);
        while (owned.size() < n) {
            if (!g_batch_pool.empty()) {
                owned.push_back(std::move(g_batch_pool.back()));
                g_batch_pool.pop_back();
            } else {
                owned.push_back(std::make_unique<Batch>());
            }
            batches.push_back(owned.back().get());
        }
    }
    ~BatchLease() {
        std::lock_guard lk(g_batch_mu);
        for (auto& b : owned) {
            b->clear();
            g_batch_pool.push_back(std::move(b));
        }
    }
};

// SketchWriter (sketch.cpp:102-141): header now, count patched on close/destruction
class SketchWriter {
public:
    SketchWriter(const std::string& path, const Family& f, uint8_t b, bool emit_minima) {
        f_ = open_or_fail(path, "wb");
        uint8_t h[36];
        std::memcpy(h, "BBMH", 4);
        h[4] = 1;
        h[5] = uint8_t(f.scheme);
        h[6] = b;
        h[7] = 0;
        put_u32(h + 8, f.k);
        put_u64(h + 12, f.dim);
        put_u64(h + 20, f.seed);
        put_u64(h + 28, 0);
        write_all(f_, h, sizeof h);
        if (emit_minima) fmin_ = open_or_fail(path + ".min64", "wb");
    }
    ~SketchWriter() {
        try {
            close();
        } catch (...) {
        }
    }
    void append(const OutBatch& ob) {
        write_all(f_, ob.recs.data(), ob.recs.size());
        if (fmin_) write_all(fmin_, ob.minima.data(), ob.minima.size() * sizeof(uint64_t));
        count_ += ob.n;
    }
    void close() {
        if (!f_) return;
        FILE* f = f_;
        f_ = nullptr;
        uint8_t c[8];
        put_u64(c, count_);
        const bool ok = std::fseek(f, 28, SEEK_SET) == 0 && std::fwrite(c, 1, 8, f) == 8;
        std::fclose(f);
        if (fmin_) std::fclose(fmin_);
        fmin_ = nullptr;
        if (!ok) fail(Errc::Io, "seek failed");
    }

private:
    FILE* f_ = nullptr;
    FILE* fmin_ = nullptr;
    uint64_t count_ = 0;
};


// Shared engine of the file pipelines: reader thread -> pinned batches ->
// one lane per GPU -> `append(OutBatch)` on the calling thread, in order.
template <typename Append>
PipelineStats run_stream(const Family& f, CorpusReader& reader, uint8_t b, bool emit_minima,
                         const ScoreModel* score, Append&& append) {
    trace("stream: start");
    PipelineStats stats;
    const size_t cb = packed_code_bytes(f.k, b);
    const std::vector<int> devs = pipeline_devices();
    const uint64_t max_docs = chunk_docs_setting();
    const bool b_ok = b >= 1 && b <= 32;

    // One GPU that also parses the text: its batches keep their ids on the
    // device (no D2H after parsing, no H2D before sketching).
    const bool device_ids = devs.size() == 1 && reader.parser_device() == devs[0] && opt(Opt::DeviceIds);
    const size_t nbatches = 3 * devs.size() + 3;
    BatchLease storage(nbatches);  // pinned batches reused across calls
    trace("stream: batches leased");
    BlockingQueue<Batch*> free_q, in_q;
    for (Batch* bt : storage.batches) free_q.push(bt);
    Reorder done;
    std::mutex err_mu;
    std::exception_ptr error;
    auto record_error = [&](std::exception_ptr e) {
        {
            std::lock_guard lk(err_mu);
            if (!error) error = e;
        }
        free_q.abort();
        in_q.abort();
        done.abort();
    };

    std::thread rd([&] {
        try {
            double read_s = 0;
            uint64_t seq = 0, first = 0;
            for (;;) {
                Batch* bt = nullptr;
                if (!free_q.pop(bt)) return;
                const auto t0 = Clock::now();
                bt->clear();
                bt->want_device_ids = device_ids;
                // (device-resident ids need host room only for rows the CPU
                // parser takes, reserved on demand: 84 MB of page-locked memory
                // per batch cost ~35 ms to allocate on a process's first call)
                if (!device_ids) bt->reserve_ids(kBatchIds + kBatchIds / 4);
                const bool got = reader.fill(*bt, max_docs, kBatchIds);
                read_s += since(t0);
                trace("reader: batch filled");
                if (!got) break;
                if (!b_ok) fail(Errc::InvalidArgument, "b must be in 1..32");  // sketch.cpp:73
                bt->seq = seq++;
                bt->first_record = first;
                first += bt->n;
                in_q.push(bt);
            }
            stats.read_seconds = read_s;
            stats.records = first;
            in_q.close();
            done.set_total(seq);
        } catch (...) {
            record_error(std::current_exception());
        }
    });

    std::vector<double> kernel_ms(devs.size(), 0.0);
    std::vector<std::thread> lanes;
    for (size_t di = 0; di < devs.size(); ++di) {
        lanes.emplace_back([&, di] {
            try {
                BBMH_CUDA(cudaSetDevice(devs[di]));
                Lane lane(f, devs[di], b_ok ? b : 8, emit_minima, score);
                std::map<uint64_t, Batch*> inflight;
                auto on_done = [&](const ChunkResult& r) {
                    Batch* bt = inflight.at(r.tag);
                    inflight.erase(r.tag);
                    OutBatch ob;
                    ob.n = r.n;
                    ob.recs.resize(r.n * (2 + cb));
                    uint8_t* p = ob.recs.data();
                    for (uint64_t i = 0; i < r.n; ++i, p += 2 + cb) {
                        p[0] = uint8_t(bt->labels[i]);
                        p[1] = r.flags[i];
                        std::memcpy(p + 2, r.codes + i * cb, cb);
                    }
                    if (emit_minima) ob.minima.assign(r.minima, r.minima + r.n * f.k);
                    if (r.scores) ob.scores.assign(r.scores, r.scores + r.n);
                    kernel_ms[di] += r.kernel_ms;
                    const uint64_t seq = bt->seq;
                    free_q.push(bt);
                    done.put(seq, std::move(ob));
                };
                Batch* bt = nullptr;
                while (in_q.pop(bt)) {
                    ChunkJob job;
                    job.tag = bt->seq;
                    job.row_ptr = bt->row_ptr.data();
                    job.index_base = 0;
                    job.indices = bt->ids;
                    job.n = bt->n;
                    job.pinned_input = true;
                    if (bt->want_device_ids && bt->d_dev == devs[di] && bt->d_valid == bt->nids())
                        job.d_indices = bt->d_ids;
                    inflight[bt->seq] = bt;
                    lane.submit(job, on_done);
                }
                lane.drain(on_done);
            } catch (...) {
                record_error(std::current_exception());
            }
        });
    }

    // the calling thread is the order-restoring writer (pipeline.cpp:193-204)
    try {
        OutBatch ob;
        for (uint64_t seq = 0; done.take(seq, ob); ++seq) {
            const auto t0 = Clock::now();
            append(ob);
            stats.write_seconds += since(t0);
        }
    } catch (...) {
        record_error(std::current_exception());
    }
    trace("stream: writer done");
    rd.join();
    for (auto& t : lanes) t.join();
    trace("stream: joined");
    if (error) std::rethrow_exception(error);
    for (double ms : kernel_ms) stats.compute_seconds += ms * 1e-3;
    PipelineProfile& pr = t_profile;
    pr.io_seconds = reader.io_seconds();
    pr.parse_seconds = reader.parse_seconds();
    pr.load_seconds = stats.read_seconds;
    pr.hash_seconds = stats.compute_seconds;
    pr.write_seconds = stats.write_seconds;
    pr.records = stats.records;
    pr.lanes = devs.size();
    pr.ranges = 0;
    return stats;
}

// order-restoring buffer over (range, batch) keys: range r's batches come
// before range r+1's; a range's batch count is known when its loader is done
class RangeReorder {
public:
    using Key = std::pair<uint64_t, uint64_t>;
    void put(Key key, OutBatch&& b) {
        std::lock_guard lk(m_);
        done_[key] = std::move(b);
        cv_.notify_all();
    }
    void set_range_total(uint64_t r, uint64_t total) {
        std::lock_guard lk(m_);
        totals_[r] = total;
        cv_.notify_all();
    }
    // false at the end of range r (or on abort)
    bool take(Key key, OutBatch& out) {
        std::unique_lock lk(m_);
        cv_.wait(lk, [&] {
            if (aborted_ || done_.count(key)) return true;
            auto t = totals_.find(key.first);
            return t != totals_.end() && key.second >= t->second;
        });
        if (aborted_) return false;
        auto it = done_.find(key);
        if (it == done_.end()) return false;
        out = std::move(it->second);
        done_.erase(it);
        return true;
    }
    void abort() {
        std::lock_guard lk(m_);
        aborted_ = true;
        cv_.notify_all();
    }

private:
    std::mutex m_;
    std::condition_variable cv_;
    std::map<Key, OutBatch> done_;
    std::map<uint64_t, uint64_t> totals_;
    bool aborted_ = false;
};

// Range-sharded LibSVM text (several GPUs sketching one text file): the file
// is cut at line starts into `lanes * range_shards` byte ranges. Every lane
// has its own loader thread, which claims ranges in order and reads, parses
// (on the lane's own GPU, ids left there) and batches them; its lane thread
// sketches them. Nothing goes back through the host or another GPU, and no
// single reader or parser bounds the file. The calling thread writes range 0's
// batches, then range 1's, ... so the bytes equal the one-reader pipeline's
// (pipeline.cpp:76-119 ordering). A parse error is reported as the reference
// reports it -- the first bad line in file order, numbered from the start of
// the file: a range's error is raised when the writer reaches it, after every
// earlier range has been written and counted.
template <typename Append>
PipelineStats run_ranged(const Family& f, const std::string& path, unsigned threads, uint8_t b,
                         bool emit_minima, const ScoreModel* score, Append&& append) {
    trace("ranged: start");
    PipelineStats stats;
    const size_t cb = packed_code_bytes(f.k, b);
    // lanes: the pipeline's GPUs, repeated up to the "text_lanes" loader count
    // (several loaders per GPU overlap one range's read with another's parse)
    const std::vector<int> gpus = pipeline_devices();
    std::vector<int> devs;
    const size_t nlanes = std::max<size_t>(gpus.size(), size_t(std::max<int64_t>(1, opt(Opt::TextLanes))));
    for (size_t i = 0; i < nlanes; ++i) devs.push_back(gpus[i % gpus.size()]);
    const uint64_t max_docs = chunk_docs_setting();
    const bool b_ok = b >= 1 && b <= 32;
    const uint64_t size = file_size(path);
    const uint64_t nr = std::max<uint64_t>(1, devs.size() * uint64_t(std::max<int64_t>(1, opt(Opt::RangeShards))));
    std::vector<uint64_t> cut(nr + 1, size);
    cut[0] = 0;
    for (uint64_t r = 1; r < nr; ++r)
        cut[r] = std::max(cut[r - 1], line_start_at_or_after(path, size / nr * r));

    struct RangeErr {
        Errc code = Errc::Io;
        uint64_t line = 0;
        std::string detail;
        bool set = false;
    };
    std::vector<RangeErr> range_err(nr);
    std::vector<uint64_t> range_lines(nr, 0);
    std::atomic<uint64_t> next_range{0}, err_range{UINT64_MAX}, records{0};
    std::atomic<uint64_t> io_ns{0}, parse_ns{0}, load_ns{0};
    RangeReorder done;
    std::mutex err_mu;
    std::exception_ptr error;
    struct LaneQueues {
        BlockingQueue<Batch*> free_q, in_q;
    };
    std::vector<std::unique_ptr<LaneQueues>> qs;
    for (size_t i = 0; i < devs.size(); ++i) qs.push_back(std::make_unique<LaneQueues>());
    auto record_error = [&](std::exception_ptr e) {
        {
            std::lock_guard lk(err_mu);
            if (!error) error = e;
        }
        for (auto& q : qs) {
            q->free_q.abort();
            q->in_q.abort();
        }
        done.abort();
    };
    const size_t per_lane = 4;
    BatchLease storage(per_lane * devs.size());
    for (size_t i = 0; i < storage.batches.size(); ++i) qs[i / per_lane]->free_q.push(storage.batches[i]);
    auto ns_since = [](Clock::time_point t0) {
        return uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count());
    };

    std::vector<std::thread> loaders, lanes;
    for (size_t di = 0; di < devs.size(); ++di) {
        loaders.emplace_back([&, di] {
            LaneQueues& q = *qs[di];
            try {
                BBMH_CUDA(cudaSetDevice(devs[di]));
                for (uint64_t r; (r = next_range.fetch_add(1)) < nr;) {
                    if (r > err_range.load()) break;  // an earlier range failed: the rest is moot
                    count(Counter::RangeShards);
                    uint64_t seq = 0;
                    auto reader = open_libsvm_range(path, threads, cut[r], cut[r + 1]);
                    const bool device_ids = reader->parser_device() == devs[di] && opt(Opt::DeviceIds);
                    try {
                        for (;;) {
                            Batch* bt = nullptr;
                            if (!q.free_q.pop(bt)) return;
                            const auto t0 = Clock::now();
                            bt->clear();
                            bt->want_device_ids = device_ids;
                            if (!device_ids) bt->reserve_ids(kBatchIds + kBatchIds / 4);
                            bool got = false;
                            try {
                                got = reader->fill(*bt, max_docs, kBatchIds);
                            } catch (...) {
                                q.free_q.push(bt);
                                throw;
                            }
                            load_ns += ns_since(t0);
                            if (!got) {
                                q.free_q.push(bt);
                                break;
                            }
                            if (!b_ok) fail(Errc::InvalidArgument, "b must be in 1..32");  // sketch.cpp:73
                            bt->seq = r;
                            bt->first_record = seq++;  // (range, batch) key of this batch
                            records += bt->n;
                            if (bt->want_device_ids && bt->d_dev == devs[di] && bt->d_valid == bt->nids())
                                count(Counter::DeviceIdBatches);
                            q.in_q.push(bt);
                            if (r > err_range.load()) break;
                        }
                    } catch (const LineError& e) {
                        std::lock_guard lk(err_mu);
                        range_err[r] = {e.code(), e.line(), e.detail(), true};
                        uint64_t cur = err_range.load();
                        while (r < cur && !err_range.compare_exchange_weak(cur, r)) {
                        }
                    }
                    range_lines[r] = reader->lines_consumed();
                    io_ns += uint64_t(reader->io_seconds() * 1e9);
                    parse_ns += uint64_t(reader->parse_seconds() * 1e9);
                    done.set_range_total(r, seq);
                }
                q.in_q.close();
            } catch (...) {
                record_error(std::current_exception());
            }
        });
    }
    std::vector<double> kernel_ms(devs.size(), 0.0);
    for (size_t di = 0; di < devs.size(); ++di) {
        lanes.emplace_back([&, di] {
            LaneQueues& q = *qs[di];
            try {
                BBMH_CUDA(cudaSetDevice(devs[di]));
                Lane lane(f, devs[di], b_ok ? b : 8, emit_minima, score);
                std::map<uint64_t, Batch*> inflight;
                uint64_t tag = 0;
                auto on_done = [&](const ChunkResult& res) {
                    Batch* bt = inflight.at(res.tag);
                    inflight.erase(res.tag);
                    OutBatch ob;
                    ob.n = res.n;
                    ob.recs.resize(res.n * (2 + cb));
                    uint8_t* p = ob.recs.data();
                    for (uint64_t i = 0; i < res.n; ++i, p += 2 + cb) {
                        p[0] = uint8_t(bt->labels[i]);
                        p[1] = res.flags[i];
                        std::memcpy(p + 2, res.codes + i * cb, cb);
                    }
                    if (emit_minima) ob.minima.assign(res.minima, res.minima + res.n * f.k);
                    if (res.scores) ob.scores.assign(res.scores, res.scores + res.n);
                    kernel_ms[di] += res.kernel_ms;
                    const RangeReorder::Key key{bt->seq, bt->first_record};
                    q.free_q.push(bt);
                    done.put(key, std::move(ob));
                };
                Batch* bt = nullptr;
                while (q.in_q.pop(bt)) {
                    ChunkJob job;
                    job.tag = tag;
                    job.row_ptr = bt->row_ptr.data();
                    job.index_base = 0;
                    job.indices = bt->ids;
                    job.n = bt->n;
                    job.pinned_input = true;
                    if (bt->want_device_ids && bt->d_dev == devs[di] && bt->d_valid == bt->nids())
                        job.d_indices = bt->d_ids;
                    inflight[tag++] = bt;
                    lane.submit(job, on_done);
                }
                lane.drain(on_done);
            } catch (...) {
                record_error(std::current_exception());
            }
        });
    }

    // the calling thread writes the ranges in file order
    try {
        uint64_t lines_before = 0;
        for (uint64_t r = 0; r < nr; ++r) {
            OutBatch ob;
            for (uint64_t s = 0; done.take({r, s}, ob); ++s) {
                const auto t0 = Clock::now();
                append(ob);
                stats.write_seconds += since(t0);
            }
            {
                std::lock_guard lk(err_mu);
                if (error) break;
            }
            if (range_err[r].set) {
                const RangeErr& e = range_err[r];
                throw LineError(e.code, lines_before + e.line, e.detail);
            }
            lines_before += range_lines[r];
        }
    } catch (...) {
        record_error(std::current_exception());
    }
    for (auto& t : loaders) t.join();
    for (auto& t : lanes) t.join();
    trace("ranged: joined");
    if (error) std::rethrow_exception(error);
    stats.records = records.load();
    stats.read_seconds = double(load_ns.load()) * 1e-9;
    for (double ms : kernel_ms) stats.compute_seconds += ms * 1e-3;
    PipelineProfile& pr = t_profile;
    pr.io_seconds = double(io_ns.load()) * 1e-9;
    pr.parse_seconds = double(parse_ns.load()) * 1e-9;
    pr.load_seconds = stats.read_seconds;
    pr.hash_seconds = stats.compute_seconds;
    pr.write_seconds = stats.write_seconds;
    pr.records = stats.records;
    pr.lanes = devs.size();
    pr.ranges = nr;
    return stats;
}

// LibSVM text files are read as line-aligned ranges by several loader lanes
// (run_ranged): one per GPU at least, "text_lanes" in all (on one GPU, 4
// lanes took C4 text from 29.3 to 35.2 GB/s with 2U and from 15.8 to
// 19.3 GB/s with 4U, profiles/round2/c4_lanes_*.jsonl); "range_shards" = 0
// keeps one shared reader.
bool use_ranges(const std::string& path) {
    const int64_t rs = opt(Opt::RangeShards);
    if (rs <= 0) return false;
    const size_t lanes = std::max<size_t>(pipeline_devices().size(), size_t(std::max<int64_t>(1, opt(Opt::TextLanes))));
    return (lanes > 1 || rs > 1) && is_libsvm_text(path);
}

}  // namespace

PipelineProfile last_pipeline_profile() { return t_profile; }

PipelineStats sketch_file(const Family& f, const std::string& input_path,
                          const std::string& output_path, uint8_t b, uint64_t chunk_size,
                          uint32_t workers, bool emit_minima) {
    const auto wall0 = Clock::now();
    t_profile = PipelineProfile{};
    // open order as in sketch_file (pipeline.cpp:217-220) and sketch_stream (:125-126)
    auto reader = open_corpus(input_path, workers ? workers : 1);
    SketchWriter writer(output_path, f, b, emit_minima);
    if (chunk_size < 1) fail(Errc::InvalidArgument, "chunk_size must be >= 1");
    if (workers < 1) fail(Errc::InvalidArgument, "workers must be >= 1");
    auto sink = [&](const OutBatch& ob) { writer.append(ob); };
    PipelineStats stats;
    if (use_ranges(input_path)) {
        reader.reset();  // each lane opens its own ranges
        stats = run_ranged(f, input_path, workers, b, emit_minima, nullptr, sink);
    } else {
        stats = run_stream(f, *reader, b, emit_minima, nullptr, sink);
    }
    writer.close();
    stats.chunks = (stats.records + chunk_size - 1) / chunk_size;  // reference chunking
    stats.wall_seconds = since(wall0);
    t_profile.wall_seconds = stats.wall_seconds;
    t_profile.input_bytes = file_size(input_path);
    return stats;
}

// load_model (learner.cpp:588-612): "BBLM", u64 dim, u8 loss, u8 averaging,
// dim doubles w, [dim doubles w_avg]; decision weights = averaging ? w_avg : w
std::vector<double> load_decision_weights(const std::string& path) {
    FILE* fm = open_or_fail(path, "rb");
    struct Closer {
        FILE* f;
        ~Closer() { std::fclose(f); }
    } guard{fm};
    auto read_exact = [&](void* p, size_t n) {
        if (std::fread(p, 1, n, fm) != n) fail(Errc::Io, "short read");
    };
    char magic[4];
    if (std::fread(magic, 1, 4, fm) != 4 || std::memcmp(magic, "BBLM", 4) != 0)
        fail(Errc::MalformedLine, path + ": not a BBLM model file");
    uint8_t d8[8];
    read_exact(d8, 8);
    const uint64_t dim = get_u64(d8);
    uint8_t tags[2];
    if (std::fread(tags, 1, 2, fm) != 2 || tags[0] > 1 || tags[1] > 1)
        fail(Errc::MalformedLine, path + ": bad loss/averaging tags");
    std::vector<double> w(dim);
    read_exact(w.data(), dim * sizeof(double));
    if (tags[1]) read_exact(w.data(), dim * sizeof(double));  // w_avg replaces w
    return w;
}

PipelineStats predict_file(const Family& f, uint8_t b, const std::string& model_path,
                           const std::string& corpus_path, const std::string& scores_path,
                           uint32_t workers, double* accuracy) {
    const auto wall0 = Clock::now();
    trace("predict: start");
    // bbmh_predict order (capi.cpp:307-317): model, data, then the scores table
    std::vector<double> w = load_decision_weights(model_path);
    trace("predict: model loaded");
    auto reader = open_corpus(corpus_path, workers ? workers : 1);
    trace("predict: corpus open");
    FILE* out = nullptr;
    if (!scores_path.empty()) {
        out = scores_path == "-" ? stdout : std::fopen(scores_path.c_str(), "wb");
        if (!out) fail(Errc::Io, scores_path + ": cannot open for writing");
    }
    struct Closer {
        FILE* f;
        ~Closer() {
            if (f && f != stdout) std::fclose(f);
        }
    } guard{out};
    ScoreModel model{w.data(), w.size()};
    uint64_t n = 0, correct = 0;
    std::string line;
    PipelineStats stats = run_stream(f, *reader, b, false, &model, [&](const OutBatch& ob) {
        const size_t rb = 2 + packed_code_bytes(f.k, b);
        for (uint64_t i = 0; i < ob.n; ++i) {  // predict_file (learner.cpp:524-536)
            const double score = ob.scores[i];
            const int cls = score >= 0 ? 1 : -1;
            if (out) std::fprintf(out, "%d\t%.9g\n", cls, score);
            correct += cls == int8_t(ob.recs[i * rb]);
        }
        n += ob.n;
    });
    trace("predict: stream done");
    if (accuracy) *accuracy = n ? double(correct) / double(n) : 0.0;
    stats.wall_seconds = since(wall0);
    return stats;
}

}  // namespace bbmh
