// hostpool.cpp -- see hostpool.hpp.
#include "hostpool.hpp"
#include "options.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <new>
#include <pthread.h>
#include <thread>
#include <vector>

namespace bbmh {

namespace {

class Pool {
public:
    Pool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned n = std::min(hw, 64u) - 1;  // the caller is the last worker
        for (unsigned i = 0; i < n; ++i) threads_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    unsigned size() const { return unsigned(threads_.size()) + 1; }

    void run(unsigned tasks, const std::function<void(unsigned)>& fn) {
        if (tasks == 0) return;
        if (tasks == 1 || threads_.empty()) {
            for (unsigned w = 0; w < tasks; ++w) fn(w);
            return;
        }
        std::lock_guard turn(turn_mu_);  // one job at a time
        auto job = std::make_shared<Job>();
        job->fn = &fn;
        job->tasks = tasks;
        {
            std::lock_guard lk(mu_);
            job_ = job;
            ++gen_;
        }
        cv_.notify_all();
        work(*job);
        std::unique_lock lk(mu_);
        done_cv_.wait(lk, [&] { return job->done == job->tasks; });
        job_.reset();
        if (job->err) std::rethrow_exception(job->err);
    }

private:
    struct Job {
        const std::function<void(unsigned)>* fn = nullptr;
        unsigned tasks = 0, done = 0;  // done: under mu_
        std::atomic<unsigned> next{0};
        std::exception_ptr err;        // under mu_
    };

    // takes tasks of `j` until none are left (a worker that wakes late for a
    // finished job finds none)
    void work(Job& j) {
        unsigned ran = 0;
        std::exception_ptr err;
        for (unsigned w; (w = j.next.fetch_add(1)) < j.tasks;) {
            try {
                (*j.fn)(w);
            } catch (...) {
                if (!err) err = std::current_exception();
            }
            ++ran;
        }
        if (ran) {
            std::lock_guard lk(mu_);
            j.done += ran;
            if (err && !j.err) j.err = err;
            if (j.done == j.tasks) done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            std::shared_ptr<Job> j;
            {
                std::unique_lock lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                j = job_;
            }
            if (j) work(*j);
        }
    }

    std::vector<std::thread> threads_;
    std::mutex mu_, turn_mu_;
    std::condition_variable cv_, done_cv_;
    std::shared_ptr<Job> job_;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// Never destroyed (workers may outlive static teardown order). A forked child
// has none of the parent's threads: it starts a pool of its own.
std::mutex g_pool_mu;
Pool* g_pool = nullptr;

Pool& pool() {
    std::lock_guard lk(g_pool_mu);
    if (!g_pool) {
        static const bool registered = [] {
            pthread_atfork(nullptr, nullptr, [] {
                g_pool = nullptr;
                new (&g_pool_mu) std::mutex();
            });
            return true;
        }();
        (void)registered;
        g_pool = new Pool();
    }
    return *g_pool;
}

}  // namespace

unsigned host_threads() { return pool().size(); }

void host_parallel(unsigned tasks, const std::function<void(unsigned)>& fn) { pool().run(tasks, fn); }

void host_memcpy(void* dst, const void* src, size_t n) {
    const size_t T = std::min<size_t>(host_threads(), n >> 18);
    if (T <= 1) {
        std::memcpy(dst, src, n);
        return;
    }
    host_parallel(unsigned(T), [&](unsigned w) {
        const size_t lo = n * w / T, hi = n * (w + 1) / T;
        std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
    });
}

double host_dram_bytes_per_s() {
    if (const int64_t g = opt(Opt::HostDramGbs); g > 0) return double(g) * 1e9;
    static const double measured = [] {
        // 1 GiB, best of 4 (256 MiB, best of 3 read ~25% below a pinned
        // 1 GiB copy on the 16-core box, which skewed the transfer mix)
        constexpr size_t kBytes = size_t(1) << 30;
        char* a = static_cast<char*>(std::malloc(kBytes));
        char* b = static_cast<char*>(std::malloc(kBytes));
        if (!a || !b) {
            std::free(a);
            std::free(b);
            return 100e9;
        }
        host_parallel(host_threads(), [&](unsigned w) {  // fault the pages in on every core
            const size_t T = host_threads(), lo = kBytes * w / T, hi = kBytes * (w + 1) / T;
            std::memset(a + lo, 1, hi - lo);
            std::memset(b + lo, 0, hi - lo);
        });
        double best = 0;
        for (int rep = 0; rep < 4; ++rep) {
            const auto t0 = std::chrono::steady_clock::now();
            host_memcpy(b, a, kBytes);
            const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            best = std::max(best, 2.0 * double(kBytes) / s);
        }
        std::free(a);
        std::free(b);
        return best;
    }();
    return measured;
}

}  // namespace bbmh
