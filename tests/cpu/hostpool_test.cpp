// The host worker pool (csrc/hostpool.cpp): every task runs exactly once,
// concurrent callers take turns without losing tasks, the first exception
// reaches the caller, the pool keeps working after one, host_memcpy copies
// exactly, and a forked child gets a working pool of its own.
// Built and run by tests/test_hostpool_cpu.py.
#include "hostpool.hpp"

#include <sys/wait.h>
#include <unistd.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

using namespace bbmh;

static int fails = 0;
#define CHECK(c)                                                      \
    do {                                                              \
        if (!(c)) {                                                   \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);  \
            ++fails;                                                  \
        }                                                             \
    } while (0)

int main() {
    CHECK(host_threads() >= 1);
    // each task exactly once, many sizes
    for (unsigned tasks : {0u, 1u, 2u, 7u, 64u, 1000u}) {
        std::vector<std::atomic<int>> hit(tasks);
        for (auto& h : hit) h = 0;
        host_parallel(tasks, [&](unsigned w) { hit[w].fetch_add(1); });
        for (unsigned w = 0; w < tasks; ++w) CHECK(hit[w].load() == 1);
    }
    // concurrent callers
    {
        std::atomic<long> sum{0};
        std::vector<std::thread> ts;
        for (int c = 0; c < 6; ++c)
            ts.emplace_back([&] {
                for (int rep = 0; rep < 200; ++rep) host_parallel(37, [&](unsigned w) { sum += w + 1; });
            });
        for (auto& t : ts) t.join();
        CHECK(sum.load() == 6L * 200 * (37 * 38 / 2));
    }
    // exceptions: the first reaches the caller, every other task still runs
    {
        std::atomic<int> ran{0};
        bool caught = false;
        try {
            host_parallel(50, [&](unsigned w) {
                ran++;
                if (w % 10 == 3) throw std::runtime_error("task failed");
            });
        } catch (const std::runtime_error&) {
            caught = true;
        }
        CHECK(caught);
        CHECK(ran.load() == 50);
        std::atomic<int> after{0};
        host_parallel(20, [&](unsigned) { after++; });
        CHECK(after.load() == 20);
    }
    // host_memcpy
    for (size_t n : {size_t(0), size_t(1), size_t(1000), size_t(3) << 20, (size_t(17) << 20) + 5}) {
        std::vector<char> a(n), b(n, 0);
        for (size_t i = 0; i < n; ++i) a[i] = char(i * 31 + 7);
        host_memcpy(b.data(), a.data(), n);
        CHECK(std::memcmp(a.data(), b.data(), n) == 0);
    }
    // fork: the child has none of the parent's threads and must start its own pool
    {
        const pid_t pid = fork();
        if (pid == 0) {
            std::atomic<int> n{0};
            host_parallel(16, [&](unsigned) { n++; });
            _exit(n.load() == 16 ? 0 : 3);
        }
        int status = 0;
        waitpid(pid, &status, 0);
        CHECK(WIFEXITED(status) && WEXITSTATUS(status) == 0);
    }
    std::printf(fails ? "hostpool FAILED\n" : "hostpool ok\n");
    return fails ? 1 : 0;
}
