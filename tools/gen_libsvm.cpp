// gen_libsvm.cpp -- synthetic LibSVM corpus of a fixed shape, written fast
// enough to make tens of GB on the GPU box (config 4, the rcv1-expanded shape:
// 677,399 docs x ~12,000 ids over D = 1,010,017,424).
//
// Row r is a pure function of (seed, r): label +1/-1 from the parity of a
// hash, and `nnz` sorted unique ids uniform over [0, D) -- exponential
// spacings, so no sort: with gaps g_0..g_nnz ~ Exp(1) and partial sums S_i,
// id_i = floor(S_i / S_nnz+1 * (D - nnz)) + i is strictly increasing and < D.
// Text: "+1 <id+1>:1 <id+1>:1 ...\n" (1-based ids, binary values: the
// reference's loader grammar, dataio.cpp:60-106). Blocks of rows are
// formatted on all threads and written in row order.
//
//   g++ -O3 -march=native -pthread -o gen_libsvm tools/gen_libsvm.cpp
//   gen_libsvm OUT N_DOCS NNZ DIM SEED [THREADS] [FIRST_DOC]
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

static inline uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

static inline char* put_u32(char* p, uint32_t v) {
    char tmp[12];
    int n = 0;
    do {
        tmp[n++] = char('0' + v % 10);
        v /= 10;
    } while (v);
    while (n) *p++ = tmp[--n];
    return p;
}

int main(int argc, char** argv) {
    if (argc < 6) {
        std::fprintf(stderr, "usage: %s OUT N_DOCS NNZ DIM SEED [THREADS] [FIRST_DOC]\n", argv[0]);
        return 2;
    }
    const std::string out = argv[1];
    const uint64_t n = std::strtoull(argv[2], nullptr, 10);
    const uint64_t nnz = std::strtoull(argv[3], nullptr, 10);
    const uint64_t dim = std::strtoull(argv[4], nullptr, 10);
    const uint64_t seed = std::strtoull(argv[5], nullptr, 10);
    const unsigned T = argc > 6 ? unsigned(std::atoi(argv[6])) : std::thread::hardware_concurrency();
    const uint64_t first = argc > 7 ? std::strtoull(argv[7], nullptr, 10) : 0;
    if (nnz >= dim || dim > (1ull << 32)) {
        std::fprintf(stderr, "need nnz < dim <= 2^32\n");
        return 2;
    }
    FILE* f = std::fopen(out.c_str(), "wb");
    if (!f) {
        std::perror(out.c_str());
        return 1;
    }
    const uint64_t rows_per_block = std::max<uint64_t>(1, (32ull << 20) / (nnz * 12 + 8));
    const uint64_t nblocks = (n + rows_per_block - 1) / rows_per_block;
    std::atomic<uint64_t> next_block{0};
    uint64_t turn = 0;  // next block to write
    std::mutex mu;
    std::condition_variable cv;
    std::atomic<uint64_t> bytes{0};
    std::atomic<bool> bad{false};
    auto work = [&] {
        std::vector<double> g(nnz + 1);
        std::string buf;
        for (uint64_t blk; (blk = next_block.fetch_add(1)) < nblocks;) {
            const uint64_t r0 = blk * rows_per_block, r1 = std::min(n, r0 + rows_per_block);
            buf.resize((r1 - r0) * (nnz * 12 + 8));
            char* p = buf.data();
            for (uint64_t r = first + r0; r < first + r1; ++r) {
                uint64_t s = mix64(seed * 0x9e3779b97f4a7c15ull + r);
                *p++ = (s & 1) ? '+' : '-';
                *p++ = '1';
                double acc = 0;
                for (uint64_t i = 0; i <= nnz; ++i) {
                    s += 0x9e3779b97f4a7c15ull;
                    const double u = (double(mix64(s) >> 11) + 0.5) * 0x1.0p-53;  // (0, 1)
                    g[i] = acc;
                    acc -= std::log(u);
                }
                const double scale = double(dim - nnz) / acc;
                for (uint64_t i = 0; i < nnz; ++i) {
                    uint64_t x = uint64_t(g[i + 1] * scale);
                    if (x > dim - nnz) x = dim - nnz;
                    *p++ = ' ';
                    p = put_u32(p, uint32_t(x + i + 1));  // 1-based, strictly ascending
                    *p++ = ':';
                    *p++ = '1';
                }
                *p++ = '\n';
            }
            const size_t len = size_t(p - buf.data());
            std::unique_lock lk(mu);
            cv.wait(lk, [&] { return turn == blk; });
            if (std::fwrite(buf.data(), 1, len, f) != len) bad = true;
            bytes += len;
            ++turn;
            cv.notify_all();
        }
    };
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < std::max(1u, T); ++t) ts.emplace_back(work);
    for (auto& t : ts) t.join();
    if (std::fclose(f) != 0 || bad) {
        std::fprintf(stderr, "write failed\n");
        return 1;
    }
    std::printf("{\"docs\": %llu, \"nnz\": %llu, \"dim\": %llu, \"bytes\": %llu}\n", (unsigned long long)n,
                (unsigned long long)nnz, (unsigned long long)dim, (unsigned long long)bytes.load());
    return 0;
}
