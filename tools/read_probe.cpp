// read_probe.cpp -- page-cache read bandwidth into page-locked memory: pread
// vs memcpy out of an mmap of the file, by thread count (the LibSVM loader's
// read-ahead, csrc/io.cpp read_at). Usage: read_probe <file> (file cached).
//   nvcc -O3 -std=c++17 -o /tmp/read_probe tools/read_probe.cpp -lpthread
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
    if (argc < 2) return 1;
    const int fd = open(argv[1], O_RDONLY);
    struct stat st {};
    fstat(fd, &st);
    const size_t size = size_t(st.st_size);
    const size_t block = size_t(32) << 20;
    char* dst = nullptr;
    cudaMallocHost(&dst, block);
    // warm the page cache
    {
        std::vector<char> tmp(block);
        for (size_t off = 0; off < size; off += block) (void)!pread(fd, tmp.data(), std::min(block, size - off), off);
    }
    for (int mode = 0; mode < 3; ++mode) {
        char* map = nullptr;
        if (mode >= 1) {
            map = static_cast<char*>(mmap(nullptr, size, PROT_READ, MAP_PRIVATE | (mode == 2 ? MAP_POPULATE : 0), fd, 0));
            madvise(map, size, MADV_SEQUENTIAL);
        }
        for (unsigned T : {4u, 8u, 16u}) {
            const double t0 = now();
            for (size_t off = 0; off < size; off += block) {
                const size_t n = std::min(block, size - off);
                std::vector<std::thread> ts;
                for (unsigned w = 0; w < T; ++w)
                    ts.emplace_back([&, w] {
                        const size_t lo = n * w / T, hi = n * (w + 1) / T;
                        if (mode == 0) {
                            size_t done = 0;
                            while (lo + done < hi) {
                                const ssize_t r = pread(fd, dst + lo + done, hi - lo - done, off_t(off + lo + done));
                                if (r <= 0) break;
                                done += size_t(r);
                            }
                        } else {
                            std::memcpy(dst + lo, map + off + lo, hi - lo);
                        }
                    });
                for (auto& t : ts) t.join();
            }
            const double dt = now() - t0;
            std::printf("{\"mode\": \"%s\", \"threads\": %u, \"GBps\": %.1f}\n",
                        mode == 0 ? "pread" : mode == 1 ? "mmap" : "mmap_populate", T, size / dt / 1e9);
        }
        if (map) munmap(map, size);
    }
    return 0;
}
