// hostpool.hpp -- persistent host worker threads for the data-parallel host
// passes of the chunk pipeline (id encoding, result copies). Spawning threads
// per chunk costs ~100 us against ~1 ms of work per chunk; these are created
// once per process.
#pragma once

#include <cstddef>
#include <functional>

namespace bbmh {

// Threads available to host_parallel (the caller included).
unsigned host_threads();

// Runs fn(w) for every w in [0, tasks) on the pool, the calling thread taking
// its share; returns when all have run. Concurrent callers take turns. The
// first exception thrown by a task is rethrown here.
void host_parallel(unsigned tasks, const std::function<void(unsigned)>& fn);

// Host DRAM copy bandwidth (read + write bytes/s) of host_memcpy over the
// whole pool, measured once per process on first use (~0.2 s: 2 x 256 MiB),
// unless the "host_dram_gbs" option gives it.
double host_dram_bytes_per_s();

// memcpy split over the pool in pieces of >= 256 KiB (one thread copies ~10 GB/s).
void host_memcpy(void* dst, const void* src, size_t n);

}  // namespace bbmh
