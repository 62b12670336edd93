// replay.hpp -- epoch replay of a corpus as device CSR batches (replay.cu).
#pragma once

#include <cstdint>
#include <memory>
#include <string>

namespace bbmh {

struct ReplayInfo {
    bool sketch = false;  // BBMH sketch (expanded rows) or an original corpus (LibSVM / BBCV)
    uint8_t scheme = 0;
    uint32_t k = 0, b = 0;
    uint64_t dim = 0, seed = 0, count = 0;
    uint64_t expanded_dim = 0;  // 2^b * k (expanded_dim, expansion.cpp:9-15); 0 for corpora
};

struct ReplayStats {
    uint64_t epochs = 0, rows = 0, nnz = 0;
    double io_seconds = 0;      // pread of record blocks / corpus text
    double parse_seconds = 0;   // corpus parsing (original data only)
    double expand_seconds = 0;  // host side of next(): H2D + expansion (or upload) + sync
};

class Replay {
public:
    // `path`: BBMH (rows = the one-hot expansion of each record, SketchRowSource,
    // learner.cpp:271-297), BBCV or LibSVM (binary-mode rows, as the sketch
    // loader reads them). Batches hold up to max_rows rows, on `device`.
    Replay(const std::string& path, int device, uint64_t max_rows, unsigned threads);
    ~Replay();
    Replay(const Replay&) = delete;
    Replay& operator=(const Replay&) = delete;

    const ReplayInfo& info() const;
    ReplayStats stats() const;
    // Next batch; 0 at the end of the epoch. Device pointers and the host
    // views stay valid until the next call to next() or reset().
    uint64_t next(const uint64_t** d_row_ptr, const uint32_t** d_indices, const int8_t** labels,
                  const uint64_t** h_row_ptr);
    void reset();  // start the next epoch from the first row

private:
    struct Impl;
    std::unique_ptr<Impl> p_;
};

}  // namespace bbmh
