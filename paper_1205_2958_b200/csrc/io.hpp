// io.hpp -- corpus readers (BBCV binary, LibSVM text) that fill pinned CSR
// batches, and the little-endian helpers shared by the BBMH/BBCV writers.
//
// Byte formats and validation follow the reference:
//   BBCV   dataio.hpp:36-40, dataio.cpp:127-153 (writer), 192-245 (reader)
//   LibSVM dataio.cpp:60-106 (parse), 115-125 (write), 157-190 (reader)
//   BBMH   sketch.hpp:56-60, sketch.cpp:10-12, 102-141
#pragma once

#include <cstdint>
#include <cstdio>
#include <memory>
#include <string>
#include <vector>

#include "core.hpp"

namespace bbmh {

// A CSR batch of consecutive records; ids live in page-locked memory so the
// GPU lanes can DMA them directly.
struct Batch {
    uint64_t seq = 0;           // batch number
    uint64_t first_record = 0;  // index of row 0 in the corpus
    uint64_t n = 0;
    std::vector<uint64_t> row_ptr{0};
    std::vector<int8_t> labels;
    uint32_t* ids = nullptr;  // pinned
    uint64_t cap_ids = 0;
    std::vector<float> vals;  // per-id values (LibSVM value mode only)

    // Device-resident ids. A consumer on the GPU that parses LibSVM text sets
    // want_device_ids: the parser then writes the ids straight into d_ids on
    // d_dev (no D2H, and no H2D by the lane later), and when fill() returns
    // ids [0, nids()) are all valid there; `ids` on the host then holds only
    // the rows the CPU parser took (blocks outside the device grammar).
    bool want_device_ids = false;
    int d_dev = -1;
    uint32_t* d_ids = nullptr;
    uint64_t d_cap = 0;
    uint64_t d_valid = 0;  // ids [0, d_valid) are on the device

    ~Batch();
    void reserve_ids(uint64_t cap);  // keeps contents
    // device buffer of >= cap ids (+ the kernels' granule slack) on `dev`; keeps [0, d_valid)
    uint32_t* reserve_device_ids(int dev, uint64_t cap);
    void clear() {
        n = 0;
        row_ptr.assign(1, 0);
        labels.clear();
        vals.clear();
        d_valid = 0;
    }
    uint64_t nids() const { return row_ptr.back(); }
};

class CorpusReader {
public:
    virtual ~CorpusReader() = default;
    // Appends records until `max_docs` rows or `max_ids` ids are reached
    // (a single row may exceed max_ids). Returns false at end of input with
    // no record appended. Throws bbmh::Error with the reference's messages.
    virtual bool fill(Batch& b, uint64_t max_docs, uint64_t max_ids) = 0;
    // The GPU that parses this corpus (-1: none): batches filled with
    // want_device_ids get their ids there.
    virtual int parser_device() const { return -1; }
    // Lines of text consumed so far (blank ones included; 0 for binary input).
    virtual uint64_t lines_consumed() const { return 0; }
    // Seconds spent reading the file (pread, summed over the threads that
    // wait for it) and parsing blocks (GPU parser calls, CPU parser rounds).
    virtual double io_seconds() const { return 0; }
    virtual double parse_seconds() const { return 0; }
};

// open_corpus: sniff the "BBCV" magic, else LibSVM text (dataio.cpp:257-264).
// libsvm_values: keep real values instead of requiring 1 (the prediction
// row source, learner.cpp:236-256).
std::unique_ptr<CorpusReader> open_corpus(const std::string& path, unsigned parse_threads,
                                          bool libsvm_values = false);

// True if `path` is LibSVM text (no BBCV magic).
bool is_libsvm_text(const std::string& path);

// Byte size of a file.
uint64_t file_size(const std::string& path);

// The offset of the first line that starts at or after `off` (0 stays 0;
// the size of the file if no line starts there): the cut points of
// range-sharded text, so every range holds whole lines.
uint64_t line_start_at_or_after(const std::string& path, uint64_t off);

// LibSVM text (binary mode, the sketch loader) restricted to the whole lines
// in [begin, end) -- begin and end are line starts or the end of the file.
// Line numbers in its errors count from the range's first line (1-based).
// The GPU parser, if used, runs on the current device.
std::unique_ptr<CorpusReader> open_libsvm_range(const std::string& path, unsigned parse_threads,
                                                uint64_t begin, uint64_t end);

// BBMH sketch file reader (SketchReader, sketch.cpp:143-207): header checks
// with the reference's messages, then records in batches (label, flags,
// ceil(k*b/8) code bytes each). A truncated record raises Io "short read"
// after the complete records before it have been returned.
class SketchFileReader {
public:
    explicit SketchFileReader(const std::string& path);
    ~SketchFileReader();
    SketchFileReader(const SketchFileReader&) = delete;
    SketchFileReader& operator=(const SketchFileReader&) = delete;
    uint32_t k() const { return k_; }
    uint32_t b() const { return b_; }
    uint8_t scheme() const { return scheme_; }
    uint64_t dim() const { return dim_; }
    uint64_t seed() const { return seed_; }
    uint64_t count() const { return count_; }
    // Up to max_rows records; returns how many (0 at the end).
    uint64_t read(uint64_t max_rows, std::vector<uint8_t>& codes, std::vector<uint8_t>& flags,
                  std::vector<int8_t>& labels);
    // Position at record i (SketchReader::record, sketch.cpp:190-201).
    void seek(uint64_t i);

private:
    FILE* f_ = nullptr;
    uint32_t k_ = 0, b_ = 0;
    uint8_t scheme_ = 0;
    uint64_t dim_ = 0, seed_ = 0, count_ = 0, done_ = 0;
    bool short_ = false;
    std::vector<uint8_t> buf_;
};

// little-endian helpers
inline void put_u32(uint8_t* p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = uint8_t(v >> (8 * i));
}
inline void put_u64(uint8_t* p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = uint8_t(v >> (8 * i));
}
inline uint32_t get_u32(const uint8_t* p) {
    return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}
inline uint64_t get_u64(const uint8_t* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
    return v;
}

FILE* open_or_fail(const std::string& path, const char* mode);
void write_all(FILE* f, const void* data, size_t n);

}  // namespace bbmh
