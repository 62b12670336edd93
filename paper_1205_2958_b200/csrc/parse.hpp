// parse.hpp -- LibSVM text -> CSR on the GPU (the loader's fast path).
//
// The reference parses one line at a time with strtod/strtoll on one thread
// (parse_libsvm, dataio.cpp:60-106; LibsvmSource::next, :157-190). Here a
// whole block of complete lines is copied to the device and split, tokenised
// and converted by byte-parallel kernels. Only a strict subset of the grammar
// is accepted on the device -- every line "L( SEP I:1)* SEP* CR?" with
// L in {+1,-1,1,0,+0,-0}, SEP in {' ','\t'}, I a decimal in [1, 2^32-1],
// ids strictly ascending, no '#'. A block with anything else (comments,
// other spellings of numbers, errors) is reported as not parsed and the
// caller parses it with the CPU parser, which reproduces the reference's
// values, line numbers and messages exactly.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <vector>

namespace bbmh {

struct GpuParseResult {
    bool ok = false;           // false: the block must be parsed on the CPU
    bool over_budget = false;  // declined only because it holds more than max_rows / max_ids
    uint64_t lines = 0;        // lines consumed (blank ones included)
    uint64_t rows = 0;         // non-blank lines
    uint64_t ids = 0;          // ids written
    uint64_t bytes = 0;        // bytes consumed: the block, or the prefix that fit the budget
};

// Device-resident output of a block's ids: reserve(n) returns a device buffer
// (on the parser's device) of at least n ids; entries from `base` on receive
// the block's ids, which are then not copied to the host.
struct DeviceIdsOut {
    std::function<uint32_t*(uint64_t)> reserve;
    uint64_t base = 0;
};

class GpuLibsvmParser {
public:
    explicit GpuLibsvmParser(int device);
    ~GpuLibsvmParser();
    GpuLibsvmParser(const GpuLibsvmParser&) = delete;
    GpuLibsvmParser& operator=(const GpuLibsvmParser&) = delete;

    // `text` (page-locked) holds complete lines: it ends with '\n', or is the
    // end of the file (`at_eof`). On success the rows are appended: ids (0-based)
    // to ids_out (capacity checked through `reserve`, which may move it),
    // row ends (offset by `id_base`) to row_ptr, labels to labels. At most
    // max_rows rows and max_ids ids are taken: from a block holding more, the
    // longest prefix of whole lines within both (r.bytes < len); if not even
    // its first row fits, r.over_budget. `key` names the block (its file
    // offset) for matching a prefetch; `next_*`, if set, is the block expected
    // after this one, whose copy is started as soon as this one's kernels are
    // queued.
    template <typename Reserve>
    GpuParseResult parse(const char* text, uint64_t len, bool at_eof, uint64_t id_base,
                         uint64_t max_rows, uint64_t max_ids, Reserve&& reserve,
                         std::vector<uint64_t>& row_ptr, std::vector<int8_t>& labels,
                         uint64_t key, const char* next_text = nullptr, uint64_t next_len = 0,
                         uint64_t next_key = 0, const DeviceIdsOut* dev_out = nullptr) {
        GpuParseResult r = run(text, len, at_eof, max_rows, max_ids, key, next_text, next_len,
                               next_key, dev_out);
        if (!r.ok) return r;
        uint32_t* ids_out = dev_out ? nullptr : reserve(id_base + r.ids) + id_base;
        fetch(ids_out, id_base, row_ptr, labels, r);
        return r;
    }
    int device() const { return device_; }

    // Starts the H2D copy of a block on a copy stream; parse() of the same
    // (key, len) then skips its own copy. The host bytes must stay untouched
    // until that parse() returns, wait_prefetch() or cancel_prefetch().
    void prefetch(const char* text, uint64_t len, uint64_t key);
    bool prefetched(uint64_t key, uint64_t len) const { return pf_len_ && pf_key_ == key && pf_len_ == len; }
    void wait_prefetch();    // the pending copy's host bytes may be overwritten after this
    void cancel_prefetch();  // wait_prefetch() and forget it

private:
    GpuParseResult run(const char* text, uint64_t len, bool at_eof, uint64_t max_rows,
                       uint64_t max_ids, uint64_t key, const char* next_text, uint64_t next_len,
                       uint64_t next_key, const DeviceIdsOut* dev_out);
    void fetch(uint32_t* ids_out, uint64_t id_base, std::vector<uint64_t>& row_ptr,
               std::vector<int8_t>& labels, const GpuParseResult& r);
    void grow(uint64_t len);

    int device_ = 0;
    cudaStream_t st_ = nullptr;
    uint64_t cap_text_ = 0, cap_seg_ = 0, cap_lines_ = 0, cap_ids_ = 0;
    char* d_text_ = nullptr;     // text of the block being parsed
    char* d_next_ = nullptr;     // prefetched text of the next block (swapped in)
    uint64_t cap_next_ = 0;
    cudaStream_t copy_st_ = nullptr;
    cudaEvent_t copied_ = nullptr;
    uint64_t pf_key_ = 0, pf_len_ = 0;  // the prefetched block (pf_len_ > 0: one is pending)
    bool pf_waited_ = false;
    unsigned long long* d_seg_ = nullptr;   // per segment: newlines << 32 | colons, then scanned
    uint64_t* d_line_end_ = nullptr;        // position of each line's '\n' (or len)
    uint32_t* d_colons_before_ = nullptr;   // ids before each line start (lines + 1)
    uint32_t* d_line_tok_ = nullptr;        // tokens per line
    uint32_t* d_row_of_line_ = nullptr;     // 1 for non-blank lines, then scanned
    int8_t* d_line_label_ = nullptr;
    uint32_t* d_ids_ = nullptr;             // ids (host-bound blocks)
    uint32_t* ids_dst_ = nullptr;           // where the current block's ids went
    uint64_t* d_row_end_ = nullptr;         // rows: end (exclusive) in ids
    int8_t* d_labels_ = nullptr;
    uint32_t* d_flags_ = nullptr;           // [0] bad, [1] rows, [2] lines, [3] ids, [4..8) prefix
    uint32_t* h_flags_ = nullptr;           // pinned mirror
    void* d_scan_tmp_ = nullptr;
    size_t scan_tmp_bytes_ = 0;
};

// Option "gpu_parse" = 0 disables the device parser (CPU parsing only); read when a
// reader is opened. Option "gpu_parse_block" (bytes) overrides the block size.
bool gpu_parse_enabled();
uint64_t gpu_parse_block_bytes(uint64_t dflt);

}  // namespace bbmh
