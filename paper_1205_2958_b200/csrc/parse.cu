// parse.cu -- LibSVM text -> CSR on the GPU (see parse.hpp for the grammar).
//
// Byte-parallel, four kernels per block of complete lines:
//   seg_count  one thread per 16 bytes (coalesced uint4 loads), per 4 KB CTA:
//              newlines and ':' (one per id), and a check that every byte is
//              in the fast grammar's alphabet;
//   (scan)     CTA bases + a block scan -> the line and id number of each byte;
//   seg_emit   every ':' converts the digits before it into ids[g] (checking
//              "SEP digits : 1 SEP"); every '\n' records its line's end and
//              id offset; token starts are counted per line;
//   line_check one warp per line: label, tokens == 1 + ids, strictly
//              ascending ids; (scan) non-blank lines -> rows; row_emit.
// Reference semantics: parse_libsvm (dataio.cpp:60-106) in binary mode with
// 0/1 labels accepted, blank lines skipped but numbered (dataio.cpp:166-175).
#include "parse.hpp"

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <initializer_list>
#include <string>

#include "core.hpp"
#include "options.hpp"
#include "engine.hpp"
#include "kernels.cuh"

namespace bbmh {

namespace {

constexpr uint32_t kTpb = 256;  // threads per CTA, one 16-byte chunk each: a segment is kTpb * 16 bytes

__device__ __forceinline__ bool is_sep(char c) { return c == ' ' || c == '\t'; }
__device__ __forceinline__ bool is_ws_or_nl(char c) {
    return c == ' ' || c == '\t' || c == '\r' || c == '\n';
}
__device__ __forceinline__ bool in_alphabet(char c) {
    return (c >= '0' && c <= '9') || c == ' ' || c == '\t' || c == '\r' || c == '\n' ||
           c == ':' || c == '+' || c == '-';
}

// this thread's 16 bytes (zero past the end of the text)
__device__ __forceinline__ void load16(const char* t, uint64_t len, uint64_t p0, char (&c)[16]) {
    if (p0 + 16 <= len) {
        const uint4 q = *reinterpret_cast<const uint4*>(t + p0);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 16; ++k) c[k] = char(w[k >> 2] >> (8 * (k & 3)));
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) c[k] = p0 + k < len ? t[p0 + k] : '\0';
    }
}

__device__ __forceinline__ unsigned long long count16(const char (&c)[16], uint64_t p0,
                                                      uint64_t len, bool& bad) {
    uint32_t nl = 0, col = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if (p0 + k < len) {
            nl += c[k] == '\n';
            col += c[k] == ':';
            bad |= !in_alphabet(c[k]);
        }
    }
    return ((unsigned long long)nl << 32) | col;
}

// per CTA (4 KB of text): newlines << 32 | colons
__global__ void __launch_bounds__(kTpb) seg_count(const char* __restrict__ t, uint64_t len,
                                                  unsigned long long* __restrict__ seg,
                                                  uint32_t* __restrict__ flags) {
    using Reduce = cub::BlockReduce<unsigned long long, kTpb>;
    __shared__ typename Reduce::TempStorage tmp;
    const uint64_t p0 = (blockIdx.x * (uint64_t)kTpb + threadIdx.x) * 16;
    char c[16];
    load16(t, len, p0, c);
    bool bad = false;
    const unsigned long long v = count16(c, p0, len, bad);
    const unsigned long long tot = Reduce(tmp).Sum(v);
    if (threadIdx.x == 0) seg[blockIdx.x] = tot;
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

// seg holds INCLUSIVE sums per CTA. Every ':' converts the digits before it;
// every '\n' closes its line; token starts are summed per line.
__global__ void __launch_bounds__(kTpb) seg_emit(const char* __restrict__ t, uint64_t len,
                                                 uint64_t nchunk, int at_eof,
                                                 const unsigned long long* __restrict__ seg,
                                                 uint64_t* __restrict__ line_end,
                                                 uint32_t* __restrict__ colons_before,
                                                 uint32_t* __restrict__ line_tok,
                                                 uint32_t* __restrict__ ids,
                                                 uint32_t* __restrict__ flags) {
    using Scan = cub::BlockScan<unsigned long long, kTpb>;
    __shared__ typename Scan::TempStorage tmp;
    const uint64_t chunk = blockIdx.x * (uint64_t)kTpb + threadIdx.x;
    const uint64_t p0 = chunk * 16;
    char c[16];
    load16(t, len, p0, c);
    bool bad = false;
    const unsigned long long mine = count16(c, p0, len, bad);
    unsigned long long before;
    Scan(tmp).ExclusiveSum(mine, before);
    before += blockIdx.x ? seg[blockIdx.x - 1] : 0ull;
    uint32_t line = uint32_t(before >> 32), col = uint32_t(before);
    if (chunk == 0) colons_before[0] = 0;
    char prev = p0 && p0 <= len ? t[p0 - 1] : '\n';  // chunks past the end read nothing
    uint32_t tok = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const uint64_t p = p0 + k;
        if (p >= len) break;
        const char ch = c[k];
        if (ch == '\n') {
            line_end[line] = p;
            colons_before[line + 1] = col;
            if (tok) atomicAdd(&line_tok[line], tok);
            tok = 0;
            ++line;
        } else {
            if (is_ws_or_nl(prev) && !is_ws_or_nl(ch)) ++tok;  // token start
            if (ch == ':') {
                // "SEP digits : 1 (SEP | CR | NL | end)"
                uint64_t q = p;
                uint32_t nd = 0;
                while (q > 0 && nd < 11 && t[q - 1] >= '0' && t[q - 1] <= '9') {
                    --q;
                    ++nd;
                }
                uint64_t v = 0;
                for (uint64_t i = q; i < p; ++i) v = v * 10 + uint64_t(t[i] - '0');
                const char bf = q > 0 ? t[q - 1] : '\n';
                const char a1 = p + 1 < len ? t[p + 1] : '\0';
                const bool a2_ok = p + 2 < len ? is_ws_or_nl(t[p + 2]) : (p + 2 == len && at_eof);
                if (nd < 1 || nd > 10 || !is_sep(bf) || v < 1 || v > 0xffffffffull || a1 != '1' ||
                    !a2_ok)
                    bad = true;
                ids[col] = uint32_t(v - 1);
                ++col;
            } else if (ch == '\r') {
                const bool ok = p + 1 < len ? t[p + 1] == '\n' : at_eof;
                if (!ok) bad = true;
            }
        }
        prev = ch;
    }
    // tokens after this chunk's last newline: one atomic per (warp, line)
    const uint32_t peers = __match_any_sync(0xffffffffu, line);
    const uint32_t sum = __reduce_add_sync(peers, tok);
    if (sum && (threadIdx.x & 31) == uint32_t(__ffs(peers) - 1)) atomicAdd(&line_tok[line], sum);
    if (chunk == nchunk - 1) {
        const bool open_last = at_eof && len > 0 && t[len - 1] != '\n';
        if (open_last) {
            line_end[line] = len;
            colons_before[line + 1] = col;
        }
        flags[2] = line + (open_last ? 1u : 0u);  // lines
        flags[3] = col;                            // ids
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

// one warp per line: label, token count, strictly ascending ids
__global__ void line_check(const char* __restrict__ t, uint32_t nlines,
                           const uint64_t* __restrict__ line_end,
                           const uint32_t* __restrict__ colons_before,
                           const uint32_t* __restrict__ line_tok, const uint32_t* __restrict__ ids,
                           uint32_t* __restrict__ row_flag, int8_t* __restrict__ line_label,
                           uint32_t* __restrict__ flags) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t li = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    if (li >= nlines) return;
    const uint64_t start = li ? line_end[li - 1] + 1 : 0, end = line_end[li];
    const uint32_t c0 = colons_before[li], c1 = colons_before[li + 1];
    if (start == end) {  // blank line: skipped, but numbered
        if (lane == 0) row_flag[li] = 0;
        return;
    }
    bool bad = false;
    if (lane == 0) {
        uint64_t p = start;
        int sign = 1;
        if (t[p] == '+') {
            ++p;
        } else if (t[p] == '-') {
            sign = -1;
            ++p;
        }
        const char d = p < end ? t[p] : '\n';
        const char nx = p + 1 < end ? t[p + 1] : '\n';
        if ((d != '0' && d != '1') || !is_ws_or_nl(nx)) bad = true;
        // label 1 / -1 as is; 0 (any sign) -> -1 (accept01, dataio.cpp:72-78)
        line_label[li] = int8_t(d == '1' ? sign : -1);
        if (line_tok[li] != 1 + (c1 - c0)) bad = true;
        row_flag[li] = 1;
    }
    for (uint32_t g = c0 + 1 + lane; g < c1; g += 32)
        if (ids[g] <= ids[g - 1]) bad = true;
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 1u);
}

// rows (non-blank lines, in order): end offsets and labels. row_idx EXCLUSIVE.
__global__ void row_emit(uint32_t nlines, const uint32_t* __restrict__ row_flag_scan,
                         const uint32_t* __restrict__ colons_before,
                         const int8_t* __restrict__ line_label, uint64_t* __restrict__ row_end,
                         int8_t* __restrict__ labels, uint32_t* __restrict__ flags,
                         const uint64_t* __restrict__ line_end) {
    const uint64_t li = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (li >= nlines) return;
    const uint64_t start = li ? line_end[li - 1] + 1 : 0;
    const bool row = start != line_end[li];
    const uint32_t r = row_flag_scan[li];
    if (row) {
        row_end[r] = colons_before[li + 1];
        labels[r] = line_label[li];
    }
    if (li == nlines - 1) flags[1] = r + (row ? 1u : 0u);
}

// The longest prefix of whole lines within the budget when the whole block is
// not: the line count L in [1, nlines) with L lines in budget and L + 1 not
// (rows and ids before a line only grow). flags[4..8) = L, its rows, its ids,
// its bytes; untouched (0) if not even one line fits.
__global__ void prefix_cut(uint32_t nlines, const uint32_t* __restrict__ rows_before,
                           const uint32_t* __restrict__ colons_before,
                           const uint64_t* __restrict__ line_end, uint64_t max_rows,
                           uint64_t max_ids, uint32_t* __restrict__ flags) {
    const uint64_t L = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (L >= nlines) return;
    auto fits = [&](uint64_t n) { return rows_before[n] <= max_rows && colons_before[n] <= max_ids; };
    if (fits(L) && (L + 1 == nlines || !fits(L + 1))) {
        flags[4] = uint32_t(L);
        flags[5] = rows_before[L];
        flags[6] = colons_before[L];
        flags[7] = uint32_t(line_end[L - 1] + 1);
    }
}

template <typename T>
void grow_dev(T*& p, uint64_t& cap, uint64_t need) {
    if (need <= cap) return;
    if (p) BBMH_CUDA(cudaFree(p));
    p = nullptr;
    const uint64_t n = need + need / 4;
    BBMH_CUDA(cudaMalloc(&p, n * sizeof(T)));
    cap = n;
}

}  // namespace

bool gpu_parse_enabled() { return opt(Opt::GpuParse) != 0; }

uint64_t gpu_parse_block_bytes(uint64_t dflt) {
    const int64_t v = opt(Opt::GpuParseBlock);
    return v >= 64 ? uint64_t(v) : dflt;
}

GpuLibsvmParser::GpuLibsvmParser(int device) : device_(device) {
    BBMH_CUDA(cudaSetDevice(device));
    // the parse kernels share the GPU with the sketch lanes' persistent
    // kernels; at the highest stream priority their CTAs are dispatched first
    // whenever SM slots free up (option "parse_priority")
    int lo = 0, hi = 0;
    if (opt(Opt::ParsePriority) && cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess) {
        BBMH_CUDA(cudaStreamCreateWithPriority(&st_, cudaStreamNonBlocking, hi));
        BBMH_CUDA(cudaStreamCreateWithPriority(&copy_st_, cudaStreamNonBlocking, hi));
    } else {
        cudaGetLastError();
        BBMH_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
        BBMH_CUDA(cudaStreamCreateWithFlags(&copy_st_, cudaStreamNonBlocking));
    }
    BBMH_CUDA(cudaEventCreateWithFlags(&copied_, cudaEventDisableTiming));
    BBMH_CUDA(cudaMalloc(&d_flags_, 8 * sizeof(uint32_t)));
    BBMH_CUDA(cudaMallocHost(&h_flags_, 8 * sizeof(uint32_t)));
}

GpuLibsvmParser::~GpuLibsvmParser() {
    cudaSetDevice(device_);
    if (copy_st_) cudaStreamSynchronize(copy_st_);
    if (d_next_) cudaFree(d_next_);
    if (copied_) cudaEventDestroy(copied_);
    if (copy_st_) cudaStreamDestroy(copy_st_);
    for (void* p : {(void*)d_text_, (void*)d_seg_, (void*)d_line_end_, (void*)d_colons_before_,
                    (void*)d_line_tok_, (void*)d_row_of_line_, (void*)d_line_label_, (void*)d_ids_,
                    (void*)d_row_end_, (void*)d_labels_, (void*)d_flags_, d_scan_tmp_})
        if (p) cudaFree(p);
    if (h_flags_) cudaFreeHost(h_flags_);
    if (st_) cudaStreamDestroy(st_);
}

GpuParseResult GpuLibsvmParser::run(const char* text, uint64_t len, bool at_eof, uint64_t max_rows,
                                    uint64_t max_ids, uint64_t key, const char* next_text,
                                    uint64_t next_len, uint64_t next_key,
                                    const DeviceIdsOut* dev_out) {
    GpuParseResult r;
    if (len == 0 || len >= (1ull << 32)) return r;
    BBMH_CUDA(cudaSetDevice(device_));
    // 16 bytes of slack: the segment counter reads whole uint4 of full segments only
    if (prefetched(key, len)) {
        // the copy started by prefetch(): swap its buffer in, order after it
        std::swap(d_text_, d_next_);
        std::swap(cap_text_, cap_next_);
        BBMH_CUDA(cudaStreamWaitEvent(st_, copied_, 0));
        pf_len_ = 0;
    } else {
        cancel_prefetch();
        uint64_t cap_text = cap_text_;
        grow_dev(d_text_, cap_text, len + 16);
        cap_text_ = cap_text;
        BBMH_CUDA(cudaMemcpyAsync(d_text_, text, len, cudaMemcpyHostToDevice, st_));
    }
    const uint64_t nchunk = (len + 15) / 16;
    const uint64_t nseg = (nchunk + kTpb - 1) / kTpb;  // CTAs
    uint64_t cap_seg = cap_seg_;
    grow_dev(d_seg_, cap_seg, nseg);
    cap_seg_ = cap_seg;
    BBMH_CUDA(cudaMemsetAsync(d_flags_, 0, 8 * sizeof(uint32_t), st_));
    const int tpb = 128;
    seg_count<<<unsigned(nseg), kTpb, 0, st_>>>(d_text_, len, d_seg_, d_flags_);
    BBMH_CUDA(cudaGetLastError());
    // the next block's copy overlaps this block's kernels
    if (next_len) prefetch(next_text, next_len, next_key);
    size_t tmp = 0;
    BBMH_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, d_seg_, d_seg_, int(nseg), st_));
    if (tmp > scan_tmp_bytes_) {
        if (d_scan_tmp_) BBMH_CUDA(cudaFree(d_scan_tmp_));
        scan_tmp_bytes_ = tmp + tmp / 4 + 256;
        BBMH_CUDA(cudaMalloc(&d_scan_tmp_, scan_tmp_bytes_));
    }
    size_t tb = scan_tmp_bytes_;
    BBMH_CUDA(cub::DeviceScan::InclusiveSum(d_scan_tmp_, tb, d_seg_, d_seg_, int(nseg), st_));
    unsigned long long tot = 0;
    BBMH_CUDA(cudaMemcpyAsync(&h_flags_[0], d_flags_, sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
    BBMH_CUDA(cudaMemcpyAsync(&tot, d_seg_ + nseg - 1, sizeof(tot), cudaMemcpyDeviceToHost, st_));
    BBMH_CUDA(cudaStreamSynchronize(st_));
    trace("parse: counted");
    if (h_flags_[0]) return r;  // bytes outside the fast alphabet
    const uint64_t nl = tot >> 32, ncol = tot & 0xffffffffull;
    const bool open_last = at_eof && text[len - 1] != '\n';
    const uint64_t nlines = nl + (open_last ? 1 : 0);
    if (nlines == 0) return r;
    uint64_t cl = cap_lines_;
    grow_dev(d_line_end_, cl, nlines + 1);
    uint64_t cl2 = cap_lines_;
    grow_dev(d_colons_before_, cl2, nlines + 2);
    uint64_t cl3 = cap_lines_;
    grow_dev(d_line_tok_, cl3, nlines + 1);
    uint64_t cl4 = cap_lines_;
    grow_dev(d_row_of_line_, cl4, nlines + 1);
    uint64_t cl5 = cap_lines_;
    grow_dev(d_line_label_, cl5, nlines + 1);
    uint64_t cl6 = cap_lines_;
    grow_dev(d_row_end_, cl6, nlines + 1);
    uint64_t cl7 = cap_lines_;
    grow_dev(d_labels_, cl7, nlines + 1);
    cap_lines_ = std::min<uint64_t>({cl, cl2, cl3, cl4, cl5, cl6, cl7});
    if (dev_out) {  // straight into the caller's device buffer
        ids_dst_ = dev_out->reserve(dev_out->base + ncol + 1) + dev_out->base;
        BBMH_CUDA(cudaSetDevice(device_));
    } else {
        uint64_t ci = cap_ids_;
        grow_dev(d_ids_, ci, ncol + 1);
        cap_ids_ = ci;
        ids_dst_ = d_ids_;
    }
    BBMH_CUDA(cudaMemsetAsync(d_line_tok_, 0, nlines * sizeof(uint32_t), st_));
    seg_emit<<<unsigned(nseg), kTpb, 0, st_>>>(d_text_, len, nchunk, at_eof ? 1 : 0, d_seg_,
                                               d_line_end_, d_colons_before_, d_line_tok_, ids_dst_,
                                               d_flags_);
    BBMH_CUDA(cudaGetLastError());
    const uint64_t warps_tpb = 256;
    line_check<<<unsigned((nlines * 32 + warps_tpb - 1) / warps_tpb), unsigned(warps_tpb), 0, st_>>>(
        d_text_, uint32_t(nlines), d_line_end_, d_colons_before_, d_line_tok_, ids_dst_,
        d_row_of_line_, d_line_label_, d_flags_);
    BBMH_CUDA(cudaGetLastError());
    tmp = 0;
    BBMH_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, d_row_of_line_, d_row_of_line_,
                                            int(nlines), st_));
    if (tmp > scan_tmp_bytes_) {
        BBMH_CUDA(cudaFree(d_scan_tmp_));
        scan_tmp_bytes_ = tmp + tmp / 4 + 256;
        BBMH_CUDA(cudaMalloc(&d_scan_tmp_, scan_tmp_bytes_));
    }
    tb = scan_tmp_bytes_;
    BBMH_CUDA(cub::DeviceScan::ExclusiveSum(d_scan_tmp_, tb, d_row_of_line_, d_row_of_line_,
                                            int(nlines), st_));
    row_emit<<<unsigned((nlines + tpb - 1) / tpb), tpb, 0, st_>>>(
        uint32_t(nlines), d_row_of_line_, d_colons_before_, d_line_label_, d_row_end_, d_labels_,
        d_flags_, d_line_end_);
    BBMH_CUDA(cudaGetLastError());
    BBMH_CUDA(cudaMemcpyAsync(h_flags_, d_flags_, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
    BBMH_CUDA(cudaStreamSynchronize(st_));
    count_launches(4);  // seg_count, seg_emit, line_check, row_emit (+ CUB scans)
    trace("parse: checked");
    if (h_flags_[0] || h_flags_[2] != nlines || h_flags_[3] != ncol) return r;
    const uint64_t rows = h_flags_[1];
    if (rows <= max_rows && ncol <= max_ids) {
        r.ok = true;
        r.lines = nlines;
        r.rows = rows;
        r.ids = ncol;
        r.bytes = len;
        return r;
    }
    // more than the batch takes: its longest prefix of whole lines that fits
    prefix_cut<<<unsigned((nlines + tpb - 1) / tpb), tpb, 0, st_>>>(
        uint32_t(nlines), d_row_of_line_, d_colons_before_, d_line_end_, max_rows, max_ids, d_flags_);
    BBMH_CUDA(cudaGetLastError());
    count_launches(1);
    BBMH_CUDA(cudaMemcpyAsync(h_flags_ + 4, d_flags_ + 4, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
    BBMH_CUDA(cudaStreamSynchronize(st_));
    if (!h_flags_[4]) {
        r.over_budget = true;
        return r;
    }
    r.ok = true;
    r.lines = h_flags_[4];
    r.rows = h_flags_[5];
    r.ids = h_flags_[6];
    r.bytes = h_flags_[7];
    return r;
}

void GpuLibsvmParser::prefetch(const char* text, uint64_t len, uint64_t key) {
    cancel_prefetch();
    if (len == 0 || len >= (1ull << 32)) return;
    BBMH_CUDA(cudaSetDevice(device_));
    // the copy may only overwrite d_next_ once the parse that last used it as
    // its text is done: every parse synchronises st_ before returning
    uint64_t cap = cap_next_;
    grow_dev(d_next_, cap, len + 16);
    cap_next_ = cap;
    BBMH_CUDA(cudaMemcpyAsync(d_next_, text, len, cudaMemcpyHostToDevice, copy_st_));
    BBMH_CUDA(cudaEventRecord(copied_, copy_st_));
    pf_key_ = key;
    pf_len_ = len;
    pf_waited_ = false;
}

void GpuLibsvmParser::wait_prefetch() {
    if (!pf_len_ || pf_waited_) return;
    BBMH_CUDA(cudaSetDevice(device_));
    BBMH_CUDA(cudaEventSynchronize(copied_));
    pf_waited_ = true;
}

void GpuLibsvmParser::cancel_prefetch() {
    wait_prefetch();
    pf_len_ = 0;
}

void GpuLibsvmParser::fetch(uint32_t* ids_out, uint64_t id_base, std::vector<uint64_t>& row_ptr,
                            std::vector<int8_t>& labels, const GpuParseResult& r) {
    BBMH_CUDA(cudaSetDevice(device_));
    if (r.ids && ids_out)  // (null: the ids stay on the device)
        BBMH_CUDA(cudaMemcpyAsync(ids_out, ids_dst_, r.ids * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                  st_));
    const size_t r0 = row_ptr.size(), l0 = labels.size();
    row_ptr.resize(r0 + r.rows);
    labels.resize(l0 + r.rows);
    if (r.rows) {
        BBMH_CUDA(cudaMemcpyAsync(row_ptr.data() + r0, d_row_end_, r.rows * sizeof(uint64_t),
                                  cudaMemcpyDeviceToHost, st_));
        BBMH_CUDA(cudaMemcpyAsync(labels.data() + l0, d_labels_, r.rows, cudaMemcpyDeviceToHost, st_));
    }
    BBMH_CUDA(cudaStreamSynchronize(st_));
    trace("parse: fetched");
    for (size_t i = r0; i < row_ptr.size(); ++i) row_ptr[i] += id_base;
}

}  // namespace bbmh
