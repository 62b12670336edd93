// engine.hpp -- GPU execution of the sketch over CSR blocks: per-device
// family residency, pooled stream/buffer "slots", the chunked host-buffer
// pipeline (H2D -> kernel -> D2H overlapped across slots and devices).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "core.hpp"
#include "kernels.cuh"

namespace bbmh {

void cuda_check(cudaError_t e, const char* what);
#define BBMH_CUDA(call) ::bbmh::cuda_check((call), #call)

// Per-GPU copy of a family (coefficients in the kernels' layout, tables).
struct DeviceFamily {
    int device = -1;
    uint32_t* d_coef = nullptr;
    uint32_t* d_perm = nullptr;
    std::vector<uint32_t> host_coef;  // the host copy of d_coef (uniform-kernel parameters)
    KernelFamily kf;
    ~DeviceFamily();
};

const DeviceFamily& device_family(const Family& f, int device);

// Registers permutation tables already built in device memory on `device`
// (ownership passes to that device's DeviceFamily).
void adopt_device_perm(Family& f, int device, uint32_t* d_perm);

// Table j of a permutation family (D u32) into host memory, from wherever it
// lives (the host build or the device that built it).
void copy_perm_table(const Family& f, uint32_t j, uint32_t* out);

// Whether 16-bit id transfer moves more ids/s than 4-byte ids when `feeds`
// GPUs stream from this host (engine.cu); the two rates are returned too.
bool delta16_budget_pays(uint64_t feeds, double* raw_ids_s, double* enc_ids_s);
double host_encode_ids_per_s();
// Every n-th chunk of the host-buffer path as 4-byte ids (0: none) for the
// mix that moves the most ids/s from `feeds` GPUs' links, host DRAM and
// host encode rate (option delta_raw_every = -1); the rate goes to ids_s.
uint32_t mixed_raw_every(uint64_t feeds, double* ids_s);

// Devices used by the host-buffer and file pipelines (empty = current device).
std::vector<int> pipeline_devices();
void set_pipeline_devices(const std::vector<int>& ids);

uint64_t chunk_docs_setting();
void set_chunk_docs(uint64_t docs);

struct ScoreModel;

// Host buffers in, host buffers out; synchronous. Validates row_ptr. With a
// score model the rows are also scored on the device (codes may then be null).
void sketch_rows_host(const Family& f, const uint64_t* row_ptr, const uint32_t* indices,
                      uint64_t n, uint32_t b, uint8_t* codes, uint64_t* minima, uint8_t* flags,
                      const ScoreModel* score = nullptr, double* scores = nullptr);

// Device buffers on the current device; asynchronous on `stream`.
void sketch_rows_device(const Family& f, const uint64_t* d_row_ptr, uint64_t index_base,
                        const uint32_t* d_indices, uint64_t n, uint32_t b, uint8_t* d_codes,
                        uint64_t* d_minima, uint8_t* d_flags, cudaStream_t stream);

// ---- reusable chunk executor (also drives the file pipeline) -------------
// A Lane owns one device and NSLOT stream/buffer slots. submit() enqueues
// H2D + kernel + D2H for one CSR chunk into the next slot; when that slot
// was busy its previous chunk is completed first and handed to `done`.
struct ChunkJob {
    uint64_t tag = 0;                 // caller's chunk id
    const uint64_t* row_ptr = nullptr;  // n+1 entries (host)
    uint64_t index_base = 0;          // row_ptr[0] value that maps to indices[0]
    const uint32_t* indices = nullptr;  // host, starting at index_base
    uint64_t n = 0;
    bool pinned_input = false;        // row_ptr/indices already page-locked
    uint8_t* codes_out = nullptr;     // page-locked host destination of the chunk's codes:
                                      // the D2H lands there (no minima chunks)
    bool ids_as_is = false;           // send this chunk's ids as they are (see delta.hpp)
    const uint32_t* d_indices = nullptr;  // the ids already on the lane's device (then
                                          // `indices` is not read); granule slack required
};

struct ChunkResult {
    uint64_t tag = 0;
    uint64_t n = 0;
    const uint8_t* codes = nullptr;    // pinned, n * cb
    const uint64_t* minima = nullptr;  // pinned, n * k (or null)
    const uint8_t* flags = nullptr;    // pinned, n
    const double* scores = nullptr;    // pinned, n (scoring lanes only)
    float kernel_ms = 0;               // device time of the sketch kernel
};

// Linear model over the k*2^b expansion for the fused scoring path
// (learner.cpp:510-521): scores[r] = sum_j w[j*2^b + code_j].
struct ScoreModel {
    const double* w = nullptr;  // host, dim doubles
    uint64_t dim = 0;
};

class Lane {
public:
    static constexpr int kSlots = 3;
    Lane(const Family& f, int device, uint32_t b, bool want_minima,
         const ScoreModel* score = nullptr);
    ~Lane();
    Lane(const Lane&) = delete;
    Lane& operator=(const Lane&) = delete;

    template <typename Done>
    void submit(const ChunkJob& job, Done&& done) {
        Slot& s = *slots_[next_ % kSlots];
        if (s.busy) done(finish(s));
        enqueue(s, job);
        ++next_;
    }
    template <typename Done>
    void drain(Done&& done) {
        for (int i = 0; i < kSlots; ++i) {
            Slot& s = *slots_[(next_ + i) % kSlots];
            if (s.busy) done(finish(s));
        }
    }
    int device() const { return device_; }
    // Record kernel start/stop events per chunk (ChunkResult::kernel_ms).
    void set_timed(bool on) { timed_ = on; }
    // Allow the 2-byte id transfer (delta.hpp) where it pays: for callers
    // whose chunks are bound by the H2D copy (host CSR batches), not by what
    // produces them (the file pipelines' parsers share the host cores).
    void set_delta16(bool on) { delta16_ = on; }

public:
    struct Slot {
        int device = -1;
        cudaStream_t st = nullptr;
        cudaEvent_t ev0 = nullptr, ev1 = nullptr, done = nullptr;
        uint64_t* d_rp = nullptr;
        uint32_t* d_idx = nullptr;
        uint8_t* d_codes = nullptr;
        uint64_t* d_min = nullptr;
        uint8_t* d_flags = nullptr;
        int* d_err = nullptr;
        uint64_t* h_rp = nullptr;
        uint32_t* h_idx = nullptr;
        uint8_t* h_codes = nullptr;
        uint64_t* h_min = nullptr;
        uint8_t* h_flags = nullptr;
        int* h_err = nullptr;
        double* d_scores = nullptr;
        double* h_scores = nullptr;
        unsigned long long* d_bad = nullptr;
        unsigned long long* h_bad = nullptr;
        uint64_t cap_scores = 0;
        uint64_t cap_rows = 0, cap_idx = 0, cap_idx_pinned = 0, cap_codes = 0, cap_min = 0;
        // packed transfer block: one H2D [row_ptr | ids | err,bad] and one
        // D2H [err,bad | scores | flags | codes] per chunk (see enqueue)
        uint8_t* d_blk = nullptr;
        uint8_t* h_blk = nullptr;
        uint64_t cap_blk = 0;
        bool packed = false;
        size_t off_ids = 0, off_err = 0, off_scores = 0, off_flags = 0, off_codes = 0, blk_end = 0;
        bool busy = false;
        ChunkJob job;
    };

private:
    void reserve(Slot& s, uint64_t rows, uint64_t nidx, bool need_pinned_idx);
    void enqueue(Slot& s, const ChunkJob& job);
    void enqueue_packed(Slot& s, const ChunkJob& job, uint64_t nidx);
    ChunkResult finish(Slot& s);

    const Family& f_;
    const DeviceFamily* df_ = nullptr;
    int device_;
    uint32_t b_;
    size_t cb_;
    bool want_minima_;
    double* d_w_ = nullptr;  // device copy of the scoring model (owned by the lane)
    uint64_t wdim_ = 0;
    uint64_t next_ = 0;
    bool timed_ = true;
    bool delta16_ = false;
    Slot* slots_[kSlots] = {};
};

}  // namespace bbmh
