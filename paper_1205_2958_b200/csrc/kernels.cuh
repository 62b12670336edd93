// kernels.cuh -- device-side description of a hash family and the sketch
// kernel launcher (implementation in kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bbmh {

// Everything a sketch kernel needs, passed by value (lives in the kernel
// parameter bank, i.e. constant memory). Derived on the host from Family.
struct KernelFamily {
    int32_t scheme = 1;      // Scheme tag
    uint32_t k = 0;
    uint64_t dim = 0;
    uint32_t shift2u = 0;    // 2U: right shift applied to the minimum (hash_family.hpp:48-51)
    uint32_t dim_mask = 0;   // 4U: dim - 1 when dim is a power of two
    uint32_t dim_pow2 = 1;
    uint32_t dim32 = 0;      // 4U: dim (< 2^31) for the magic-division branch
    uint32_t neg_dim32 = 0;  // 2^32 - dim32 (h - q*D computed as h + q*neg_dim32)
    uint32_t magic = 0;      // 4U: h % dim = h - dim * (umulhi(h, magic) >> magic_shift)
    uint32_t magic_shift = 0;
    uint32_t p = 0;          // 4U modulus
    uint64_t barrett = 0;    // 4U-mod: floor((2^64 - 1) / p)
    const uint32_t* coef = nullptr;  // 2U: k*{a1,a2}; 4U-bit: k*{a3,2a2,2a1,2a0}; 4U-mod: k*{a3,a2,a1,a0}
    const uint32_t* perm = nullptr;  // permutation tables, k*dim
    const uint32_t* host2u = nullptr;  // 2U: the family's host k*{a1,a2} (uniform kernel parameters)
    const uint32_t* host4u = nullptr;  // 4U-bit: the host copy of coef (uniform4 kernel parameters)
    // set per launch: the persistent sketch kernel returns at once when the
    // batch averages >= yield_nnz ids per document (the uniform kernel,
    // launched beside it, takes such batches; see launch_sketch)
    uint32_t yield_nnz = 0;
};

struct LaunchShape {
    int J = 4;        // hash functions per thread (register-blocked)
    int tpb = 128;    // threads per CTA
    uint32_t jtile = 512;  // hash functions per CTA (tpb*J), multiple of 8
    uint32_t jtiles = 1;   // CTAs per document
};

// Block shape for k hash functions over n documents on a GPU with `sms` SMs
// (n = 0: throughput shape for an unbounded batch).
LaunchShape choose_shape(uint32_t k, int scheme, uint64_t n = 0, int sms = 148);

// Sketch rows [0, n) of a CSR block resident on the current device.
// row_ptr values are offsets into `indices` after subtracting index_base.
// err (device int) receives bit 1 for a permutation id >= dim and bit 2
// for a decreasing row_ptr.
// avg_nnz: ids per document of the batch when the caller knows it (host
// row_ptr), < 0 when not (device row_ptr): then a 2U batch the uniform
// kernel may take launches both 2U kernels and the batch's own row_ptr
// decides on the device which one works.
void launch_sketch(const KernelFamily& F, const uint64_t* row_ptr, uint64_t index_base,
                   const uint32_t* indices, uint64_t n, uint32_t b, uint8_t* codes,
                   uint64_t* minima, uint8_t* flags, int* err, cudaStream_t stream,
                   double avg_nnz = -1.0);

// Permutation mode with tables too large for L2: table-outer passes (perm.cu).
bool perm_tablewise_applies(const KernelFamily& F, uint64_t n);
// false: no scratch could be allocated (the caller runs the document-outer kernel)
bool launch_perm_tablewise(const KernelFamily& F, const uint64_t* row_ptr, uint64_t index_base,
                           const uint32_t* indices, uint64_t n, uint32_t b, uint8_t* codes,
                           uint64_t* minima, uint8_t* flags, int* err, cudaStream_t stream);

// Fused scoring of freshly sketched rows against a linear model over the
// k*2^b expansion (score.cu). `bad` receives min(row << 24 | j) of the first
// index >= wdim (initialise to ~0).
void launch_score(const uint8_t* codes, const uint8_t* flags, uint64_t n, uint32_t k, uint32_t b,
                  const double* w, uint64_t wdim, double* scores, unsigned long long* bad,
                  cudaStream_t stream);

// The coefficient-uniform 2U kernel (uniform.cu) for 16 < k <= 544 over
// >= 2,048 documents. uniform_min_nnz: the average row length from which it
// beats the persistent kernel for this batch (0: it does not apply).
// launch_uniform_2u with min_nnz > 0 returns on the device when the batch
// averages fewer ids per document.
uint32_t uniform_min_nnz(const KernelFamily& F, uint64_t n);
void launch_uniform_2u(const KernelFamily& F, const uint64_t* row_ptr, uint64_t index_base,
                       const uint32_t* indices, uint64_t n, uint32_t b, uint8_t* codes,
                       uint64_t* minima, uint8_t* flags, int* err, cudaStream_t stream,
                       uint32_t min_nnz);

// The coefficient-uniform 4U-bit kernel (uniform4.cu) for 16 < k <= 1024
// over >= 2,048 documents.
bool uniform4_applies(const KernelFamily& F, uint64_t n);
void launch_uniform_4u(const KernelFamily& F, const uint64_t* row_ptr, uint64_t index_base,
                       const uint32_t* indices, uint64_t n, uint32_t b, uint8_t* codes,
                       uint64_t* minima, uint8_t* flags, int* err, cudaStream_t stream);

// SM count of the current device (cached) and a zeroed {ticket, exit}
// counter pair for one launch (nullptr: none could be allocated).
int sm_count();
unsigned long long* ticket_slot(int dev);
// `pairs` consecutive zeroed pairs (2 x pairs counters); the launch leaves them zeroed
unsigned long long* ticket_block(int dev, int pairs);

uint64_t kernel_launch_count();
void count_launches(uint64_t n);

// Bytes the host-buffer sketch paths move between host and device (copies,
// and the zero-copy path's reads and writes of mapped host memory).
void count_transfer(uint64_t h2d, uint64_t d2h);
void transfer_counts(uint64_t& h2d, uint64_t& d2h);

// Path counters (bbmh_ext_counter): which of the library's routes ran.
enum class Counter : int {
    PeerCopyBytes,   // permutation tables replicated with cudaMemcpyPeer
    ZeroCopyCalls,   // host calls served by the zero-copy small-batch path
    Delta16Chunks,   // host chunks whose ids crossed as 16-bit differences
    RawChunks,       // host chunks whose ids crossed as 4-byte ids (or were device-resident)
    RangeShards,     // LibSVM text ranges sketched by range-sharded lanes
    DeviceIdBatches, // loader batches whose ids never left the parsing GPU
    UniformLaunches, // 2U launches of the coefficient-uniform kernel (uniform.cu)
    kCount
};
void count(Counter c, uint64_t n = 1);
inline void count_peer_copy(uint64_t bytes) { count(Counter::PeerCopyBytes, bytes); }
// by name: "kernel_launches", "h2d_bytes", "d2h_bytes", "peer_copy_bytes",
// "zero_copy_calls", "delta16_chunks", "raw_chunks", "range_shards",
// "device_id_batches", "uniform_launches"; false if unknown
bool counter_value(const char* name, uint64_t* out);

}  // namespace bbmh
