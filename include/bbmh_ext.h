/* bbmh_ext.h -- B200 extensions to the reference ABI (not in the reference's
 * proj/include/bbmh.h). They expose the batched form of the reference's
 * per-document sketch_one (proj/src/sketch.cpp:71-100) that the reference only
 * runs inside its chunk pipeline (proj/src/pipeline.cpp:171-191), plus device
 * selection for the document-sharded multi-GPU file pipeline.
 *
 * CSR layout everywhere: row_ptr has n+1 u64 entries (row r = indices
 * [row_ptr[r], row_ptr[r+1])), indices are u32 feature ids. Outputs follow
 * the reference's SketchRecord (proj/src/sketch.hpp:33-41):
 *   codes_out  n * ceil(k*b/8) bytes, LE bitstream per row (sketch.cpp:64-69)
 *   minima_out n * k u64 (nullable), flags_out n bytes (nullable, bit0 = empty)
 */
#ifndef BBMH_EXT_H
#define BBMH_EXT_H

#include "bbmh.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Host buffers (pinned or pageable). Rows are streamed to the selected
 * GPU(s) in chunks over double-buffered pinned staging: H2D copy, sketch
 * kernel and D2H copy of the codes overlap. Synchronous. */
BBMH_API bbmh_status bbmh_ext_sketch_csr(const bbmh_family* family, const uint64_t* row_ptr,
                                         const uint32_t* indices, uint64_t n, uint32_t b,
                                         uint8_t* codes_out, uint64_t* minima_out,
                                         uint8_t* flags_out);

/* Device buffers on the CURRENT device; enqueued on `stream` (a
 * cudaStream_t, NULL = legacy default stream) and returns without
 * synchronising. row_ptr values are offsets into d_indices after subtracting
 * `index_base` (lets a caller pass a slice of a larger row_ptr).
 * Ids are fetched with bulk copies in whole 16-byte granules: the granule
 * holding a row's first id is read from its start and the granule holding its
 * last id to its end -- up to 12 bytes before d_indices + row_ptr[0] -
 * index_base and up to 12 bytes past the last id, never across a page; the
 * values there are never used. An allocation that starts 16-byte aligned
 * (cudaMalloc's always do) and whose size is a multiple of 16 bytes (or has
 * 12 bytes of slack) keeps compute-sanitizer memcheck quiet. The host entry
 * points handle this themselves. */
BBMH_API bbmh_status bbmh_ext_sketch_csr_device(const bbmh_family* family,
                                                const uint64_t* d_row_ptr, uint64_t index_base,
                                                const uint32_t* d_indices, uint64_t n,
                                                uint32_t b, uint8_t* d_codes,
                                                uint64_t* d_minima, uint8_t* d_flags,
                                                void* stream);

/* Fused test-time scoring (the reference's prediction on a sketch, run
 * without materialising the sketch or its expansion): each row is sketched
 * and scored on the GPU against a linear model over the k*2^b expansion,
 *   scores_out[r] = sum_{j ascending} weights[j*2^b + code_j]
 * in double precision and in the reference's summation order
 * (predict_score, proj/src/learner.cpp:510-521); rows with no ids score 0
 * (learner.cpp:528). An expanded index >= weights_dim fails with
 * BBMH_E_DIMENSION_EXCEEDED "feature <idx> >= dim <dim>" (learner.cpp:515). */
BBMH_API bbmh_status bbmh_ext_sketch_score_csr(const bbmh_family* family, const uint64_t* row_ptr,
                                               const uint32_t* indices, uint64_t n, uint32_t b,
                                               const double* weights, uint64_t weights_dim,
                                               double* scores_out);

/* File form: corpus (LibSVM text or BBCV) + BBLM model -> "%d\t%.9g\n" per
 * row and the accuracy, byte-identical to bbmh_sketch_file followed by
 * bbmh_predict on the resulting sketch (proj/src/capi.cpp:307-317).
 * scores_path may be NULL/"" (no table) or "-" (stdout). */
BBMH_API bbmh_status bbmh_ext_predict_corpus(const bbmh_family* family, uint32_t b,
                                             const char* model_path, const char* corpus_path,
                                             const char* scores_path, uint32_t workers,
                                             double* accuracy_out,
                                             bbmh_pipeline_stats* stats_out /* nullable */);

/* All-pairs b-bit matching counts (near-duplicate detection): the count of
 * estimate_bbit (proj/src/estimator.cpp:53-58) for every pair of two sketch
 * sets, on the GPU. codes_a: na rows, codes_b: nb rows, ceil(k*b/8) bytes
 * each (LE bitstream); counts_out[i*nb + j] = #{t < k : code_t(A_i) ==
 * code_t(B_j)}. Feed counts/k to the Theorem-1 correction
 * (bbmh_correction_terms) for resemblance estimates. */
BBMH_API bbmh_status bbmh_ext_match_counts(const uint8_t* codes_a, uint64_t na,
                                           const uint8_t* codes_b, uint64_t nb, uint32_t k,
                                           uint32_t b, uint32_t* counts_out);
/* Same on device buffers, enqueued on `stream` (cudaStream_t). */
BBMH_API bbmh_status bbmh_ext_match_counts_device(const uint8_t* d_codes_a, uint64_t na,
                                                  const uint8_t* d_codes_b, uint64_t nb,
                                                  uint32_t k, uint32_t b, uint32_t* d_counts,
                                                  void* stream);

/* Device list used by bbmh_ext_sketch_csr and bbmh_sketch_file (default:
 * the current device only). Chunks are assigned dynamically; output order
 * and bytes do not depend on the device count. */
BBMH_API bbmh_status bbmh_ext_set_devices(const int32_t* ids, uint32_t count);
BBMH_API bbmh_status bbmh_ext_get_devices(int32_t* ids_out, uint32_t capacity,
                                          uint32_t* count_out);

/* Upload the family's coefficients / permutation tables to `device` now
 * instead of on first use. */
BBMH_API bbmh_status bbmh_ext_family_prepare(const bbmh_family* family, int32_t device);

/* Pinned host memory for callers that want zero-copy-staged H2D. */
BBMH_API bbmh_status bbmh_ext_host_alloc(size_t bytes, void** out);
BBMH_API void bbmh_ext_host_free(void* p);

/* Number of CUDA kernels this library has launched in this process
 * (monotonic; used by benchmarks to report gpu_launches). */
BBMH_API uint64_t bbmh_ext_kernel_launches(void);

/* Bytes the host-buffer sketch paths (bbmh_ext_sketch_csr, bbmh_sketch_set
 * batches, the file pipelines' chunks) have moved host->device and
 * device->host in this process (monotonic). Ids may travel 2 bytes each
 * (16-bit row differences, rebuilt on the device) where the copy would bound
 * the call; these counts are the bytes actually moved. */
BBMH_API void bbmh_ext_transfer_bytes(uint64_t* h2d_out, uint64_t* d2h_out);

/* Chunk size (documents) used by the host-buffer and file pipelines;
 * 0 restores the default. */
BBMH_API bbmh_status bbmh_ext_set_chunk_docs(uint64_t docs);

/* Tuning and test switches (the reference has none and reads no environment,
 * SPEC.md:502). Every switch defaults to what the product runs; names and
 * meanings are listed in csrc/options.hpp, in order by bbmh_ext_option_name
 * (returns "" past the end). For developer A/B runs BBMH_OPT_<NAME> in the
 * environment sets a start value, read once. Unknown names fail with
 * BBMH_E_INVALID_ARGUMENT. */
BBMH_API bbmh_status bbmh_ext_set_option(const char* name, int64_t value);
BBMH_API bbmh_status bbmh_ext_get_option(const char* name, int64_t* value_out);
BBMH_API const char* bbmh_ext_option_name(uint32_t i);

/* The host-bandwidth budget that picks the id transfer of the host-buffer
 * paths when `feeds` GPUs stream ids from this host at once (lanes x the
 * "host_sharers" option): ids/s with 4-byte ids (link and DRAM bound) and
 * with 16-bit differences (link and measured host-encode bound), and whether
 * the encoded form is used. Measures the host on first use (~0.3 s). */
BBMH_API bbmh_status bbmh_ext_host_budget(uint32_t feeds, double* raw_ids_per_s,
                                          double* encoded_ids_per_s, int32_t* encoded_pays);

/* The mixed transfer the host-buffer path uses by default (option
 * "delta_raw_every" = -1): every raw_every-th chunk crosses as 4-byte ids and
 * the rest as 16-bit differences, so the link carries the ids the host cannot
 * encode in time. raw_every is 3..8 (near ties go to more raw chunks), or 0
 * when the encoded form beats every mix by 2%. ids_per_s: the budget's rate
 * for that mix, min(link, host DRAM, host encode). */
BBMH_API bbmh_status bbmh_ext_host_mix(uint32_t feeds, uint32_t* raw_every, double* ids_per_s);

/* The two host rates the budget rests on, measured once per process: host
 * DRAM copy bandwidth (read + write bytes/s, all cores) and the 16-bit
 * encoder's ids/s on all cores. */
BBMH_API bbmh_status bbmh_ext_host_rates(double* dram_bytes_per_s, double* encode_ids_per_s);

/* Stage breakdown of the calling thread's last bbmh_sketch_file /
 * bbmh_ext_predict_corpus call. Seconds are summed over lanes (one lane per
 * GPU) except wall_seconds. */
typedef struct bbmh_ext_pipeline_profile {
    double wall_seconds;
    double io_seconds;     /* pread of the input, summed over waiting threads */
    double parse_seconds;  /* LibSVM parse calls (GPU parser incl. its text H2D, or CPU rounds) */
    double load_seconds;   /* loader threads busy producing batches (read + parse) */
    double hash_seconds;   /* sketch kernels, device time */
    double write_seconds;  /* in-order writer */
    uint64_t input_bytes;
    uint64_t records;
    uint64_t lanes;        /* GPUs (lanes) that sketched */
    uint64_t ranges;       /* line-aligned text ranges (range-sharded loaders); 0 = one reader */
} bbmh_ext_pipeline_profile;
BBMH_API bbmh_status bbmh_ext_last_pipeline_profile(bbmh_ext_pipeline_profile* out);

/* Epoch replay (the consumer of sketch files; the reference's RowSource,
 * learner.cpp:215-312): a corpus streamed as batches of device CSR rows, once
 * per epoch. For a BBMH sketch every record becomes the row of its k one-hot
 * features in the 2^b*k expansion, ones[j] = j*2^b + code_j ascending, and
 * a flagged empty record an empty row (SketchRowSource, learner.cpp:271-297;
 * expansion.cpp:17-27). Record blocks are read ahead in page-locked memory
 * and expanded on `device`. A LibSVM or BBCV corpus gives its rows as the
 * sketch loader parses them (binary values). Header errors are
 * SketchReader's (sketch.cpp:143-163); a truncated sketch returns its
 * complete records, then fails with BBMH_E_IO "short read". */
typedef struct bbmh_ext_replay bbmh_ext_replay;
typedef struct bbmh_ext_replay_info {
    int32_t sketch;        /* 1: BBMH sketch, 0: LibSVM / BBCV corpus */
    uint32_t scheme, k, b; /* sketch header (0 for a corpus) */
    uint64_t dim, seed, count;
    uint64_t expanded_dim; /* 2^b * k (expanded_dim, expansion.cpp:9-15) */
} bbmh_ext_replay_info;
typedef struct bbmh_ext_replay_stats {
    uint64_t epochs, rows, nnz;
    double io_seconds, parse_seconds, expand_seconds;
} bbmh_ext_replay_stats;
BBMH_API bbmh_status bbmh_ext_replay_open(const char* path, int32_t device, uint64_t max_rows,
                                          uint32_t threads, bbmh_ext_replay** out,
                                          bbmh_ext_replay_info* info_out /* nullable */);
/* Next batch: *rows_out rows (0 at the end of the epoch); d_row_ptr (rows+1,
 * from 0) and d_indices on the device, labels and row_ptr_host on the host,
 * all owned by the replay and valid until its next call. Outputs nullable. */
BBMH_API bbmh_status bbmh_ext_replay_next(bbmh_ext_replay* replay, uint64_t* rows_out,
                                          const uint64_t** d_row_ptr, const uint32_t** d_indices,
                                          const int8_t** labels, const uint64_t** row_ptr_host);
BBMH_API bbmh_status bbmh_ext_replay_reset(bbmh_ext_replay* replay);
BBMH_API bbmh_status bbmh_ext_replay_get_stats(const bbmh_ext_replay* replay, bbmh_ext_replay_stats* out);
BBMH_API void bbmh_ext_replay_close(bbmh_ext_replay* replay);

/* Monotonic per-process counters of which routes ran: "kernel_launches",
 * "h2d_bytes", "d2h_bytes", "peer_copy_bytes", "zero_copy_calls",
 * "delta16_chunks", "raw_chunks", "range_shards", "device_id_batches",
 * "uniform_launches". */
BBMH_API bbmh_status bbmh_ext_counter(const char* name, uint64_t* value_out);

/* Permutation table j (dim u32 values, the reference's perm_[j*D .. j*D+D),
 * hash_family.hpp:88-89) copied into table_out, wherever the family keeps it
 * (host build or the GPU that built it). */
BBMH_API bbmh_status bbmh_ext_family_perm_table(const bbmh_family* family, uint32_t j,
                                                uint32_t* table_out);

#ifdef __cplusplus
}
#endif

#endif /* BBMH_EXT_H */
