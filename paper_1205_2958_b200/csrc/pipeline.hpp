// pipeline.hpp -- file-level entry points (bbmh_sketch_file / bbmh_expand_file).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "core.hpp"

namespace bbmh {

// Same meanings as the reference's PipelineStats (pipeline.hpp:13-20), with
// compute_seconds = summed device time of the sketch kernels.
struct PipelineStats {
    uint64_t records = 0;
    uint64_t chunks = 0;
    double read_seconds = 0;
    double compute_seconds = 0;
    double write_seconds = 0;
    double wall_seconds = 0;
};

// Stage breakdown of the calling thread's last file pipeline
// (bbmh_ext_last_pipeline_profile). Seconds are summed over lanes except
// wall_seconds; per-lane figures divide by `lanes`.
struct PipelineProfile {
    double wall_seconds = 0;
    double io_seconds = 0;      // pread of the text / BBCV bytes (threads waiting on it)
    double parse_seconds = 0;   // LibSVM parse calls (GPU parser incl. its H2D, or CPU rounds)
    double load_seconds = 0;    // loader threads busy producing batches (read + parse)
    double hash_seconds = 0;    // sketch kernels, device time
    double write_seconds = 0;   // in-order writer
    uint64_t input_bytes = 0;
    uint64_t records = 0;
    uint64_t lanes = 0;
    uint64_t ranges = 0;        // text ranges (range-sharded loaders), 0 = one shared reader
};
PipelineProfile last_pipeline_profile();

// sketch_file (pipeline.cpp:215-226): corpus -> BBMH sketch (+ .min64).
PipelineStats sketch_file(const Family& f, const std::string& input_path,
                          const std::string& output_path, uint8_t b, uint64_t chunk_size,
                          uint32_t workers, bool emit_minima);

// Fused test-time path: corpus -> GPU sketch -> GPU score
// against a BBLM model -> "%d\t%.9g\n" rows, exactly what sketch_file followed
// by bbmh_predict on the sketch produces (capi.cpp:307-317, learner.cpp:524-536).
PipelineStats predict_file(const Family& f, uint8_t b, const std::string& model_path,
                           const std::string& corpus_path, const std::string& scores_path,
                           uint32_t workers, double* accuracy);

// load_model (learner.cpp:588-612) -> decision weights (w_avg when averaged).
std::vector<double> load_decision_weights(const std::string& path);

// bbmh_predict (capi.cpp:307-317) on the GPU: BBMH / BBCV / LibSVM rows scored
// against a BBLM model; writes the "%d\t%.9g" table (path "" = none, "-" =
// stdout) and returns the accuracy.
double predict_data(const std::string& model_path, const char* data_path,
                    const std::string& scores_path, unsigned threads);

// vw_project_file (vw.cpp:61-77): corpus -> signed random-bin LibSVM rows (GPU).
uint64_t vw_project_file(const std::string& corpus_path, const std::string& out_path,
                         uint32_t bins, uint64_t seed);

// expand_stream (expansion.cpp:47-90): BBMH sketch -> BBCV rows or LibSVM text.
uint64_t expand_file(const std::string& sketch_path, const std::string& out_path, bool binary);

}  // namespace bbmh
