// pipeline.hpp -- file-level entry points (bbmh_sketch_file / bbmh_expand_file).
#pragma once

#include <cstdint>
#include <string>

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

// sketch_file (pipeline.cpp:215-226): corpus -> BBMH sketch (+ .min64).
PipelineStats sketch_file(const Family& f, const std::string& input_path,
                          const std::string& output_path, uint8_t b, uint64_t chunk_size,
                          uint32_t workers, bool emit_minima);

// expand_stream (expansion.cpp:47-90): BBMH sketch -> BBCV rows or LibSVM text.
uint64_t expand_file(const std::string& sketch_path, const std::string& out_path, bool binary);

}  // namespace bbmh
