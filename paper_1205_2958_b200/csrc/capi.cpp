// capi.cpp -- the drop-in C ABI (include/bbmh.h, include/bbmh_ext.h).
//
// Mirrors the reference's exception->status shim (capi.cpp:21-59): every
// entry point clears a thread-local detail string, runs inside `guarded`, and
// maps bbmh::Error codes to the same bbmh_status values. No exception crosses
// the ABI. Validation order and messages follow the reference entry points
// cited per function (reference file:line, relative to /root/reference/proj).
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "../../include/bbmh.h"
#include "../../include/bbmh_ext.h"
#include "core.hpp"
#include "engine.hpp"
#include "hostpool.hpp"
#include "estimate.hpp"
#include "options.hpp"
#include "replay.hpp"
#include "pipeline.hpp"

using namespace bbmh;

struct bbmh_family {
    std::unique_ptr<Family> impl;
};

struct bbmh_ext_replay {
    std::unique_ptr<Replay> impl;
};

namespace {

thread_local std::string t_last_error;

bbmh_status status_of(Errc code) {  // capi.cpp:23-41
    switch (code) {
        case Errc::InvalidArgument: return BBMH_E_INVALID_ARGUMENT;
        case Errc::UnsupportedUniverse: return BBMH_E_UNSUPPORTED_UNIVERSE;
        case Errc::PermutationTooLarge: return BBMH_E_PERMUTATION_TOO_LARGE;
        case Errc::HeaderMismatch: return BBMH_E_HEADER_MISMATCH;
        case Errc::MissingMinima: return BBMH_E_MISSING_MINIMA;
        case Errc::DegenerateProfile: return BBMH_E_DEGENERATE_PROFILE;
        case Errc::EmptySketch: return BBMH_E_EMPTY_SKETCH;
        case Errc::DimensionExceeded: return BBMH_E_DIMENSION_EXCEEDED;
        case Errc::NonBinaryLabel: return BBMH_E_NON_BINARY_LABEL;
        case Errc::MalformedLine:
        case Errc::NonBinaryValue:
        case Errc::NonAscendingIndex: return BBMH_E_PARSE;
        case Errc::InfeasibleProfile: return BBMH_E_INFEASIBLE_PROFILE;
        case Errc::Io: return BBMH_E_IO;
        case Errc::Cuda: return BBMH_E_INTERNAL;
    }
    return BBMH_E_INTERNAL;
}

template <typename Fn>
bbmh_status guarded(Fn&& fn) {  // capi.cpp:43-59
    try {
        t_last_error.clear();
        fn();
        return BBMH_OK;
    } catch (const Error& e) {
        t_last_error = e.what();
        return status_of(e.code());
    } catch (const std::exception& e) {
        t_last_error = e.what();
        return BBMH_E_INTERNAL;
    } catch (...) {
        t_last_error = "unknown error";
        return BBMH_E_INTERNAL;
    }
}

Scheme scheme_of(int32_t tag) {  // capi.cpp:97-101
    if (tag < BBMH_SCHEME_PERMUTATION || tag > BBMH_SCHEME_4U_BIT)
        fail(Errc::InvalidArgument, "unknown scheme tag " + std::to_string(tag));
    return Scheme(uint8_t(tag));
}

const char* require(const char* p, const char* what) {  // capi.cpp:103-106
    if (!p) fail(Errc::InvalidArgument, std::string(what) + " must not be NULL");
    return p;
}

uint32_t narrow_b(uint32_t b) {  // capi.cpp:163 narrows b to uint8_t; sketch.cpp:73 checks it
    const uint32_t b8 = uint8_t(b);
    if (b8 < 1 || b8 > 32) fail(Errc::InvalidArgument, "b must be in 1..32");
    return b8;
}

bbmh_status not_provided(const char* name) {
    return guarded([&] {
        fail(Errc::Cuda, std::string(name) + ": not provided by the B200 preprocessing library");
    });
}

}  // namespace

extern "C" {

uint32_t bbmh_version(void) { return 10000; }  // capi.cpp:109 (1.0.0)

const char* bbmh_strerror(bbmh_status status) {  // capi.cpp:111-128
    switch (status) {
        case BBMH_OK: return "ok";
        case BBMH_E_INVALID_ARGUMENT: return "invalid argument";
        case BBMH_E_UNSUPPORTED_UNIVERSE: return "unsupported universe";
        case BBMH_E_PERMUTATION_TOO_LARGE: return "permutation tables exceed the memory cap";
        case BBMH_E_HEADER_MISMATCH: return "sketch header mismatch";
        case BBMH_E_MISSING_MINIMA: return "full minima not available";
        case BBMH_E_DEGENERATE_PROFILE: return "degenerate pair profile";
        case BBMH_E_EMPTY_SKETCH: return "flagged empty-set sketch";
        case BBMH_E_DIMENSION_EXCEEDED: return "dimension exceeded";
        case BBMH_E_NON_BINARY_LABEL: return "label is not +-1";
        case BBMH_E_PARSE: return "parse error";
        case BBMH_E_INFEASIBLE_PROFILE: return "infeasible pair profile";
        case BBMH_E_IO: return "i/o error";
        default: return "internal error";
    }
}

const char* bbmh_last_error(void) { return t_last_error.c_str(); }

// capi.cpp:132-140 -> hash_family.cpp:53-119
bbmh_status bbmh_family_create(int32_t scheme, uint64_t dim, uint32_t k, uint64_t seed,
                               uint64_t prime, uint64_t perm_cap_bytes, bbmh_family** out) {
    return guarded([&] {
        if (!out) fail(Errc::InvalidArgument, "out must not be NULL");
        const Scheme s = scheme_of(scheme);
        auto fam = build_family(s, dim, k, seed, prime ? prime : kMersenne31,
                                perm_cap_bytes ? perm_cap_bytes : kDefaultPermCapBytes);
        *out = new bbmh_family{std::move(fam)};
    });
}

void bbmh_family_destroy(bbmh_family* family) { delete family; }

// capi.cpp:142-151
bbmh_status bbmh_family_map(const bbmh_family* family, uint32_t j, uint32_t t, uint32_t* out) {
    return guarded([&] {
        if (!family || !out) fail(Errc::InvalidArgument, "family and out must not be NULL");
        if (j >= family->impl->k) fail(Errc::InvalidArgument, "j out of range");
        if (uint64_t(t) >= family->impl->dim) fail(Errc::InvalidArgument, "t out of range");
        *out = family->impl->map(j, t);
    });
}

uint64_t bbmh_mod_mersenne31(uint64_t v) { return mod_mersenne31(v); }

// capi.cpp:155-169 -> sketch.cpp:71-100, computed by the CUDA kernel
bbmh_status bbmh_sketch_set(const bbmh_family* family, const uint32_t* indices, size_t count,
                            uint32_t b, uint64_t* minima_out, uint8_t* codes_out,
                            int32_t* empty_out) {
    return guarded([&] {
        if (!family || !codes_out) fail(Errc::InvalidArgument, "family and codes_out required");
        if (count > 0 && !indices) fail(Errc::InvalidArgument, "indices must not be NULL");
        const uint32_t b8 = narrow_b(b);
        const uint64_t row_ptr[2] = {0, uint64_t(count)};
        uint8_t flag = 0;
        static const uint32_t kNone = 0;
        sketch_rows_host(*family->impl, row_ptr, count ? indices : &kNone, 1, b8, codes_out,
                         minima_out, &flag);
        if (empty_out) *empty_out = flag & 1;
    });
}

// capi.cpp:171-185 -> pipeline.cpp:215-226, GPU streaming pipeline
bbmh_status bbmh_sketch_file(const bbmh_family* family, const char* input_path,
                             const char* output_path, uint32_t b, uint64_t chunk_size,
                             uint32_t workers, int32_t emit_minima,
                             bbmh_pipeline_stats* stats_out) {
    return guarded([&] {
        if (!family) fail(Errc::InvalidArgument, "family must not be NULL");
        // the reference evaluates require(output_path) before require(input_path)
        const char* out = require(output_path, "output_path");
        const char* in = require(input_path, "input_path");
        PipelineStats st = sketch_file(*family->impl, in, out, uint8_t(b), chunk_size, workers,
                                       emit_minima != 0);
        if (stats_out)
            *stats_out = {st.records,         st.chunks,        st.read_seconds,
                          st.compute_seconds, st.write_seconds, st.wall_seconds};
    });
}

// capi.cpp:268-275 -> expansion.cpp:47-90
bbmh_status bbmh_expand_file(const char* sketch_path, const char* out_path, int32_t row_format) {
    return guarded([&] {
        if (row_format != BBMH_ROWS_LIBSVM && row_format != BBMH_ROWS_BINARY)
            fail(Errc::InvalidArgument, "unknown row format");
        const char* out = require(out_path, "out_path");
        const char* in = require(sketch_path, "sketch_path");
        expand_file(in, out, row_format == BBMH_ROWS_BINARY);
    });
}

// ---- extensions (bbmh_ext.h) ----------------------------------------------
bbmh_status bbmh_ext_sketch_csr(const bbmh_family* family, const uint64_t* row_ptr,
                                const uint32_t* indices, uint64_t n, uint32_t b,
                                uint8_t* codes_out, uint64_t* minima_out, uint8_t* flags_out) {
    return guarded([&] {
        if (!family || !codes_out) fail(Errc::InvalidArgument, "family and codes_out required");
        if (n > 0 && !row_ptr) fail(Errc::InvalidArgument, "row_ptr must not be NULL");
        const uint32_t b8 = narrow_b(b);
        if (n == 0) return;
        if (row_ptr[n] > row_ptr[0] && !indices)
            fail(Errc::InvalidArgument, "indices must not be NULL");
        static const uint32_t kNone = 0;
        sketch_rows_host(*family->impl, row_ptr, indices ? indices : &kNone, n, b8, codes_out,
                         minima_out, flags_out);
    });
}

bbmh_status bbmh_ext_sketch_csr_device(const bbmh_family* family, const uint64_t* d_row_ptr,
                                       uint64_t index_base, const uint32_t* d_indices,
                                       uint64_t n, uint32_t b, uint8_t* d_codes,
                                       uint64_t* d_minima, uint8_t* d_flags, void* stream) {
    return guarded([&] {
        if (!family || !d_codes || (n && !d_row_ptr))
            fail(Errc::InvalidArgument, "family, row_ptr and codes required");
        const uint32_t b8 = narrow_b(b);
        sketch_rows_device(*family->impl, d_row_ptr, index_base, d_indices, n, b8, d_codes,
                           d_minima, d_flags, static_cast<cudaStream_t>(stream));
    });
}

bbmh_status bbmh_ext_sketch_score_csr(const bbmh_family* family, const uint64_t* row_ptr,
                                      const uint32_t* indices, uint64_t n, uint32_t b,
                                      const double* weights, uint64_t weights_dim,
                                      double* scores_out) {
    return guarded([&] {
        if (!family || !scores_out) fail(Errc::InvalidArgument, "family and scores_out required");
        if (n > 0 && !row_ptr) fail(Errc::InvalidArgument, "row_ptr must not be NULL");
        if (weights_dim > 0 && !weights) fail(Errc::InvalidArgument, "weights must not be NULL");
        const uint32_t b8 = narrow_b(b);
        if (n == 0) return;
        if (row_ptr[n] > row_ptr[0] && !indices)
            fail(Errc::InvalidArgument, "indices must not be NULL");
        static const uint32_t kNone = 0;
        ScoreModel model{weights, weights_dim};
        sketch_rows_host(*family->impl, row_ptr, indices ? indices : &kNone, n, b8, nullptr,
                         nullptr, nullptr, &model, scores_out);
    });
}

bbmh_status bbmh_ext_predict_corpus(const bbmh_family* family, uint32_t b, const char* model_path,
                                    const char* corpus_path, const char* scores_path,
                                    uint32_t workers, double* accuracy_out,
                                    bbmh_pipeline_stats* stats_out) {
    return guarded([&] {
        if (!family) fail(Errc::InvalidArgument, "family must not be NULL");
        const char* model = require(model_path, "model_path");
        const char* data = require(corpus_path, "corpus_path");
        if (workers < 1) fail(Errc::InvalidArgument, "workers must be >= 1");
        PipelineStats st = predict_file(*family->impl, uint8_t(b), model, data,
                                        scores_path ? scores_path : "", workers, accuracy_out);
        if (stats_out)
            *stats_out = {st.records,         st.chunks,        st.read_seconds,
                          st.compute_seconds, st.write_seconds, st.wall_seconds};
    });
}

bbmh_status bbmh_ext_set_devices(const int32_t* ids, uint32_t count) {
    return guarded([&] {
        if (count && !ids) fail(Errc::InvalidArgument, "ids must not be NULL");
        set_pipeline_devices(std::vector<int>(ids, ids + count));
    });
}

bbmh_status bbmh_ext_get_devices(int32_t* ids_out, uint32_t capacity, uint32_t* count_out) {
    return guarded([&] {
        const std::vector<int> d = pipeline_devices();
        if (count_out) *count_out = uint32_t(d.size());
        for (uint32_t i = 0; ids_out && i < capacity && i < d.size(); ++i) ids_out[i] = d[i];
    });
}

bbmh_status bbmh_ext_family_prepare(const bbmh_family* family, int32_t device) {
    return guarded([&] {
        if (!family) fail(Errc::InvalidArgument, "family must not be NULL");
        int count = 0;
        BBMH_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count)
            fail(Errc::InvalidArgument, "device " + std::to_string(device) + " does not exist");
        device_family(*family->impl, device);
    });
}

bbmh_status bbmh_ext_host_alloc(size_t bytes, void** out) {
    return guarded([&] {
        if (!out) fail(Errc::InvalidArgument, "out must not be NULL");
        *out = nullptr;
        BBMH_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
    });
}

void bbmh_ext_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

uint64_t bbmh_ext_kernel_launches(void) { return kernel_launch_count(); }

void bbmh_ext_transfer_bytes(uint64_t* h2d_out, uint64_t* d2h_out) {
    uint64_t a = 0, b = 0;
    transfer_counts(a, b);
    if (h2d_out) *h2d_out = a;
    if (d2h_out) *d2h_out = b;
}

bbmh_status bbmh_ext_set_chunk_docs(uint64_t docs) {
    return guarded([&] { set_chunk_docs(docs); });
}

bbmh_status bbmh_ext_set_option(const char* name, int64_t value) {
    return guarded([&] {
        require(name, "name");
        if (!set_opt(name, value)) fail(Errc::InvalidArgument, std::string("unknown option ") + name);
    });
}

bbmh_status bbmh_ext_get_option(const char* name, int64_t* value_out) {
    return guarded([&] {
        require(name, "name");
        if (!value_out) fail(Errc::InvalidArgument, "value_out must not be NULL");
        if (!get_opt(name, value_out)) fail(Errc::InvalidArgument, std::string("unknown option ") + name);
    });
}

const char* bbmh_ext_option_name(uint32_t i) { return opt_name(int(i)); }

bbmh_status bbmh_ext_replay_open(const char* path, int32_t device, uint64_t max_rows, uint32_t threads,
                                 bbmh_ext_replay** out, bbmh_ext_replay_info* info_out) {
    return guarded([&] {
        if (!out) fail(Errc::InvalidArgument, "out must not be NULL");
        *out = nullptr;
        const std::string p = require(path, "path");
        int count = 0;
        BBMH_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count)
            fail(Errc::InvalidArgument, "device " + std::to_string(device) + " does not exist");
        auto r = std::make_unique<bbmh_ext_replay>();
        r->impl = std::make_unique<Replay>(p, device, max_rows ? max_rows : 32768, threads ? threads : 1);
        if (info_out) {
            const ReplayInfo& i = r->impl->info();
            *info_out = {i.sketch ? 1 : 0, i.scheme, i.k, i.b, i.dim, i.seed, i.count, i.expanded_dim};
        }
        *out = r.release();
    });
}

bbmh_status bbmh_ext_replay_next(bbmh_ext_replay* replay, uint64_t* rows_out, const uint64_t** d_row_ptr,
                                 const uint32_t** d_indices, const int8_t** labels,
                                 const uint64_t** row_ptr_host) {
    return guarded([&] {
        if (!replay) fail(Errc::InvalidArgument, "replay must not be NULL");
        const uint64_t n = replay->impl->next(d_row_ptr, d_indices, labels, row_ptr_host);
        if (rows_out) *rows_out = n;
    });
}

bbmh_status bbmh_ext_replay_reset(bbmh_ext_replay* replay) {
    return guarded([&] {
        if (!replay) fail(Errc::InvalidArgument, "replay must not be NULL");
        replay->impl->reset();
    });
}

bbmh_status bbmh_ext_replay_get_stats(const bbmh_ext_replay* replay, bbmh_ext_replay_stats* out) {
    return guarded([&] {
        if (!replay || !out) fail(Errc::InvalidArgument, "replay and out must not be NULL");
        const ReplayStats s = replay->impl->stats();
        *out = {s.epochs, s.rows, s.nnz, s.io_seconds, s.parse_seconds, s.expand_seconds};
    });
}

void bbmh_ext_replay_close(bbmh_ext_replay* replay) { delete replay; }

bbmh_status bbmh_ext_last_pipeline_profile(bbmh_ext_pipeline_profile* out) {
    return guarded([&] {
        if (!out) fail(Errc::InvalidArgument, "out must not be NULL");
        const PipelineProfile p = last_pipeline_profile();
        *out = {p.wall_seconds,  p.io_seconds,  p.parse_seconds, p.load_seconds, p.hash_seconds,
                p.write_seconds, p.input_bytes, p.records,       p.lanes,        p.ranges};
    });
}

bbmh_status bbmh_ext_host_budget(uint32_t feeds, double* raw_ids_per_s, double* encoded_ids_per_s,
                                 int32_t* encoded_pays) {
    return guarded([&] {
        double raw = 0, enc = 0;
        const bool pays = delta16_budget_pays(feeds, &raw, &enc);
        if (raw_ids_per_s) *raw_ids_per_s = raw;
        if (encoded_ids_per_s) *encoded_ids_per_s = enc;
        if (encoded_pays) *encoded_pays = pays ? 1 : 0;
    });
}

bbmh_status bbmh_ext_host_mix(uint32_t feeds, uint32_t* raw_every, double* ids_per_s) {
    return guarded([&] {
        double rate = 0;
        const uint32_t every = mixed_raw_every(feeds, &rate);
        if (raw_every) *raw_every = every;
        if (ids_per_s) *ids_per_s = rate;
    });
}

bbmh_status bbmh_ext_host_rates(double* dram_bytes_per_s, double* encode_ids_per_s) {
    return guarded([&] {
        if (dram_bytes_per_s) *dram_bytes_per_s = host_dram_bytes_per_s();
        if (encode_ids_per_s) *encode_ids_per_s = host_encode_ids_per_s();
    });
}

bbmh_status bbmh_ext_counter(const char* name, uint64_t* value_out) {
    return guarded([&] {
        require(name, "name");
        if (!value_out) fail(Errc::InvalidArgument, "value_out must not be NULL");
        if (!counter_value(name, value_out)) fail(Errc::InvalidArgument, std::string("unknown counter ") + name);
    });
}

bbmh_status bbmh_ext_family_perm_table(const bbmh_family* family, uint32_t j, uint32_t* table_out) {
    return guarded([&] {
        if (!family) fail(Errc::InvalidArgument, "family must not be NULL");
        if (!table_out) fail(Errc::InvalidArgument, "table_out must not be NULL");
        const Family& f = *family->impl;
        if (f.scheme != Scheme::Permutation) fail(Errc::InvalidArgument, "not a permutation family");
        copy_perm_table(f, j, table_out);
    });
}

// ---- resemblance estimation (capi.cpp:187-240) ---------------
static void put_estimate(const Estimate& e, bbmh_estimate* out) {
    *out = {e.r_hat, e.r_raw, e.p_hat, e.c1b, e.c2b, e.var_theory};
}

bbmh_status bbmh_correction_terms(uint64_t f1, uint64_t f2, uint64_t a, uint64_t dim, uint32_t b,
                                  double* c1b_out, double* c2b_out) {
    return guarded([&] {
        if (!c1b_out || !c2b_out) fail(Errc::InvalidArgument, "outputs must not be NULL");
        const Correction c = correction_terms(Profile{f1, f2, a, dim}, b);
        *c1b_out = c.c1b;
        *c2b_out = c.c2b;
    });
}

bbmh_status bbmh_theoretical_variance(uint64_t f1, uint64_t f2, uint64_t a, uint64_t dim,
                                      uint32_t b, uint32_t k, double* out) {
    return guarded([&] {
        if (!out) fail(Errc::InvalidArgument, "out must not be NULL");
        *out = theoretical_variance(Profile{f1, f2, a, dim}, b, k);
    });
}

bbmh_status bbmh_estimate_codes(const uint8_t* codes1, const uint8_t* codes2, uint32_t k,
                                uint32_t b, uint64_t f1, uint64_t f2, uint64_t a, uint64_t dim,
                                bbmh_estimate* out) {
    return guarded([&] {
        if (!codes1 || !codes2 || !out) fail(Errc::InvalidArgument, "codes and out required");
        if (k < 1) fail(Errc::InvalidArgument, "k must be >= 1");
        put_estimate(estimate_codes(codes1, codes2, k, b, Profile{f1, f2, a, dim}), out);
    });
}

bbmh_status bbmh_estimate_minima(const uint64_t* minima1, const uint64_t* minima2, uint32_t k,
                                 double* r_hat_out) {
    return guarded([&] {
        if (!minima1 || !minima2 || !r_hat_out)
            fail(Errc::InvalidArgument, "minima and out required");
        *r_hat_out = estimate_minima(minima1, minima2, k);
    });
}

bbmh_status bbmh_estimate_file(const char* sketch_path, uint64_t record1, uint64_t record2,
                               uint64_t f1, uint64_t f2, uint64_t a, int32_t use_minima,
                               bbmh_estimate* out, double* r_full_out) {
    return guarded([&] {
        if (!out) fail(Errc::InvalidArgument, "out must not be NULL");
        Estimate e;
        // *out is filled before the full-minima step can fail (capi.cpp:235-239)
        struct Fill {
            Estimate* e;
            bbmh_estimate* out;
            bool armed = false;
            ~Fill() {
                if (armed) put_estimate(*e, out);
            }
        } fill{&e, out};
        const std::string path = require(sketch_path, "sketch_path");
        try {
            estimate_file(path, record1, record2, f1, f2, a, use_minima || r_full_out, r_full_out,
                          &e);
        } catch (const Error& err) {
            fill.armed = e.p_hat != 0 || e.c1b != 0;  // the b-bit part completed
            throw;
        }
        put_estimate(e, out);
    });
}

bbmh_status bbmh_ext_match_counts(const uint8_t* codes_a, uint64_t na, const uint8_t* codes_b,
                                  uint64_t nb, uint32_t k, uint32_t b, uint32_t* counts_out) {
    return guarded([&] {
        if ((na && !codes_a) || (nb && !codes_b) || (na && nb && !counts_out))
            fail(Errc::InvalidArgument, "codes and counts required");
        if (k < 1) fail(Errc::InvalidArgument, "k must be >= 1");
        if (b < 1 || b > 32) fail(Errc::InvalidArgument, "b must be in 1..32");
        match_counts_host(codes_a, na, codes_b, nb, k, b, counts_out);
    });
}

bbmh_status bbmh_ext_match_counts_device(const uint8_t* d_codes_a, uint64_t na,
                                         const uint8_t* d_codes_b, uint64_t nb, uint32_t k,
                                         uint32_t b, uint32_t* d_counts, void* stream) {
    return guarded([&] {
        if ((na && !d_codes_a) || (nb && !d_codes_b) || (na && nb && !d_counts))
            fail(Errc::InvalidArgument, "codes and counts required");
        if (k < 1) fail(Errc::InvalidArgument, "k must be >= 1");
        if (b < 1 || b > 32) fail(Errc::InvalidArgument, "b must be in 1..32");
        match_counts_device(d_codes_a, na, d_codes_b, nb, k, b, d_counts,
                            static_cast<cudaStream_t>(stream));
    });
}
bbmh_status bbmh_mse_experiment(int32_t, uint64_t, uint64_t, uint64_t, uint64_t, const uint32_t*,
                                size_t, const uint32_t*, size_t, uint64_t, uint64_t, uint32_t,
                                const char*) {
    return not_provided("bbmh_mse_experiment");
}
// capi.cpp:277-283 -> vw_project_file (vw.cpp:61-77), hashed/aggregated on the GPU
bbmh_status bbmh_vw_project_file(const char* corpus_path, const char* out_path, uint32_t bins,
                                 uint64_t seed) {
    return guarded([&] {
        // argument evaluation order of the reference build: out_path, then corpus_path
        const char* out = require(out_path, "out_path");
        const char* in = require(corpus_path, "corpus_path");
        vw_project_file(in, out, bins, seed);
    });
}
bbmh_status bbmh_train(const char*, const char*, const char*, const char*,
                       const bbmh_train_config*) {
    return not_provided("bbmh_train");
}
// capi.cpp:307-317 -> predict_file (learner.cpp:524-536), scored on the GPU
bbmh_status bbmh_predict(const char* model_path, const char* data_path, const char* scores_path,
                         double* accuracy_out) {
    return guarded([&] {
        const char* model = require(model_path, "model_path");
        const double acc = predict_data(model, data_path,
                                        scores_path && *scores_path ? scores_path : "", 8);
        if (accuracy_out) *accuracy_out = acc;
    });
}
bbmh_status bbmh_synth_pair(uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, const char*,
                            int32_t) {
    return not_provided("bbmh_synth_pair");
}
bbmh_status bbmh_synth_classification(const char*, uint64_t, uint64_t, double, double, double,
                                      uint64_t, int32_t) {
    return not_provided("bbmh_synth_classification");
}
bbmh_status bbmh_corpus_convert(const char*, const char*, int32_t, uint64_t) {
    return not_provided("bbmh_corpus_convert");
}
bbmh_status bbmh_bench_preprocess(const char*, const int32_t*, size_t, uint32_t, uint32_t,
                                  const uint64_t*, size_t, const uint32_t*, size_t, uint32_t,
                                  uint64_t, const char*) {
    return not_provided("bbmh_bench_preprocess");
}
bbmh_status bbmh_bench_epochs(const char*, const char*, uint32_t, uint32_t,
                              const bbmh_train_config*, const char*) {
    return not_provided("bbmh_bench_epochs");
}

}  // extern "C"
