// predict.cu -- bbmh_predict on the GPU (the consumer of
// sketches right after the preprocessing path).
//
// Reference: bbmh_predict (capi.cpp:307-317) = load_model (learner.cpp:588-612)
// + open_rows (learner.cpp:301-312: BBMH sketch -> runtime expansion, BBCV,
// or LibSVM text with real values) + predict_file (learner.cpp:524-536):
//   score = sum_i w[idx_i] * value_i   (double; value 1 for binary rows),
//   empty rows score 0, class = score >= 0 ? +1 : -1,
//   table rows "%d\t%.9g\n", accuracy = correct / n.
// Here every batch of rows is scored on the device:
//   * BBMH input: packed codes + flags go to the GPU and score.cu's kernel
//     expands and scores them (device-side SketchReader + expansion);
//   * BBCV / LibSVM input: one thread per row accumulates w[idx] * value in the
//     reference's order with separately rounded multiply and add (the
//     reference's x86-64 build does not contract to FMA), so scores are
//     bit-identical doubles.
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "engine.hpp"
#include "io.hpp"
#include "pipeline.hpp"

namespace bbmh {

namespace {

__global__ void __launch_bounds__(128) raw_score_kernel(const uint64_t* __restrict__ row_ptr,
                                                        const uint32_t* __restrict__ ids,
                                                        const float* __restrict__ vals,
                                                        uint64_t n, const double* __restrict__ w,
                                                        uint64_t wdim, double* __restrict__ scores,
                                                        unsigned long long* bad) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t beg = row_ptr[r], end = row_ptr[r + 1];
        double s = 0.0;
        for (uint64_t i = beg; i < end; ++i) {
            const uint32_t idx = ids[i];
            if ((uint64_t)idx >= wdim) {
                atomicMin(bad, (unsigned long long)(r << 32 | ((i - beg) & 0xffffffffu)));
                break;
            }
            s = __dadd_rn(s, vals ? __dmul_rn(w[idx], (double)vals[i]) : w[idx]);
        }
        scores[r] = s;  // empty rows: 0.0 (learner.cpp:528)
    }
}

template <typename T>
struct DevVec {
    T* p = nullptr;
    size_t cap = 0;
    void reserve(size_t n) {
        if (n <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        cap = std::max<size_t>(n, cap + cap / 2);
        BBMH_CUDA(cudaMalloc(&p, cap * sizeof(T)));
    }
    ~DevVec() {
        if (p) cudaFree(p);
    }
};

class ScoreTable {
public:
    explicit ScoreTable(const std::string& path) {  // open_table (capi.cpp:80-85)
        if (path.empty()) return;
        if (path == "-") {
            f_ = stdout;
            return;
        }
        f_ = std::fopen(path.c_str(), "wb");
        if (!f_) fail(Errc::Io, path + ": cannot open for writing");
    }
    ~ScoreTable() {
        if (f_ && f_ != stdout) std::fclose(f_);
    }
    void add(const double* scores, const int8_t* labels, uint64_t n) {
        for (uint64_t i = 0; i < n; ++i) {
            const int cls = scores[i] >= 0 ? 1 : -1;
            if (f_) std::fprintf(f_, "%d\t%.9g\n", cls, scores[i]);
            correct_ += cls == labels[i];
        }
        n_ += n;
    }
    double accuracy() const { return n_ ? double(correct_) / double(n_) : 0.0; }

private:
    FILE* f_ = nullptr;
    uint64_t n_ = 0, correct_ = 0;
};

[[noreturn]] void dim_exceeded(uint32_t idx, uint64_t dim) {
    fail(Errc::DimensionExceeded,
         "feature " + std::to_string(idx) + " >= dim " + std::to_string(dim));
}

constexpr uint64_t kPredictRows = 65536;
constexpr uint64_t kPredictIds = 1ull << 24;

}  // namespace

double predict_data(const std::string& model_path, const char* data_path_c,
                    const std::string& scores_path, unsigned threads) {
    const std::vector<double> w = load_decision_weights(model_path);
    const uint64_t wdim = w.size();
    if (!data_path_c) fail(Errc::InvalidArgument, "data_path must not be NULL");  // capi.cpp:311
    const std::string data_path = data_path_c;
    FILE* probe = open_or_fail(data_path, "rb");
    char magic[4] = {0, 0, 0, 0};
    const size_t got = std::fread(magic, 1, 4, probe);
    std::fclose(probe);
    const bool sketch = got == 4 && std::memcmp(magic, "BBMH", 4) == 0;

    cudaStream_t st;
    BBMH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    DevVec<double> d_w, d_scores;
    DevVec<unsigned long long> d_bad;
    d_w.reserve(std::max<uint64_t>(wdim, 1));
    d_bad.reserve(1);
    if (wdim) BBMH_CUDA(cudaMemcpy(d_w.p, w.data(), wdim * sizeof(double), cudaMemcpyHostToDevice));
    std::vector<double> scores;
    unsigned long long h_bad = 0;

    if (sketch) {
        // SketchRowSource (learner.cpp:271-297): SketchReader header, then expanded_dim
        SketchFileReader rd(data_path);
        const uint32_t k = rd.k(), b = rd.b();
        if (b < 1 || b > 32) fail(Errc::InvalidArgument, "b must be in 1..32");
        if ((uint64_t(1) << b) * k > (uint64_t(1) << 32))
            fail(Errc::DimensionExceeded, "2^b * k exceeds 32-bit row indices");
        ScoreTable table(scores_path);
        const size_t cb = packed_code_bytes(k, b);
        DevVec<uint8_t> d_codes, d_flags;
        std::vector<uint8_t> codes, flags;
        std::vector<int8_t> labels;
        for (;;) {
            const uint64_t n = rd.read(kPredictRows, codes, flags, labels);
            if (n == 0) break;
            d_codes.reserve(std::max<uint64_t>(n * cb, 1));
            d_flags.reserve(n);
            d_scores.reserve(n);
            BBMH_CUDA(cudaMemcpyAsync(d_codes.p, codes.data(), n * cb, cudaMemcpyHostToDevice, st));
            BBMH_CUDA(cudaMemcpyAsync(d_flags.p, flags.data(), n, cudaMemcpyHostToDevice, st));
            BBMH_CUDA(cudaMemsetAsync(d_bad.p, 0xff, sizeof(unsigned long long), st));
            launch_score(d_codes.p, d_flags.p, n, k, b, d_w.p, wdim, d_scores.p, d_bad.p, st);
            BBMH_CUDA(cudaGetLastError());
            scores.resize(n);
            BBMH_CUDA(cudaMemcpyAsync(scores.data(), d_scores.p, n * sizeof(double),
                                      cudaMemcpyDeviceToHost, st));
            BBMH_CUDA(cudaMemcpyAsync(&h_bad, d_bad.p, sizeof h_bad, cudaMemcpyDeviceToHost, st));
            BBMH_CUDA(cudaStreamSynchronize(st));
            if (h_bad != ~0ull) {
                const uint64_t r = h_bad >> 24;
                const uint32_t j = uint32_t(h_bad & 0xffffff);
                uint32_t code = 0;
                for (uint32_t i = 0; i < b; ++i) {
                    const uint64_t pos = uint64_t(j) * b + i;
                    code |= uint32_t((codes[r * cb + (pos >> 3)] >> (pos & 7)) & 1u) << i;
                }
                dim_exceeded(uint32_t((uint64_t(j) << b) + code), wdim);
            }
            table.add(scores.data(), labels.data(), n);
        }
        return table.accuracy();
    }

    auto reader = open_corpus(data_path, threads, /*libsvm_values=*/true);
    ScoreTable table(scores_path);
    Batch batch;
    DevVec<uint64_t> d_rp;
    DevVec<uint32_t> d_ids;
    DevVec<float> d_vals;
    for (;;) {
        batch.clear();
        batch.reserve_ids(kPredictIds + kPredictIds / 4);
        if (!reader->fill(batch, kPredictRows, kPredictIds)) break;
        const uint64_t n = batch.n, nid = batch.nids();
        d_rp.reserve(n + 1);
        d_ids.reserve(std::max<uint64_t>(nid, 1));
        d_scores.reserve(n);
        BBMH_CUDA(cudaMemcpyAsync(d_rp.p, batch.row_ptr.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
        if (nid)
            BBMH_CUDA(cudaMemcpyAsync(d_ids.p, batch.ids, nid * 4, cudaMemcpyHostToDevice, st));
        const float* vals = nullptr;
        if (!batch.vals.empty()) {
            d_vals.reserve(nid);
            BBMH_CUDA(cudaMemcpyAsync(d_vals.p, batch.vals.data(), nid * 4, cudaMemcpyHostToDevice, st));
            vals = d_vals.p;
        }
        BBMH_CUDA(cudaMemsetAsync(d_bad.p, 0xff, sizeof(unsigned long long), st));
        int dev = 0, sms = 148;
        BBMH_CUDA(cudaGetDevice(&dev));
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const uint64_t want = (n + 127) / 128;
        const unsigned grid = unsigned(want < uint64_t(sms) * 16 ? want : uint64_t(sms) * 16);
        raw_score_kernel<<<grid, 128, 0, st>>>(d_rp.p, d_ids.p, vals, n, d_w.p, wdim, d_scores.p,
                                               d_bad.p);
        BBMH_CUDA(cudaGetLastError());
        count_launches(1);
        scores.resize(n);
        BBMH_CUDA(cudaMemcpyAsync(scores.data(), d_scores.p, n * sizeof(double),
                                  cudaMemcpyDeviceToHost, st));
        BBMH_CUDA(cudaMemcpyAsync(&h_bad, d_bad.p, sizeof h_bad, cudaMemcpyDeviceToHost, st));
        BBMH_CUDA(cudaStreamSynchronize(st));
        if (h_bad != ~0ull) {
            const uint64_t r = h_bad >> 32, i = h_bad & 0xffffffffu;
            dim_exceeded(batch.ids[batch.row_ptr[r] + i], wdim);
        }
        table.add(scores.data(), batch.labels.data(), n);
    }
    return table.accuracy();
}

}  // namespace bbmh
