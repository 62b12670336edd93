// residency_probe.cu -- are the persistent sketch kernel's CTAs co-resident?
//
// Builds the product kernel (csrc/kernels.cu, included) with TRACE on: thread
// 0 of every CTA records %smid, %globaltimer at start and end, and the
// documents it finished. Runs the library's own launch shape for 2U and
// 4U-bit at k = 500 on a webspam-shaped corpus and prints, per scheme, CTAs
// per SM, how late the last CTA started, and the number of CTAs resident per
// SM over time (time-weighted mean and max), as one JSON line each.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 \
//     -I paper_1205_2958_b200/csrc tools/residency_probe.cu \
//     paper_1205_2958_b200/csrc/perm.cu paper_1205_2958_b200/csrc/options.cpp -o residency_probe
#include "../paper_1205_2958_b200/csrc/kernels.cu"

#include <cstdio>
#include <random>
#include <vector>

using namespace bbmh;

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));       \
            std::exit(1);                                                       \
        }                                                                       \
    } while (0)

template <int SCHEME, bool POW2, int J>
void probe(const char* name, KernelFamily F, uint64_t n, const uint64_t* d_rp, const uint32_t* d_idx,
           uint8_t* d_codes, uint8_t* d_flags, int* d_err) {
    const int sms = device_sms();
    LaunchShape sh = choose_shape(F.k, F.scheme, n, sms);
    if (sh.J != J) {
        std::fprintf(stderr, "%s: library shape J=%d, probe built for J=%d\n", name, sh.J, J);
        return;
    }
    const uint64_t max_ctas = (uint64_t)sms * 64 * sh.jtiles;
    unsigned long long* d_trace = nullptr;
    CK(cudaMalloc(&d_trace, max_ctas * 4 * sizeof(unsigned long long)));
    CK(cudaMemset(d_trace, 0, max_ctas * 4 * sizeof(unsigned long long)));
    for (int rep = 0; rep < 2; ++rep)  // warm-up, then the traced run
        launch_one<SCHEME, POW2, J, true>(F, sh, d_rp, 0, d_idx, n, 8, d_codes, nullptr, d_flags, d_err,
                                          0, d_trace);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> tr(max_ctas * 4);
    CK(cudaMemcpy(tr.data(), d_trace, tr.size() * 8, cudaMemcpyDeviceToHost));
    struct Cta {
        unsigned sm;
        double t0, t1;
        unsigned long long docs;
    };
    std::vector<Cta> ctas;
    unsigned long long tmin = ~0ull, tmax = 0;
    for (uint64_t i = 0; i < max_ctas; ++i) {
        if (tr[4 * i + 2] == 0) continue;
        tmin = std::min(tmin, tr[4 * i + 1]);
        tmax = std::max(tmax, tr[4 * i + 2]);
        ctas.push_back({(unsigned)tr[4 * i], (double)tr[4 * i + 1], (double)tr[4 * i + 2], tr[4 * i + 3]});
    }
    std::vector<std::vector<std::pair<double, int>>> ev(sms);
    std::vector<int> per_sm(sms, 0);
    double last_start = 0;
    for (auto& c : ctas) {
        c.t0 -= tmin;
        c.t1 -= tmin;
        last_start = std::max(last_start, c.t0);
        if (c.sm < (unsigned)sms) {
            per_sm[c.sm]++;
            ev[c.sm].push_back({c.t0, +1});
            ev[c.sm].push_back({c.t1, -1});
        }
    }
    const double span = double(tmax - tmin);
    double mean_res = 0;
    int max_res = 0;
    for (int s = 0; s < sms; ++s) {
        auto& e = ev[s];
        std::sort(e.begin(), e.end());
        int cur = 0;
        double prev = 0, area = 0;
        for (auto& [t, d] : e) {
            area += cur * (t - prev);
            prev = t;
            cur += d;
            max_res = std::max(max_res, cur);
        }
        mean_res += area / span;
    }
    mean_res /= sms;
    int lo = 1 << 30, hi = 0;
    for (int v : per_sm) lo = std::min(lo, v), hi = std::max(hi, v);
    double first_end = 1e300;
    for (auto& c : ctas) first_end = std::min(first_end, c.t1);
    std::printf("{\"scheme\": \"%s\", \"k\": %u, \"docs\": %llu, \"J\": %d, \"tpb\": %d, \"ctas\": %zu, "
                "\"ctas_per_sm_min\": %d, \"ctas_per_sm_max\": %d, \"kernel_us\": %.1f, "
                "\"last_cta_start_us\": %.2f, \"first_cta_end_us\": %.1f, "
                "\"resident_ctas_per_sm_mean\": %.2f, \"resident_ctas_per_sm_max\": %d, "
                "\"warps_per_cta\": %d}\n",
                name, F.k, (unsigned long long)n, sh.J, sh.tpb, ctas.size(), lo, hi, span / 1e3,
                last_start / 1e3, first_end / 1e3, mean_res, max_res, sh.tpb / 32);
    CK(cudaFree(d_trace));
}

int main(int argc, char** argv) {
    const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 50000;
    const uint32_t nnz = 3728, k = 500;
    std::vector<uint64_t> rp(n + 1);
    std::vector<uint32_t> idx((size_t)n * nnz);
    std::mt19937_64 g(1);
    for (uint64_t i = 0; i <= n; ++i) rp[i] = i * nnz;
    for (auto& v : idx) v = uint32_t(g() % 16609143);
    uint64_t* d_rp;
    uint32_t* d_idx;
    uint8_t *d_codes, *d_flags;
    int* d_err;
    CK(cudaMalloc(&d_rp, rp.size() * 8));
    CK(cudaMalloc(&d_idx, idx.size() * 4 + 16));
    CK(cudaMalloc(&d_codes, n * ((k * 8 + 7) / 8)));
    CK(cudaMalloc(&d_flags, n));
    CK(cudaMalloc(&d_err, 4));
    CK(cudaMemcpy(d_rp, rp.data(), rp.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_idx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice));
    std::vector<uint32_t> coef(4 * k);
    for (auto& c : coef) c = uint32_t(g()) | 1u;
    uint32_t* d_coef;
    CK(cudaMalloc(&d_coef, coef.size() * 4));
    CK(cudaMemcpy(d_coef, coef.data(), coef.size() * 4, cudaMemcpyHostToDevice));
    for (auto& c : coef) c &= 0x7ffffffeu;  // 4U operands < p (doubled ones even)
    uint32_t* d_coef4;
    CK(cudaMalloc(&d_coef4, coef.size() * 4));
    CK(cudaMemcpy(d_coef4, coef.data(), coef.size() * 4, cudaMemcpyHostToDevice));

    KernelFamily f2;
    f2.scheme = 1;
    f2.k = k;
    f2.dim = 1ull << 24;
    f2.shift2u = 8;
    f2.coef = d_coef;
    probe<S_2U, true, 8>("2u", f2, n, d_rp, d_idx, d_codes, d_flags, d_err);

    KernelFamily f4;
    f4.scheme = 3;
    f4.k = k;
    f4.dim = 16609143;
    f4.dim_pow2 = 0;
    f4.p = 0x7fffffffu;
    f4.coef = d_coef4;
    // magic division by D (the library computes it in family.cpp; any valid pair works here)
    f4.dim32 = 16609143u;
    f4.neg_dim32 = 0u - 16609143u;
    f4.magic = uint32_t(((1ull << 56) + 16609143u - 1) / 16609143u);
    f4.magic_shift = 24;
    const LaunchShape s4 = choose_shape(k, 3, n, device_sms());
    if (s4.J == 2) probe<S_4UBIT, false, 2>("4u-bit", f4, n, d_rp, d_idx, d_codes, d_flags, d_err);
    else if (s4.J == 4) probe<S_4UBIT, false, 4>("4u-bit", f4, n, d_rp, d_idx, d_codes, d_flags, d_err);
    else if (s4.J == 8) probe<S_4UBIT, false, 8>("4u-bit", f4, n, d_rp, d_idx, d_codes, d_flags, d_err);
    else if (s4.J == 7) probe<S_4UBIT, false, 7>("4u-bit", f4, n, d_rp, d_idx, d_codes, d_flags, d_err);
    else probe<S_4UBIT, false, 1>("4u-bit", f4, n, d_rp, d_idx, d_codes, d_flags, d_err);
    return 0;
}
