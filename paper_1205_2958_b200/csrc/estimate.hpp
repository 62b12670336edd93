// estimate.hpp -- b-bit resemblance estimation.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "core.hpp"

namespace bbmh {

// PairProfile (estimator.hpp:16-33)
struct Profile {
    uint64_t f1 = 0, f2 = 0, a = 0, dim = 0;
    double r1() const { return double(f1) / double(dim); }
    double r2() const { return double(f2) / double(dim); }
    double resemblance() const { return double(a) / double(f1 + f2 - a); }
    void validate() const;
};

struct Correction {
    double c1b = 0, c2b = 0;
};

// the fields of bbmh_estimate, in ABI order
struct Estimate {
    double r_hat = 0, r_raw = 0, p_hat = 0, c1b = 0, c2b = 0, var_theory = 0;
};

Correction correction_terms(const Profile& p, uint32_t b);
double theoretical_variance(const Profile& p, uint32_t b, uint32_t k);
Estimate estimate_from_matches(uint64_t matches, uint32_t k, uint32_t b, const Profile& p);
Estimate estimate_codes(const uint8_t* c1, const uint8_t* c2, uint32_t k, uint32_t b,
                        const Profile& p);
double estimate_minima(const uint64_t* m1, const uint64_t* m2, uint64_t k);
Estimate estimate_file(const std::string& path, uint64_t rec1, uint64_t rec2, uint64_t f1,
                       uint64_t f2, uint64_t a, bool want_full, double* r_full, Estimate* out);

// All-pairs matching-code counts on the GPU (match.cu): counts[i*nb + j] =
// #{t < k : code_t(A_i) == code_t(B_j)} over packed b-bit codes.
void match_counts_host(const uint8_t* codes_a, uint64_t na, const uint8_t* codes_b, uint64_t nb,
                       uint32_t k, uint32_t b, uint32_t* counts);
void match_counts_device(const uint8_t* d_codes_a, uint64_t na, const uint8_t* d_codes_b,
                         uint64_t nb, uint32_t k, uint32_t b, uint32_t* d_counts,
                         cudaStream_t stream);

}  // namespace bbmh
