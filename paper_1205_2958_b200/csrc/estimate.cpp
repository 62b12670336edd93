// estimate.cpp -- b-bit resemblance estimation (host side).
//
// Theorem 1 of the paper: the b-bit collision probability is
// P_b = C1b + (1 - C2b) R, so R_hat = (P_hat - C1b) / (1 - C2b). Semantics,
// validation order and messages follow the reference (estimator.hpp:16-33,
// estimator.cpp:14-101, capi.cpp:187-240). The per-pair arithmetic is scalar
// double math, evaluated in the same operation order as the reference so
// results are bit-identical; the batched all-pairs matching counts run on
// the GPU (match.cu).
#include "estimate.hpp"

#include <algorithm>
#include <cmath>

#include "io.hpp"

namespace bbmh {

void Profile::validate() const {  // estimator.hpp:26-33
    if (dim == 0 || f1 > dim || f2 > dim) fail(Errc::InvalidArgument, "bad profile sizes");
    if (a > f1 || a > f2 || f1 + f2 - a > dim)
        fail(Errc::InvalidArgument, "infeasible intersection");
    if (f1 == 0 || f2 == 0) fail(Errc::DegenerateProfile, "resemblance undefined for empty sets");
}

// A(r) = r (1-r)^(2^b) / ((1-r) (1 - (1-r)^(2^b))), with (1-r)^(2^b) formed as
// exp(2^b log1p(-r)) and its complement as -expm1(...) so r -> 0 stays exact.
static double a_term(double r, double m) {
    if (r >= 1.0) return 0.0;
    const double lg = m * std::log1p(-r);
    const double pw = std::exp(lg);
    const double den = -std::expm1(lg);
    return r * pw / (1.0 - r) / den;
}

Correction correction_terms(const Profile& p, uint32_t b) {  // estimator.cpp:14-30
    p.validate();
    if (b < 1 || b > 32) fail(Errc::InvalidArgument, "b must be in 1..32");
    const double r1 = p.r1(), r2 = p.r2();
    const double m = std::ldexp(1.0, int(b));
    const double A1 = a_term(r1, m), A2 = a_term(r2, m);
    const double sum = r1 + r2;
    return {A1 * r2 / sum + A2 * r1 / sum, A1 * r1 / sum + A2 * r2 / sum};
}

double theoretical_variance(const Profile& p, uint32_t b, uint32_t k) {  // estimator.cpp:32-37
    if (k < 1) fail(Errc::InvalidArgument, "k must be >= 1");
    const Correction c = correction_terms(p, b);
    const double pb = c.c1b + (1.0 - c.c2b) * p.resemblance();
    return pb * (1.0 - pb) / (double(k) * (1.0 - c.c2b) * (1.0 - c.c2b));
}

static uint32_t code_at(const uint8_t* codes, uint32_t j, uint32_t b) {  // sketch.cpp:55-62
    uint32_t out = 0;
    uint64_t pos = uint64_t(j) * b;
    for (uint32_t i = 0; i < b; ++i, ++pos) out |= uint32_t((codes[pos >> 3] >> (pos & 7)) & 1u) << i;
    return out;
}

Estimate estimate_from_matches(uint64_t matches, uint32_t k, uint32_t b, const Profile& p) {
    const Correction c = correction_terms(p, b);  // estimator.cpp:53-69
    Estimate e;
    e.c1b = c.c1b;
    e.c2b = c.c2b;
    e.p_hat = double(matches) / double(k);
    e.r_raw = (e.p_hat - c.c1b) / (1.0 - c.c2b);
    e.r_hat = std::clamp(e.r_raw, 0.0, 1.0);
    e.var_theory = theoretical_variance(p, b, k);
    return e;
}

Estimate estimate_codes(const uint8_t* c1, const uint8_t* c2, uint32_t k, uint32_t b,
                        const Profile& p) {
    correction_terms(p, b);  // validation precedes decoding, as in the reference
    uint64_t matches = 0;
    for (uint32_t j = 0; j < k; ++j) matches += code_at(c1, j, b) == code_at(c2, j, b);
    return estimate_from_matches(matches, k, b, p);
}

double estimate_minima(const uint64_t* m1, const uint64_t* m2, uint64_t k) {  // estimator.cpp:45-51
    if (k == 0) fail(Errc::InvalidArgument, "minima vectors must have equal positive length");
    uint64_t matches = 0;
    for (uint64_t j = 0; j < k; ++j) matches += m1[j] == m2[j];
    return double(matches) / double(k);
}

// estimate_file (capi.cpp:225-240) through SketchReader::record (sketch.cpp:190-201)
Estimate estimate_file(const std::string& path, uint64_t rec1, uint64_t rec2, uint64_t f1,
                       uint64_t f2, uint64_t a, bool want_full, double* r_full, Estimate* out) {
    SketchFileReader rd(path);
    FILE* fm = std::fopen((path + ".min64").c_str(), "rb");  // optional sibling
    struct Closer {
        FILE* f;
        ~Closer() {
            if (f) std::fclose(f);
        }
    } guard{fm};
    const size_t cb = packed_code_bytes(rd.k(), rd.b());
    struct Rec {
        int8_t label;
        uint8_t flags;
        std::vector<uint8_t> codes;
        std::vector<uint64_t> minima;
    };
    auto record = [&](uint64_t i) {
        if (i >= rd.count()) fail(Errc::InvalidArgument, "record index out of range");
        Rec r;
        std::vector<uint8_t> codes, flags;
        std::vector<int8_t> labels;
        rd.seek(i);
        if (rd.read(1, codes, flags, labels) != 1) fail(Errc::Io, "short read");
        r.label = labels[0];
        r.flags = flags[0];
        r.codes = std::move(codes);
        if (fm) {
            if (std::fseek(fm, long(i) * long(rd.k()) * 8, SEEK_SET) != 0)
                fail(Errc::Io, "seek failed");
            r.minima.resize(rd.k());
            std::vector<uint8_t> raw(size_t(rd.k()) * 8);
            if (std::fread(raw.data(), 1, raw.size(), fm) != raw.size()) fail(Errc::Io, "short read");
            for (uint32_t j = 0; j < rd.k(); ++j) r.minima[j] = get_u64(raw.data() + 8 * size_t(j));
        }
        return r;
    };
    const Rec r1 = record(rec1);
    const Rec r2 = record(rec2);
    (void)cb;
    const Profile p{f1, f2, a, rd.dim()};
    // estimate_bbit with header checks (estimator.cpp:85-101): same file, so the
    // headers match; empty-set records are degenerate
    if ((r1.flags & 1) || (r2.flags & 1))
        fail(Errc::DegenerateProfile, "resemblance undefined for an empty set");
    *out = estimate_codes(r1.codes.data(), r2.codes.data(), rd.k(), rd.b(), p);
    if (want_full) {  // estimate_full (estimator.cpp:76-83)
        if (r1.minima.empty() || r2.minima.empty())
            fail(Errc::MissingMinima, "full minima not available (no .min64 file)");
        const double full = estimate_minima(r1.minima.data(), r2.minima.data(), rd.k());
        if (r_full) *r_full = full;
    }
    return *out;
}

}  // namespace bbmh
