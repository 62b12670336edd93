// family.cpp -- host construction of the k index mappings.
//
// Restates HashFamily::build (reference src/hash_family.cpp:53-119) with the
// same validation order, error codes and messages, and bit-identical
// coefficients / permutation tables. Two B200-side changes:
//   * permutation tables (k sequential Fisher-Yates shuffles, 64 MiB each at
//     D = 2^24) are built by a pool of host threads, one table at a time per
//     thread -- the per-table sequence is unchanged, so tables are identical;
//   * everything the kernels need (doubled 4U coefficients, the division-free
//     `% D` magic) is derived once here, on the host.
#include <algorithm>
#include <atomic>
#include <bit>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>

#include "core.hpp"
#include "options.hpp"

namespace bbmh {

bool trace_on() {
    return opt(Opt::Trace) != 0;
}

void trace(const char* what) {
    if (!trace_on()) return;
    static const auto t0 = std::chrono::steady_clock::now();
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "bbmh-trace %10.3f %s\n", ms, what);
}

bool is_prime_u64(uint64_t n) {  // hash_family.cpp:28-37
    if (n < 2) return false;
    for (uint64_t d : {2ull, 3ull, 5ull, 7ull})
        if (n % d == 0) return n == d;
    for (uint64_t d = 11; d * d <= n; d += 2)
        if (n % d == 0) return false;
    return true;
}

MagicDiv make_magic31(uint64_t d) {
    MagicDiv m;
    if (d < 3 || d >= (1ull << 31) || (d & (d - 1)) == 0) return m;
    const uint32_t l = 64 - std::countl_zero(d - 1);  // ceil(log2 d), d not a power of two
    const unsigned __int128 num = (unsigned __int128)1 << (31 + l);
    const unsigned __int128 M = (num + d - 1) / d;
    if (M >= ((unsigned __int128)1 << 32)) return m;
    m.magic = uint32_t(M);
    m.shift = l - 1;
    m.ok = true;
    return m;
}

namespace {

// hash_family.cpp:43-49
uint64_t keyed_below(uint64_t seed, uint64_t tag, uint64_t j, uint64_t i, uint64_t bound) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    for (uint64_t attempt = 0;; ++attempt) {
        uint64_t v = keyed_u64(seed, tag, j, i * 64 + attempt);
        if (v < limit) return v % bound;
    }
}

void build_perm_tables(Family& f) {
    const uint64_t dim = f.dim;
    const uint32_t k = f.k;
    f.perm.resize(size_t(dim) * k);
    std::atomic<uint32_t> next{0};
    auto worker = [&] {
        for (uint32_t j; (j = next.fetch_add(1)) < k;) {
            uint32_t* tab = f.perm.data() + size_t(j) * dim;
            for (uint64_t t = 0; t < dim; ++t) tab[t] = uint32_t(t);
            SplitMix64 rng{keyed_u64(f.seed, rngtag::kPermutation, j, 0)};
            // hash_family.cpp:108-112, the same draws and swaps in the same
            // order; the draws run kAhead steps ahead of the swaps so the
            // random entry each swap touches is prefetched (the shuffle is
            // bound by cache misses into the 64 MB table otherwise)
            constexpr uint64_t kAhead = 32;
            uint64_t ring[kAhead];
            uint64_t t_draw = dim - 1;  // next t whose r is drawn
            auto draw = [&] {
                const uint64_t r = rng.next_below(t_draw + 1);
                ring[t_draw % kAhead] = r;
                __builtin_prefetch(tab + r, 1, 0);
                --t_draw;
            };
            for (uint64_t i = 0; i < kAhead && t_draw > 0; ++i) draw();
            for (uint64_t t = dim - 1; t > 0; --t) {
                const uint64_t r = ring[t % kAhead];
                std::swap(tab[t], tab[r]);
                if (t_draw > 0) draw();
            }
        }
    };
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    unsigned nthreads = std::min<uint64_t>(hw, k);
    if (uint64_t(dim) * k < (1u << 20)) nthreads = 1;  // not worth threads
    std::vector<std::thread> pool;
    for (unsigned i = 1; i < nthreads; ++i) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
}

}  // namespace

uint32_t Family::map(uint32_t j, uint32_t t) const {
    auto reduce_dim = [&](uint64_t h) {
        return uint32_t(dim_pow2 ? (h & (dim - 1)) : (h % dim));
    };
    switch (scheme) {
        case Scheme::TwoU: {  // hash_family.hpp:48-51 (shift count & 31: see oracle note)
            uint32_t h = twou[2 * j] + twou[2 * j + 1] * t;
            return s >= 32 ? h : h >> ((32 - s) & 31);
        }
        case Scheme::FourUBit: {
            const uint64_t* a = &fouru[4 * size_t(j)];
            uint64_t h = a[3];
            h = mod_mersenne31(h * t + a[2]);
            h = mod_mersenne31(h * t + a[1]);
            h = mod_mersenne31(h * t + a[0]);
            return reduce_dim(h);
        }
        case Scheme::FourUMod: {
            const uint64_t* a = &fouru[4 * size_t(j)];
            uint64_t h = a[3];
            h = (h * t + a[2]) % p;
            h = (h * t + a[1]) % p;
            h = (h * t + a[0]) % p;
            return reduce_dim(h);
        }
        case Scheme::Permutation:
            if (!perm.empty()) return perm[size_t(j) * dim + t];
            return perm_value_on_device(*this, j, t);
    }
    return 0;
}

std::unique_ptr<Family> build_family(Scheme scheme, uint64_t dim, uint32_t k, uint64_t seed,
                                     uint64_t prime, uint64_t perm_cap_bytes) {
    if (dim < 1) fail(Errc::InvalidArgument, "universe size must be >= 1");
    if (k < 1) fail(Errc::InvalidArgument, "k must be >= 1");

    auto fam = std::make_unique<Family>();
    Family& f = *fam;
    f.scheme = scheme;
    f.dim = dim;
    f.k = k;
    f.seed = seed;
    f.dim_pow2 = (dim & (dim - 1)) == 0;
    f.s = f.dim_pow2 ? uint32_t(std::countr_zero(dim)) : 0;

    switch (scheme) {
        case Scheme::TwoU: {
            if (!f.dim_pow2 || dim > (1ull << 32))
                fail(Errc::UnsupportedUniverse,
                     "2u requires a power-of-two universe <= 2^32, got " + std::to_string(dim));
            f.twou.resize(2 * size_t(k));
            for (uint32_t j = 0; j < k; ++j) {
                f.twou[2 * j] = uint32_t(keyed_u64(seed, rngtag::kTwoU, j, 0));
                f.twou[2 * j + 1] = uint32_t(keyed_u64(seed, rngtag::kTwoU, j, 1)) | 1u;
            }
            break;
        }
        case Scheme::FourUMod:
        case Scheme::FourUBit: {
            const uint64_t p = prime;
            if (scheme == Scheme::FourUBit && p != kMersenne31)
                fail(Errc::InvalidArgument, "4u-bit is fixed to p = 2^31-1");
            if (p > kMersenne31) fail(Errc::InvalidArgument, "prime modulus must be <= 2^31-1");
            if (!is_prime_u64(p)) fail(Errc::InvalidArgument, "modulus is not prime");
            if (dim >= p)
                fail(Errc::UnsupportedUniverse, "universe size " + std::to_string(dim) +
                                                    " must be < p = " + std::to_string(p));
            f.p = p;
            f.fouru.resize(4 * size_t(k));
            for (uint32_t j = 0; j < k; ++j)
                for (uint64_t i = 0; i < 4; ++i)
                    f.fouru[4 * size_t(j) + i] = keyed_below(seed, rngtag::kFourU, j, i, p);
            break;
        }
        case Scheme::Permutation: {
            const uint64_t bytes = dim * uint64_t(k) * sizeof(uint32_t);
            if (dim > (1ull << 32) || bytes / sizeof(uint32_t) / k != dim ||
                bytes > perm_cap_bytes)
                fail(Errc::PermutationTooLarge,
                     "permutation tables need " + std::to_string(dim * k * 4) +
                         " bytes, cap is " + std::to_string(perm_cap_bytes));
            if (!build_perm_tables_gpu(f)) build_perm_tables(f);
            break;
        }
    }
    return fam;
}

}  // namespace bbmh
