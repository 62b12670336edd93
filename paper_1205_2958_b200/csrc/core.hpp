// core.hpp -- host-side core of libbbmh: error taxonomy, counter-based PRNG
// and the hash-family description shared by the host and the CUDA kernels.
//
// Semantics follow the reference (arxiv/paper_1205_2958, /root/reference/proj):
//   errors      src/errors.hpp:9-35
//   PRNG        src/prng.hpp:10-61
//   families    src/hash_family.hpp:12-119, src/hash_family.cpp:28-119
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace bbmh {

// src/errors.hpp:9-24 -- mapped to bbmh_status in capi.cpp
enum class Errc {
    InvalidArgument = 1,
    UnsupportedUniverse,
    PermutationTooLarge,
    HeaderMismatch,
    MissingMinima,
    DegenerateProfile,
    EmptySketch,
    DimensionExceeded,
    NonBinaryLabel,
    MalformedLine,
    NonBinaryValue,
    NonAscendingIndex,
    InfeasibleProfile,
    Io,
    Cuda,  // B200 build only: a failed CUDA call (reported as BBMH_E_INTERNAL)
};

class Error : public std::runtime_error {
public:
    Error(Errc code, std::string msg) : std::runtime_error(std::move(msg)), code_(code) {}
    Errc code() const { return code_; }

private:
    Errc code_;
};

[[noreturn]] inline void fail(Errc code, std::string msg) { throw Error(code, std::move(msg)); }

// A parse error at a (1-based) line of the text: the message is the
// reference's "line N: <detail>" (dataio.cpp:60-106). Range-sharded loaders
// count lines per range and renumber with the lines of the ranges before.
class LineError : public Error {
public:
    LineError(Errc code, uint64_t line, std::string detail)
        : Error(code, "line " + std::to_string(line) + ": " + detail), line_(line), detail_(std::move(detail)) {}
    uint64_t line() const { return line_; }
    const std::string& detail() const { return detail_; }

private:
    uint64_t line_;
    std::string detail_;
};

// Developer tracing: with the "trace" option on (options.hpp), prints
// "bbmh-trace <ms since first call> <what>" to stderr (pipeline stage timing).
void trace(const char* what);
bool trace_on();

// ---- counter-based PRNG (src/prng.hpp:10-61), bit-exact ------------------
constexpr uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

constexpr uint64_t keyed_u64(uint64_t seed, uint64_t tag, uint64_t j, uint64_t i) {
    uint64_t x = mix64(seed + 0x9e3779b97f4a7c15ull * (tag + 1));
    x = mix64(x ^ (j + 0xd1b54a32d192ed03ull));
    x = mix64(x ^ (i + 0x8cb92ba72f3d8dd7ull));
    return x;
}

namespace rngtag {
inline constexpr uint64_t kPermutation = 1;
inline constexpr uint64_t kTwoU = 2;
inline constexpr uint64_t kFourU = 3;
}  // namespace rngtag

struct SplitMix64 {
    uint64_t state;
    uint64_t next() {
        state += 0x9e3779b97f4a7c15ull;
        return mix64(state);
    }
    uint64_t next_below(uint64_t bound) {
        if ((bound & (bound - 1)) == 0) return next() & (bound - 1);
        const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
        uint64_t v;
        do {
            v = next();
        } while (v >= limit);
        return v % bound;
    }
};

// ---- hash families --------------------------------------------------------
enum class Scheme : uint8_t { Permutation = 0, TwoU = 1, FourUMod = 2, FourUBit = 3 };

inline constexpr uint64_t kMersenne31 = (1ull << 31) - 1;
inline constexpr uint64_t kDefaultPermCapBytes = 1ull << 30;

// src/hash_family.hpp:24-32
inline uint64_t mod_mersenne31(uint64_t v) {
    constexpr uint64_t p = kMersenne31;
    v = (v >> 31) + (v & p);
    if (v >= 2 * p) v = (v >> 31) + (v & p);
    if (v >= p) return v - p;
    return v;
}

// Exact division-free `h % d` for h < 2^31 (Granlund-Montgomery with N = 31):
// q = umulhi(h, magic) >> shift. Valid when `ok`; d a power of two uses a mask.
struct MagicDiv {
    uint32_t magic = 0;
    uint32_t shift = 0;
    bool ok = false;
};
MagicDiv make_magic31(uint64_t d);

struct DeviceFamily;  // per-GPU residency (device.cu)

// Immutable after build; shareable across threads (hash_family.hpp:65-66).
struct Family {
    Scheme scheme = Scheme::TwoU;
    uint64_t dim = 0;
    uint32_t k = 0;
    uint64_t seed = 0;
    uint32_t s = 0;        // log2(dim) for power-of-two dim
    bool dim_pow2 = false;
    uint64_t p = kMersenne31;
    std::vector<uint32_t> twou;   // k * {a1, a2}      (hash_family.cpp:72-75)
    std::vector<uint64_t> fouru;  // k * {a0,a1,a2,a3} (hash_family.cpp:90-95)
    std::vector<uint32_t> perm;   // k * dim, table j at [j*dim, (j+1)*dim) (host-built)
    // tables built on a GPU instead (permgen.cu): they live in device memory
    // only, owned by that device's DeviceFamily; `perm` stays empty
    const uint32_t* perm_dev = nullptr;
    int perm_dev_id = -1;

    // host-side single evaluation (bbmh_family_map; hash_family.hpp:77-92)
    uint32_t map(uint32_t j, uint32_t t) const;

    // lazily created per-device copies
    mutable std::mutex dev_mu;
    mutable std::vector<std::unique_ptr<DeviceFamily>> dev;  // indexed by device ordinal
    Family();
    ~Family();
};

// Permutation tables built on the current GPU (permgen.cu): the same
// Fisher-Yates draws and swaps as hash_family.cpp:105-114. Returns false
// (nothing changed) when no GPU / not enough memory; the caller then builds
// them on the host.
bool build_perm_tables_gpu(Family& f);
// One entry of device-resident tables read back (bbmh_family_map).
uint32_t perm_value_on_device(const Family& f, uint32_t j, uint32_t t);

// src/hash_family.cpp:53-119 (same validation order, codes and messages).
std::unique_ptr<Family> build_family(Scheme scheme, uint64_t dim, uint32_t k, uint64_t seed,
                                     uint64_t prime, uint64_t perm_cap_bytes);

bool is_prime_u64(uint64_t n);

inline size_t packed_code_bytes(uint32_t k, uint32_t b) { return (size_t(k) * b + 7) / 8; }

}  // namespace bbmh
