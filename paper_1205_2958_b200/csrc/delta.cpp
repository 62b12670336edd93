// delta.cpp -- host side of the 2-byte id transfer encoding (see delta.hpp).
//
// The encode is bound by host DRAM bandwidth (it runs beside the DMA that
// reads its output), so each task streams over a contiguous range of ids:
// 8 differences per AVX2 step (two overlapping loads give each id and its
// predecessor), stored with non-temporal stores -- no read-for-ownership of
// the output lines, 2 B of traffic per id saved (+12% measured with the DMA
// running, profiles/r11/host_encode_probe.jsonl). Row starts (difference to
// 0, not to the previous row's last id) are patched afterwards, and the
// escape positions recorded on the way are assigned to rows.
#include "delta.hpp"

#include <immintrin.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "hostpool.hpp"

namespace bbmh {

namespace {

// d in [1, 2^16) travels as is; 0 and >= 2^16 escape
inline bool escapes(uint32_t d) { return d - 1u >= 65535u; }

inline void encode_one(const uint32_t* s, uint16_t* o, uint64_t i, std::vector<uint64_t>& pos) {
    const uint32_t d = s[i] - (i ? s[i - 1] : 0u);
    const bool e = escapes(d);
    o[i] = e ? 0 : uint16_t(d);
    if (e) pos.push_back(i);
}

// Plain differences s[i] - s[i-1] over [a, b); escape positions appended in order.
void encode_range_scalar(const uint32_t* s, uint16_t* o, uint64_t a, uint64_t b,
                         std::vector<uint64_t>& pos) {
    for (uint64_t i = a; i < b; ++i) encode_one(s, o, i, pos);
}

__attribute__((target("avx2"))) void encode_range_avx2(const uint32_t* s, uint16_t* o, uint64_t a,
                                                       uint64_t b, std::vector<uint64_t>& pos) {
    const bool aligned = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
    uint64_t i = a;
    for (; i < b && ((i & 7) || i == 0); ++i) encode_one(s, o, i, pos);
    const __m256i hi = _mm256_set1_epi32(int(0xffff0000u));
    const __m256i zero = _mm256_setzero_si256();
    const __m256i ones = _mm256_set1_epi32(-1);
    for (; i + 8 <= b; i += 8) {
        const __m256i x = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        const __m256i p = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i - 1));
        const __m256i d = _mm256_sub_epi32(x, p);
        // escape: d has high bits, or d == 0
        const __m256i small = _mm256_cmpeq_epi32(_mm256_and_si256(d, hi), zero);
        const __m256i esc = _mm256_or_si256(_mm256_xor_si256(small, ones), _mm256_cmpeq_epi32(d, zero));
        const __m256i v = _mm256_andnot_si256(esc, d);
        const __m256i packed = _mm256_packus_epi32(v, v);  // per 128-bit lane: d0-3 d0-3 | d4-7 d4-7
        const __m128i out = _mm256_castsi256_si128(_mm256_permute4x64_epi64(packed, 0x08));
        if (aligned) _mm_stream_si128(reinterpret_cast<__m128i*>(o + i), out);
        else _mm_storeu_si128(reinterpret_cast<__m128i*>(o + i), out);
        unsigned m = unsigned(_mm256_movemask_ps(_mm256_castsi256_ps(esc)));
        while (m) {
            pos.push_back(i + unsigned(__builtin_ctz(m)));
            m &= m - 1;
        }
    }
    for (; i < b; ++i) encode_one(s, o, i, pos);
    _mm_sfence();  // the streamed lines are visible before the row-start patches
}

bool have_avx2() {
    static const bool on = __builtin_cpu_supports("avx2");
    return on;
}

}  // namespace

bool delta16_worthwhile(const uint64_t* row_ptr, uint64_t n, uint64_t base, const uint32_t* ids) {
    // sample up to 8 rows spread over the chunk: sorted, and a mean gap well
    // under 2^16 (then escapes are rare: P(gap >= 2^16) ~ exp(-2^16 / mean))
    uint64_t span = 0, cnt = 0;
    const uint64_t step = std::max<uint64_t>(1, n / 8);
    for (uint64_t r = 0; r < n; r += step) {
        const uint64_t a = row_ptr[r] - base, b = row_ptr[r + 1] - base;
        if (b - a < 2) continue;
        const uint32_t* s = ids + a;
        const uint64_t m = b - a;
        for (uint64_t i = 1; i < std::min<uint64_t>(m, 64); ++i)
            if (s[i] <= s[i - 1]) return false;
        if (s[m - 1] <= s[0]) return false;
        span += uint64_t(s[m - 1] - s[0]);
        cnt += m - 1;
    }
    return cnt > 0 && span / cnt <= 8192;
}

bool encode_delta16(const uint64_t* row_ptr, uint64_t n, uint64_t base, const uint32_t* ids,
                    uint16_t* deltas, uint32_t* exc_ptr, uint32_t* exc, uint64_t exc_cap,
                    uint64_t& nexc) {
    const uint64_t nidx = row_ptr[n] - base;
    // tasks of >= 64 Ki ids, up to 4 per pool thread (taken dynamically: a
    // thread the driver or the DMA interrupts holds nobody up), split at row
    // boundaries by id count
    const unsigned T = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(4 * host_threads(), nidx >> 16)));
    std::vector<uint64_t> r0(T + 1);
    for (unsigned w = 0; w <= T; ++w) {
        const uint64_t target = base + nidx * w / T;
        r0[w] = w == T ? n : uint64_t(std::lower_bound(row_ptr, row_ptr + n, target) - row_ptr);
    }
    std::vector<std::vector<uint64_t>> pos(T);  // per task: escape positions, in order
    std::vector<uint64_t> tot(T + 1, 0);
    const bool avx2 = have_avx2();
    host_parallel(T, [&](unsigned w) {
        const uint64_t a = row_ptr[r0[w]] - base, b = row_ptr[r0[w + 1]] - base;
        std::vector<uint64_t> raw;
        if (avx2) encode_range_avx2(ids, deltas, a, b, raw);
        else encode_range_scalar(ids, deltas, a, b, raw);
        // row starts: the difference is to 0; keep the escapes in row order
        std::vector<uint64_t>& out = pos[w];
        size_t k = 0;
        for (uint64_t r = r0[w]; r < r0[w + 1]; ++r) {
            const uint64_t ra = row_ptr[r] - base, rb = row_ptr[r + 1] - base;
            if (ra == rb) continue;
            const bool e0 = escapes(ids[ra]);
            deltas[ra] = e0 ? 0 : uint16_t(ids[ra]);
            if (e0) out.push_back(ra);
            for (; k < raw.size() && raw[k] < rb; ++k)
                if (raw[k] != ra) out.push_back(raw[k]);
        }
        tot[w + 1] = out.size();
    });
    for (unsigned w = 0; w < T; ++w) tot[w + 1] += tot[w];
    nexc = tot[T];
    if (nexc > exc_cap) return false;
    // each task's escape offsets per row and values; escapes are rare where
    // the encoding is used, so one serial pass unless there are many
    auto place = [&](unsigned w) {
        uint64_t at = tot[w];
        size_t k = 0;
        const std::vector<uint64_t>& p = pos[w];
        for (uint64_t r = r0[w]; r < r0[w + 1]; ++r) {
            exc_ptr[r] = uint32_t(at);
            const uint64_t ra = row_ptr[r] - base, rb = row_ptr[r + 1] - base;
            for (; k < p.size() && p[k] < rb; ++k)
                exc[at++] = p[k] == ra ? ids[ra] : ids[p[k]] - ids[p[k] - 1];
        }
    };
    if (nexc > (1u << 16)) {
        host_parallel(T, place);
    } else {
        for (unsigned w = 0; w < T; ++w) place(w);
    }
    exc_ptr[n] = uint32_t(nexc);
    return true;
}

}  // namespace bbmh
