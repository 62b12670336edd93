// Round trip of the host encoder (csrc/delta.cpp) against a scalar decoder:
// random chunks with sorted, unsorted, repeated, wide-gap, empty and one-id
// rows at random row offsets. Built and run by tests/test_delta_cpu.py.
#include "delta.hpp"
#include <cstdio>
#include <random>
#include <vector>
#include <algorithm>
using namespace bbmh;
int main() {
    std::mt19937_64 g(7);
    uint64_t total_bad = 0, trials = 0;
    for (int trial = 0; trial < 300; ++trial) {
        const uint64_t n = 1 + g() % 3000;
        const uint64_t base = g() % 1000;
        std::vector<uint64_t> rp(n + 1);
        std::vector<uint32_t> ids;
        rp[0] = base;
        for (uint64_t r = 0; r < n; ++r) {
            int kind = g() % 6;
            uint64_t m = kind == 0 ? 0 : (kind == 1 ? 1 + g() % 3 : g() % 2000);
            std::vector<uint32_t> row(m);
            if (kind == 2) { for (auto& x : row) x = uint32_t(g()); }  // unsorted, wide
            else if (kind == 3) { uint32_t v = uint32_t(g() % 70000); for (auto& x : row) { x = v; v += uint32_t(g() % 3); } } // repeats (d=0)
            else { uint32_t v = uint32_t(g() % 100000); for (auto& x : row) { x = v; v += 1 + uint32_t(g() % (kind == 4 ? 200000 : 9000)); } }
            ids.insert(ids.end(), row.begin(), row.end());
            rp[r + 1] = rp[r] + m;
        }
        const uint64_t nidx = ids.size();
        std::vector<uint16_t> d(nidx + 8);
        std::vector<uint32_t> ep(n + 1), ex(nidx + 64);
        uint64_t nexc = 0;
        bool ok = encode_delta16(rp.data(), n, base, ids.data(), d.data(), ep.data(), ex.data(), ex.size(), nexc);
        if (!ok) { printf("overflow?\n"); return 1; }
        uint64_t bad = 0;
        for (uint64_t r = 0; r < n; ++r) {
            uint32_t acc = 0, e = ep[r];
            for (uint64_t i = rp[r] - base; i < rp[r + 1] - base; ++i) {
                uint32_t v = d[i] ? d[i] : ex[e++];
                acc += v;
                bad += acc != ids[i];
            }
            if (e != ep[r + 1]) ++bad;
        }
        total_bad += bad; ++trials;
    }
    printf("trials %lu bad %lu\n", trials, total_bad);
}
