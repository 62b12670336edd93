// options.cpp -- see options.hpp.
#include "options.hpp"

#include <atomic>
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

namespace bbmh {

namespace {

struct Def {
    const char* name;
    int64_t dflt;
};

// table order == enum order
constexpr Def kDefs[] = {
    {"tile", 0},
    {"smem_cap", 1},
    {"ctas_per_sm", 0},
    {"shape_j", 0},
    {"shape_tpb", 0},
    {"carveout", -1},
    {"dynamic_docs", 1},
    {"split_small_k", 1},
    {"uniform_2u", 1},
    {"uniform_sb_docs", 0},
    {"uniform_4u", 1},
    {"perm_tablewise", -1},
    {"perm_scratch_mb", 2048},
    {"gpu_permgen", 1},
    {"force_peer_copy", 0},
    {"gpu_parse", 1},
    {"gpu_parse_block", 0},
    {"parse_priority", 0},
    {"device_ids", 1},
    {"range_shards", 1},
    {"text_lanes", 4},
    {"read_threads", 16},
    {"delta16", -1},
    {"delta_raw_every", -1},
    {"host_sharers", 1},
    {"host_dram_gbs", 0},
    {"pcie_gbs", 55},
    {"zero_copy", 1},
    {"chunk_ids", 0},
    {"trace", 0},
};
static_assert(sizeof(kDefs) / sizeof(kDefs[0]) == size_t(Opt::kCount));

std::atomic<int64_t> g_vals[size_t(Opt::kCount)];
std::once_flag g_once;

void init() {
    std::call_once(g_once, [] {
        for (size_t i = 0; i < size_t(Opt::kCount); ++i) {
            int64_t v = kDefs[i].dflt;
            std::string env = "BBMH_OPT_";
            for (const char* p = kDefs[i].name; *p; ++p) env += char(std::toupper((unsigned char)*p));
            if (const char* e = std::getenv(env.c_str()); e && *e) v = std::strtoll(e, nullptr, 10);
            g_vals[i].store(v, std::memory_order_relaxed);
        }
    });
}

int find(const char* name) {
    if (!name) return -1;
    for (size_t i = 0; i < size_t(Opt::kCount); ++i)
        if (std::strcmp(kDefs[i].name, name) == 0) return int(i);
    return -1;
}

}  // namespace

int64_t opt(Opt o) {
    init();
    return g_vals[size_t(o)].load(std::memory_order_relaxed);
}

bool set_opt(const char* name, int64_t value) {
    init();
    const int i = find(name);
    if (i < 0) return false;
    g_vals[i].store(value, std::memory_order_relaxed);
    return true;
}

bool get_opt(const char* name, int64_t* value) {
    init();
    const int i = find(name);
    if (i < 0) return false;
    if (value) *value = g_vals[i].load(std::memory_order_relaxed);
    return true;
}

const char* opt_name(int i) {
    return i >= 0 && i < int(Opt::kCount) ? kDefs[i].name : "";
}

}  // namespace bbmh
