// engine.cu -- host orchestration of the sketch kernels.
//
// Replaces the reference's worker pool (pipeline.cpp:171-191: k*nnz
// HashFamily::map calls per document on CPU threads) with chunked GPU
// execution: each chunk's CSR slice is copied H2D on a slot stream, sketched
// by one kernel launch, and its codes/minima/flags copied D2H, with three
// slots in flight per device so copies of one chunk overlap the kernel of
// another. Several devices pull chunks from one shared counter (document
// sharding, no collective): output position depends only on the chunk index.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>

#include "engine.hpp"
#include "delta.hpp"
#include "hostpool.hpp"
#include "options.hpp"

namespace bbmh {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(Errc::Cuda, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

DeviceFamily::~DeviceFamily() {
    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess) return;
    if (cudaSetDevice(device) != cudaSuccess) return;
    if (d_coef) cudaFree(d_coef);
    if (d_perm) cudaFree(d_perm);
    cudaSetDevice(prev);
}

Family::Family() = default;
Family::~Family() = default;

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        BBMH_CUDA(cudaGetDevice(&prev));
        if (prev != dev) BBMH_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

std::mutex g_cfg_mu;
std::vector<int> g_devices;
uint64_t g_chunk_docs = 0;

constexpr uint64_t kDefaultChunkDocs = 32768;
constexpr uint64_t kChunkIdxCap = 1ull << 24;        // 16 Mi ids (64 MiB) per chunk
constexpr uint64_t kChunkMinimaBytes = 256ull << 20;  // cap on a chunk's minima buffer
constexpr uint64_t kMinSplitIds = 1ull << 20;         // smallest chunk a batch is split into
// The sketch kernel's bulk copies read ids in whole 16-byte granules, i.e. up
// to 3 ids past a row's last one: every id buffer we allocate carries that slack.
constexpr uint64_t kIdsSlack = 4;

// Host -> device copy of a large pageable buffer (permutation tables: 31.25 GiB
// at C3). A plain cudaMemcpy from pageable memory runs at ~11 GB/s; here the
// bytes go through two page-locked staging buffers, filled by several threads,
// while the other buffer's DMA runs.
void upload_large(void* dst, const void* src, size_t bytes) {
    constexpr size_t kStage = size_t(128) << 20;
    if (bytes < 2 * kStage) {
        BBMH_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
        return;
    }
    char* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    cudaStream_t st = nullptr;
    struct Cleanup {
        char** stage;
        cudaEvent_t* done;
        cudaStream_t* st;
        ~Cleanup() {
            if (*st) cudaStreamSynchronize(*st);
            for (int i = 0; i < 2; ++i) {
                if (stage[i]) cudaFreeHost(stage[i]);
                if (done[i]) cudaEventDestroy(done[i]);
            }
            if (*st) cudaStreamDestroy(*st);
        }
    } cleanup{stage, done, &st};
    BBMH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        BBMH_CUDA(cudaMallocHost(&stage[i], kStage));
        BBMH_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    const unsigned T = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    const char* s = static_cast<const char*>(src);
    char* d = static_cast<char*>(dst);
    for (size_t off = 0, i = 0; off < bytes; off += kStage, ++i) {
        const int k = int(i & 1);
        const size_t n = std::min(kStage, bytes - off);
        BBMH_CUDA(cudaEventSynchronize(done[k]));  // this buffer's previous DMA is finished
        std::vector<std::thread> ts;
        for (unsigned w = 1; w < T; ++w)
            ts.emplace_back([&, w] {
                std::memcpy(stage[k] + n * w / T, s + off + n * w / T, n * (w + 1) / T - n * w / T);
            });
        std::memcpy(stage[k], s + off, n / T);
        for (auto& t : ts) t.join();
        BBMH_CUDA(cudaMemcpyAsync(d + off, stage[k], n, cudaMemcpyHostToDevice, st));
        BBMH_CUDA(cudaEventRecord(done[k], st));
    }
    BBMH_CUDA(cudaStreamSynchronize(st));
}

std::unique_ptr<DeviceFamily> upload_family(const Family& f, int device,
                                           uint32_t* adopt_perm = nullptr) {
    auto df = std::make_unique<DeviceFamily>();
    df->device = device;
    KernelFamily& kf = df->kf;
    // 4U-mod with the Mersenne prime (the default, capi.cpp:137) computes the
    // same residues as 4U-bit (hash_family.hpp:84-87 vs 24-32, SURVEY App. B:
    // 0 mismatches), so it runs the shift-add kernel: strength reduction of
    // `% p`, bit-identical output. Other primes keep the Barrett kernel.
    const Scheme scheme =
        f.scheme == Scheme::FourUMod && f.p == kMersenne31 ? Scheme::FourUBit : f.scheme;
    kf.scheme = int32_t(scheme);
    kf.k = f.k;
    kf.dim = f.dim;
    kf.shift2u = f.s >= 32 ? 0 : ((32 - f.s) & 31);  // see Family::map
    kf.dim_pow2 = f.dim_pow2 ? 1 : 0;
    kf.dim_mask = uint32_t(f.dim - 1);
    kf.dim32 = uint32_t(f.dim);
    kf.neg_dim32 = 0u - uint32_t(f.dim);
    kf.p = uint32_t(f.p);
    kf.barrett = f.p ? (~0ull) / f.p : 0;
    if (scheme == Scheme::FourUBit || scheme == Scheme::FourUMod) {
        if (!f.dim_pow2) {
            MagicDiv md = make_magic31(f.dim);
            if (!md.ok) fail(Errc::Cuda, "no 31-bit magic divisor for dim " + std::to_string(f.dim));
            kf.magic = md.magic;
            kf.magic_shift = md.shift;
        }
    }
    std::vector<uint32_t> coef;
    switch (scheme) {
        case Scheme::TwoU:
            coef = f.twou;
            break;
        case Scheme::FourUBit:  // {a3, 2a2, 2a1, 2a0}: doubled operands of the fold
            coef.resize(4 * size_t(f.k));
            for (uint32_t j = 0; j < f.k; ++j) {
                const uint64_t* a = &f.fouru[4 * size_t(j)];
                coef[4 * j + 0] = uint32_t(a[3]);
                coef[4 * j + 1] = uint32_t(2 * a[2]);
                coef[4 * j + 2] = uint32_t(2 * a[1]);
                coef[4 * j + 3] = uint32_t(2 * a[0]);
            }
            break;
        case Scheme::FourUMod:
            coef.resize(4 * size_t(f.k));
            for (uint32_t j = 0; j < f.k; ++j) {
                const uint64_t* a = &f.fouru[4 * size_t(j)];
                coef[4 * j + 0] = uint32_t(a[3]);
                coef[4 * j + 1] = uint32_t(a[2]);
                coef[4 * j + 2] = uint32_t(a[1]);
                coef[4 * j + 3] = uint32_t(a[0]);
            }
            break;
        case Scheme::Permutation:
            break;
    }
    DeviceGuard g(device);
    if (!coef.empty()) {
        BBMH_CUDA(cudaMalloc(&df->d_coef, coef.size() * sizeof(uint32_t)));
        BBMH_CUDA(cudaMemcpy(df->d_coef, coef.data(), coef.size() * sizeof(uint32_t),
                             cudaMemcpyHostToDevice));
        kf.coef = df->d_coef;
        if (scheme == Scheme::TwoU) kf.host2u = f.twou.data();  // lives as long as f (and df)
        if (scheme == Scheme::FourUBit) {
            df->host_coef = coef;
            kf.host4u = df->host_coef.data();
        }
    }
    if (f.scheme == Scheme::Permutation) {
        const size_t bytes = size_t(f.dim) * f.k * sizeof(uint32_t);
        if (adopt_perm) {  // built in place on this device (permgen.cu)
            df->d_perm = adopt_perm;
        } else if (f.perm.empty()) {
            // device-built tables live on another GPU: copy peer to peer
            // (NVLink when the devices can reach each other)
            BBMH_CUDA(cudaMalloc(&df->d_perm, bytes));
            int can = 0;
            cudaDeviceCanAccessPeer(&can, device, f.perm_dev_id);
            if (can) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(f.perm_dev_id, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    BBMH_CUDA(e);
                cudaGetLastError();
            }
            BBMH_CUDA(cudaMemcpyPeer(df->d_perm, device, f.perm_dev, f.perm_dev_id, bytes));
            count_peer_copy(bytes);
        } else {
            BBMH_CUDA(cudaMalloc(&df->d_perm, bytes));
            upload_large(df->d_perm, f.perm.data(), bytes);
        }
        kf.perm = df->d_perm;
    }
    return df;
}

// ---- per-device slot pool ------------------------------------------------
struct SlotPool {
    std::mutex mu;
    std::vector<Lane::Slot*> free;
};
std::mutex g_pool_mu;
std::vector<std::unique_ptr<SlotPool>> g_pools;

SlotPool& pool_for(int device) {
    std::lock_guard lk(g_pool_mu);
    if (size_t(device) >= g_pools.size()) g_pools.resize(device + 1);
    if (!g_pools[device]) g_pools[device] = std::make_unique<SlotPool>();
    return *g_pools[device];
}

Lane::Slot* acquire_slot(int device) {
    SlotPool& p = pool_for(device);
    {
        std::lock_guard lk(p.mu);
        if (!p.free.empty()) {
            Lane::Slot* s = p.free.back();
            p.free.pop_back();
            return s;
        }
    }
    auto* s = new Lane::Slot();
    s->device = device;
    DeviceGuard g(device);
    BBMH_CUDA(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
    BBMH_CUDA(cudaEventCreate(&s->ev0));
    BBMH_CUDA(cudaEventCreate(&s->ev1));
    BBMH_CUDA(cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming));
    BBMH_CUDA(cudaMalloc(&s->d_err, sizeof(int)));
    BBMH_CUDA(cudaMallocHost(&s->h_err, sizeof(int)));
    return s;
}

void release_slot(Lane::Slot* s) {
    if (!s) return;
    s->busy = false;
    SlotPool& p = pool_for(s->device);
    std::lock_guard lk(p.mu);
    p.free.push_back(s);
}

template <typename T>
void grow_device(T*& p, uint64_t& cap, uint64_t need) {
    if (need <= cap) return;
    if (p) BBMH_CUDA(cudaFree(p));
    p = nullptr;
    const uint64_t n = std::max<uint64_t>(need, cap + cap / 2);
    BBMH_CUDA(cudaMalloc(&p, n * sizeof(T)));
    cap = n;
}

template <typename T>
void grow_host(T*& p, uint64_t& cap, uint64_t need) {
    if (need <= cap) return;
    if (p) BBMH_CUDA(cudaFreeHost(p));
    p = nullptr;
    const uint64_t n = std::max<uint64_t>(need, cap + cap / 2);
    BBMH_CUDA(cudaMallocHost(&p, n * sizeof(T)));
    cap = n;
}

bool is_pinned(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void check_row_ptr(const uint64_t* rp, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i)
        if (rp[i + 1] < rp[i]) fail(Errc::InvalidArgument, "row_ptr must be non-decreasing");
}

}  // namespace

void adopt_device_perm(Family& f, int device, uint32_t* d_perm) {
    std::lock_guard lk(f.dev_mu);
    if (size_t(device) >= f.dev.size()) f.dev.resize(device + 1);
    f.perm_dev = d_perm;
    f.perm_dev_id = device;
    if (opt(Opt::ForcePeerCopy)) {
        // test hook: replicate through the peer-copy branch other GPUs take
        // (a same-device cudaMemcpyPeer), then serve from the replica
        f.dev[device] = upload_family(f, device);
        DeviceGuard g(device);
        BBMH_CUDA(cudaFree(d_perm));
        f.perm_dev = f.dev[device]->d_perm;
        return;
    }
    f.dev[device] = upload_family(f, device, d_perm);
}

void copy_perm_table(const Family& f, uint32_t j, uint32_t* out) {
    if (j >= f.k) fail(Errc::InvalidArgument, "j must be < k");
    if (!f.perm.empty()) {
        std::memcpy(out, f.perm.data() + size_t(j) * f.dim, size_t(f.dim) * sizeof(uint32_t));
        return;
    }
    DeviceGuard g(f.perm_dev_id);
    BBMH_CUDA(cudaMemcpy(out, f.perm_dev + size_t(j) * f.dim, size_t(f.dim) * sizeof(uint32_t),
                         cudaMemcpyDeviceToHost));
}

uint32_t perm_value_on_device(const Family& f, uint32_t j, uint32_t t) {
    DeviceGuard g(f.perm_dev_id);
    uint32_t v = 0;
    BBMH_CUDA(cudaMemcpy(&v, f.perm_dev + size_t(j) * f.dim + t, sizeof v, cudaMemcpyDeviceToHost));
    return v;
}

const DeviceFamily& device_family(const Family& f, int device) {
    std::lock_guard lk(f.dev_mu);
    if (size_t(device) >= f.dev.size()) f.dev.resize(device + 1);
    if (!f.dev[device]) f.dev[device] = upload_family(f, device);
    return *f.dev[device];
}

std::vector<int> pipeline_devices() {
    {
        std::lock_guard lk(g_cfg_mu);
        if (!g_devices.empty()) return g_devices;
    }
    int dev = 0;
    BBMH_CUDA(cudaGetDevice(&dev));
    return {dev};
}

void set_pipeline_devices(const std::vector<int>& ids) {
    int count = 0;
    BBMH_CUDA(cudaGetDeviceCount(&count));
    for (int id : ids)
        if (id < 0 || id >= count)
            fail(Errc::InvalidArgument, "device " + std::to_string(id) + " does not exist");
    std::lock_guard lk(g_cfg_mu);
    g_devices = ids;
}

uint64_t chunk_docs_setting() {
    std::lock_guard lk(g_cfg_mu);
    return g_chunk_docs ? g_chunk_docs : kDefaultChunkDocs;
}

void set_chunk_docs(uint64_t docs) {
    std::lock_guard lk(g_cfg_mu);
    g_chunk_docs = docs;
}

// ---- Lane ------------------------------------------------------------------
Lane::Lane(const Family& f, int device, uint32_t b, bool want_minima, const ScoreModel* score)
    : f_(f), device_(device), b_(b), cb_(packed_code_bytes(f.k, b)), want_minima_(want_minima) {
    trace("lane: ctor");
    df_ = &device_family(f, device);
    trace("lane: family resident");
    for (int i = 0; i < kSlots; ++i) slots_[i] = acquire_slot(device);
    trace("lane: slots acquired");
    if (score) {
        DeviceGuard g(device);
        wdim_ = score->dim;
        BBMH_CUDA(cudaMalloc(&d_w_, std::max<uint64_t>(wdim_, 1) * sizeof(double)));
        if (wdim_)
            BBMH_CUDA(cudaMemcpy(d_w_, score->w, wdim_ * sizeof(double), cudaMemcpyHostToDevice));
        trace("lane: model uploaded");
    }
}

Lane::~Lane() {
    trace("lane: dtor");
    for (int i = 0; i < kSlots; ++i) {
        if (slots_[i] && slots_[i]->busy) cudaStreamSynchronize(slots_[i]->st);
        release_slot(slots_[i]);
    }
    if (d_w_) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device_);
        cudaFree(d_w_);
        cudaSetDevice(prev);
    }
    trace("lane: dtor done");
}

void Lane::reserve(Slot& s, uint64_t rows, uint64_t nidx, bool need_pinned_idx) {
    if (rows + 1 > s.cap_rows) {  // row-sized buffers: row_ptr (device + pinned mirror), flags
        const uint64_t cap = std::max<uint64_t>(rows + 1, s.cap_rows + s.cap_rows / 2);
        if (s.d_rp) BBMH_CUDA(cudaFree(s.d_rp));
        if (s.d_flags) BBMH_CUDA(cudaFree(s.d_flags));
        if (s.h_rp) BBMH_CUDA(cudaFreeHost(s.h_rp));
        if (s.h_flags) BBMH_CUDA(cudaFreeHost(s.h_flags));
        BBMH_CUDA(cudaMalloc(&s.d_rp, cap * sizeof(uint64_t)));
        BBMH_CUDA(cudaMalloc(&s.d_flags, cap));
        BBMH_CUDA(cudaMallocHost(&s.h_rp, cap * sizeof(uint64_t)));
        BBMH_CUDA(cudaMallocHost(&s.h_flags, cap));
        s.cap_rows = cap;
    }
    grow_device(s.d_idx, s.cap_idx, nidx + kIdsSlack);
    if (need_pinned_idx) grow_host(s.h_idx, s.cap_idx_pinned, std::max<uint64_t>(nidx, 4));
    const uint64_t ncodes = std::max<uint64_t>(rows * cb_, 1);
    if (ncodes > s.cap_codes) {
        uint64_t c1 = s.cap_codes, c2 = s.cap_codes;
        grow_device(s.d_codes, c1, ncodes);
        grow_host(s.h_codes, c2, ncodes);
        s.cap_codes = std::min(c1, c2);
    }
    if (want_minima_) {
        const uint64_t nmin = std::max<uint64_t>(rows * f_.k, 1);
        if (nmin > s.cap_min) {
            uint64_t c1 = s.cap_min, c2 = s.cap_min;
            grow_device(s.d_min, c1, nmin);
            grow_host(s.h_min, c2, nmin);
            s.cap_min = std::min(c1, c2);
        }
    }
    if (d_w_) {
        if (!s.d_bad) {
            BBMH_CUDA(cudaMalloc(&s.d_bad, sizeof(unsigned long long)));
            BBMH_CUDA(cudaMallocHost(&s.h_bad, sizeof(unsigned long long)));
        }
        if (rows > s.cap_scores) {
            uint64_t c1 = s.cap_scores, c2 = s.cap_scores;
            grow_device(s.d_scores, c1, std::max<uint64_t>(rows, 1));
            grow_host(s.h_scores, c2, std::max<uint64_t>(rows, 1));
            s.cap_scores = std::min(c1, c2);
        }
    }
}

namespace {
constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// the lanes' host<->device copies, counted (bbmh_ext_transfer_bytes)
void h2d(void* d, const void* h, size_t n, cudaStream_t st) {
    BBMH_CUDA(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, st));
    count_transfer(n, 0);
}
void d2h(void* h, const void* d, size_t n, cudaStream_t st) {
    BBMH_CUDA(cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, st));
    count_transfer(0, n);
}
}  // namespace

// Chunks without minima: everything small the chunk moves goes through one
// pinned block per slot, so a chunk costs one H2D (plus one for page-locked
// caller ids, DMA'd in place), the kernel(s) and one D2H (the online
// small-batch case is bound by these API calls, not by bytes).
//   H2D  [0, off_err+16):        row_ptr | ids (pageable input only) | err=0, bad=~0
//   D2H  [off_err, blk_end):     err, bad | scores | flags | codes
// When the ids' H2D would bound the chunk they go 2 bytes each instead
// (delta.hpp), from pinned or pageable input alike:
//   H2D  [0, off_err+16):        row_ptr | exc_ptr | u16 deltas | escapes | err, bad
// and decode_delta16 rebuilds them in the slot's id buffer before the sketch.
namespace {

// option "delta16": 0 off, 1 on whenever possible (tests), -1: where it
// pays, on lanes that allow it (Lane::set_delta16)
int delta16_mode() {
    const int64_t v = opt(Opt::Delta16);
    return v < 0 ? 2 : v == 0 ? 0 : 1;
}

// The H2D of 4 B per id bounds the chunk when the kernel's time per id is
// below the copy's: 2U up to k ~ 1,000, 4U only at tiny k (kernel rates:
// 14.5 T and 1.3 T evals/s against ~55 GB/s of PCIe, profiles/r10).
bool delta16_pays(const KernelFamily& kf) {
    if (kf.scheme == int32_t(Scheme::TwoU)) return kf.k <= 1024;
    if (kf.scheme == int32_t(Scheme::Permutation)) return false;
    return kf.k <= 64;
}

// Below ~2 Mi ids a chunk's encode does not hide behind the previous chunk's
// copy and kernel: mid-size online batches (C5, 1,024 docs in 4 chunks of
// ~1 Mi ids) measured 0.41 ms with 4-byte ids and 0.56 ms encoded.
constexpr uint64_t kDeltaMinIds = 1ull << 21;

uint64_t chunk_idx_cap() {
    const int64_t v = opt(Opt::ChunkIds);
    return v >= (1 << 16) ? uint64_t(v) : kChunkIdxCap;
}

}  // namespace

// Ids/s the host encodes on all its cores (the shipped encoder on a
// webspam-shaped 32 Mi-id chunk, larger than the host's L3; best of 3),
// measured once per process. This rate includes the encode's own DRAM
// traffic (4 B read + 2 B written per id).
double host_encode_ids_per_s() {
    static const double rate = [] {
        constexpr uint64_t kRows = 8192, kPerRow = 4096, kIds = kRows * kPerRow;
        std::vector<uint64_t> rp(kRows + 1);
        std::vector<uint32_t> ids(kIds);
        std::vector<uint16_t> deltas(kIds);
        std::vector<uint32_t> exc_ptr(kRows + 1), exc(kIds / 8 + 64);
        for (uint64_t r = 0; r <= kRows; ++r) rp[r] = r * kPerRow;
        host_parallel(host_threads(), [&](unsigned w) {
            const uint64_t T = host_threads(), lo = kRows * w / T, hi = kRows * (w + 1) / T;
            for (uint64_t r = lo; r < hi; ++r) {
                uint32_t v = uint32_t(mix64(r) & 1023);
                for (uint64_t i = 0; i < kPerRow; ++i) {
                    v += 1 + uint32_t(mix64(r * kPerRow + i) % 8191);  // mean gap ~4,096
                    ids[r * kPerRow + i] = v;
                }
            }
        });
        double best = 0;
        for (int rep = 0; rep < 3; ++rep) {
            uint64_t nexc = 0;
            const auto t0 = std::chrono::steady_clock::now();
            encode_delta16(rp.data(), kRows, 0, ids.data(), deltas.data(), exc_ptr.data(), exc.data(),
                           exc.size(), nexc);
            const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            best = std::max(best, double(kIds) / s);
        }
        return best;
    }();
    return rate;
}

// Host bandwidth budget of the id transfer when `feeds` GPUs stream ids from
// this host at once (lanes of this process x "host_sharers", e.g. the ranks
// of one node). 4-byte ids cost 4 B of link per id and 4 B of DRAM reads
// (the DMA): min(feeds x link / 4, DRAM / 4) ids/s. 2-byte ids cost 2 B of
// link, but every id is first encoded by the host cores, which all feeds
// share: min(feeds x link / 2, the host's measured encode rate). The encode
// pays when it moves more ids per second (on a 16-core B200 host with one
// GPU: ~17 G against ~14 G ids/s; with two GPUs the raw copy wins).
bool delta16_budget_pays(uint64_t feeds, double* raw_ids_s, double* enc_ids_s) {
    feeds = std::max<uint64_t>(1, feeds);
    const double link = double(std::max<int64_t>(1, opt(Opt::PcieGbs))) * 1e9;
    const double dram = host_dram_bytes_per_s();
    const double raw = std::min(double(feeds) * link / 4, dram / 4);
    const double enc = std::min(double(feeds) * link / 2, host_encode_ids_per_s());
    if (raw_ids_s) *raw_ids_s = raw;
    if (enc_ids_s) *enc_ids_s = enc;
    return enc > 1.05 * raw;
}

uint32_t mixed_raw_every(uint64_t feeds, double* ids_s) {
    feeds = std::max<uint64_t>(1, feeds);
    const double link = double(feeds) * double(std::max<int64_t>(1, opt(Opt::PcieGbs))) * 1e9;
    const double enc = host_encode_ids_per_s();
    // The copy benchmark reads 106..185 GB/s on the 16-core box depending on
    // what else the process is doing; the encoder alone moves 6 B per id at
    // its measured rate, a floor under it. The pipeline interleaves encoder
    // traffic with DMA reads and sees ~85% of a pure copy: derated, the model
    // puts the optimum at every 3rd-4th chunk raw, where the measured curve
    // peaks (profiles/round2/e2e_mix.jsonl: 1/6 9.03, 1/4 9.34, 1/3 9.46,
    // 1/2 8.76 T evals/s against 8.67 all-encoded).
    const double dram = 0.85 * std::max(host_dram_bytes_per_s(), 6 * enc);
    // a fraction f of the ids crosses as 4-byte ids (4 B of link and of host
    // DRAM per id, no host cores), the rest encoded (2 B of link; 4 B read +
    // 2 B written by the encoder + 2 B read by the DMA; host cores)
    auto rate = [&](double f) {
        return std::min({link / (2 + 2 * f), dram / (8 - 4 * f), f < 1 ? enc / (1 - f) : 1e30});
    };
    // from the most raw chunks down, switching only for a 2% better rate:
    // near ties go to more raw chunks, where the measured curve is flat
    // (every 3rd / 4th: 9.46 / 9.34 T evals/s) and the model's link term is
    // the optimistic one
    uint32_t best = 3;
    double best_rate = rate(1.0 / 3);
    for (uint32_t every = 4; every <= 8; ++every) {
        const double r = rate(1.0 / every);
        if (r > 1.02 * best_rate) {
            best = every;
            best_rate = r;
        }
    }
    if (rate(0) > 1.02 * best_rate) {
        best = 0;
        best_rate = rate(0);
    }
    if (ids_s) *ids_s = best_rate;
    return best;
}

namespace {

}  // namespace

void Lane::enqueue_packed(Slot& s, const ChunkJob& job, uint64_t nidx) {
    const uint64_t n = job.n;
    const int dmode = delta16_mode();
    bool delta = dmode != 0 && nidx > 0 && !job.d_indices &&
                 (dmode == 1 || (delta16_ && !job.ids_as_is && nidx >= kDeltaMinIds && delta16_pays(df_->kf) &&
                                 delta16_worthwhile(job.row_ptr, n, job.index_base, job.indices)));
    const bool inline_ids = !job.pinned_input && !job.d_indices;
    const size_t raw_err = align16(align16((n + 1) * sizeof(uint64_t)) + (inline_ids ? nidx * sizeof(uint32_t) : 0));
    const size_t d_exc_ptr = align16((n + 1) * sizeof(uint64_t));
    const size_t d_deltas = align16(d_exc_ptr + (n + 1) * sizeof(uint32_t));
    const size_t d_exc = align16(d_deltas + nidx * sizeof(uint16_t));
    const uint64_t exc_cap = nidx / 8 + 64;
    const size_t tail = 16 + (d_w_ ? n * sizeof(double) : 0) + n + n * cb_;
    const size_t need = std::max(raw_err, delta ? align16(d_exc + exc_cap * sizeof(uint32_t)) : 0) + tail;
    if (need > s.cap_blk) {
        const uint64_t cap = std::max<uint64_t>(need, s.cap_blk + s.cap_blk / 2);
        if (s.d_blk) BBMH_CUDA(cudaFree(s.d_blk));
        if (s.h_blk) BBMH_CUDA(cudaFreeHost(s.h_blk));
        s.d_blk = nullptr;
        s.h_blk = nullptr;
        BBMH_CUDA(cudaMalloc(&s.d_blk, cap));
        BBMH_CUDA(cudaMallocHost(&s.h_blk, cap));
        s.cap_blk = cap;
    }
    s.packed = true;
    uint8_t* h = s.h_blk;
    uint8_t* d = s.d_blk;
    uint64_t nexc = 0;
    if (delta)
        delta = encode_delta16(job.row_ptr, n, job.index_base, job.indices,
                               reinterpret_cast<uint16_t*>(h + d_deltas),
                               reinterpret_cast<uint32_t*>(h + d_exc_ptr),
                               reinterpret_cast<uint32_t*>(h + d_exc), exc_cap, nexc);
    if (delta) trace("lane: ids encoded");
    count(delta ? Counter::Delta16Chunks : Counter::RawChunks);
    // from here on the slot's stream may hold work: the slot must be drained
    // before it is reused or returned, even if queueing below fails
    s.busy = true;
    s.off_ids = delta ? d_deltas : align16((n + 1) * sizeof(uint64_t));
    s.off_err = delta ? align16(d_exc + nexc * sizeof(uint32_t)) : raw_err;
    s.off_scores = s.off_err + 16;
    s.off_flags = s.off_scores + (d_w_ ? n * sizeof(double) : 0);
    s.off_codes = s.off_flags + n;  // no gap: every byte copied back is written by a kernel
    s.blk_end = s.off_codes + n * cb_;
    std::memcpy(h, job.row_ptr, (n + 1) * sizeof(uint64_t));
    // zero the alignment gaps too: every byte of the H2D block is defined
    auto zero_gap = [&](size_t from, size_t to) {
        if (to > from) std::memset(h + from, 0, to - from);
    };
    if (delta) {
        zero_gap((n + 1) * sizeof(uint64_t), d_exc_ptr);
        zero_gap(d_exc_ptr + (n + 1) * sizeof(uint32_t), d_deltas);
        zero_gap(d_deltas + nidx * sizeof(uint16_t), d_exc);
        zero_gap(d_exc + nexc * sizeof(uint32_t), s.off_err);
    } else {
        zero_gap((n + 1) * sizeof(uint64_t), s.off_ids);
        const size_t ids_end = s.off_ids + (inline_ids ? nidx * sizeof(uint32_t) : 0);
        zero_gap(ids_end, s.off_err);
        if (inline_ids && nidx) host_memcpy(h + s.off_ids, job.indices, nidx * sizeof(uint32_t));
    }
    std::memset(h + s.off_err, 0, 8);
    std::memset(h + s.off_err + 8, 0xff, 8);
    const uint32_t* d_ids = reinterpret_cast<const uint32_t*>(d + s.off_ids);
    if (job.d_indices) {
        d_ids = job.d_indices;
    } else if (delta || (!inline_ids && nidx)) {
        grow_device(s.d_idx, s.cap_idx, nidx + kIdsSlack);
        d_ids = s.d_idx;
    }
    if (!job.d_indices && !delta && !inline_ids && nidx)
        h2d(s.d_idx, job.indices, nidx * sizeof(uint32_t), s.st);
    h2d(s.d_blk, h, s.off_err + 16, s.st);
    if (delta) {
        launch_decode_delta16(reinterpret_cast<const uint64_t*>(d), job.index_base, n,
                              reinterpret_cast<const uint16_t*>(d + d_deltas),
                              reinterpret_cast<const uint32_t*>(d + d_exc_ptr),
                              reinterpret_cast<const uint32_t*>(d + d_exc), s.d_idx, s.st);
        BBMH_CUDA(cudaGetLastError());
    }
    auto* d_err = reinterpret_cast<int*>(d + s.off_err);
    auto* d_bad = reinterpret_cast<unsigned long long*>(d + s.off_err + 8);
    if (timed_) BBMH_CUDA(cudaEventRecord(s.ev0, s.st));
    launch_sketch(df_->kf, reinterpret_cast<const uint64_t*>(d), job.index_base, d_ids, n, b_,
                  d + s.off_codes,
                  nullptr, d + s.off_flags, d_err, s.st, n ? double(nidx) / double(n) : 0.0);
    BBMH_CUDA(cudaGetLastError());
    if (d_w_) {
        launch_score(d + s.off_codes, d + s.off_flags, n, f_.k, b_, d_w_, wdim_,
                     reinterpret_cast<double*>(d + s.off_scores), d_bad, s.st);
        BBMH_CUDA(cudaGetLastError());
    }
    if (timed_) BBMH_CUDA(cudaEventRecord(s.ev1, s.st));
    if (job.codes_out) {  // codes straight into the caller's page-locked buffer
        d2h(h + s.off_err, d + s.off_err, s.off_codes - s.off_err, s.st);
        if (n && cb_) d2h(job.codes_out, d + s.off_codes, n * cb_, s.st);
    } else {
        d2h(h + s.off_err, d + s.off_err, s.blk_end - s.off_err, s.st);
    }
    BBMH_CUDA(cudaEventRecord(s.done, s.st));
    s.busy = true;
    trace("lane: enqueued");
}

void Lane::enqueue(Slot& s, const ChunkJob& job) {
    trace("lane: enqueue");
    const uint64_t n = job.n;
    const uint64_t nidx = job.row_ptr[n] - job.index_base;
    const bool stage = !job.pinned_input;
    DeviceGuard g(device_);
    s.job = job;
    if (!want_minima_) {
        enqueue_packed(s, job, nidx);
        return;
    }
    s.packed = false;
    reserve(s, n, job.d_indices ? 0 : nidx, stage && !job.d_indices);
    count(Counter::RawChunks);
    s.busy = true;  // (see enqueue_packed)
    // row_ptr always goes through the slot's pinned mirror (small)
    std::memcpy(s.h_rp, job.row_ptr, (n + 1) * sizeof(uint64_t));
    h2d(s.d_rp, s.h_rp, (n + 1) * sizeof(uint64_t), s.st);
    const uint32_t* src = job.indices;
    if (stage && nidx && !job.d_indices) {
        host_memcpy(s.h_idx, job.indices, nidx * sizeof(uint32_t));
        src = s.h_idx;
    }
    if (nidx && !job.d_indices)
        h2d(s.d_idx, src, nidx * sizeof(uint32_t), s.st);
    BBMH_CUDA(cudaMemsetAsync(s.d_err, 0, sizeof(int), s.st));
    if (timed_) BBMH_CUDA(cudaEventRecord(s.ev0, s.st));
    launch_sketch(df_->kf, s.d_rp, job.index_base, job.d_indices ? job.d_indices : s.d_idx, n, b_, s.d_codes,
                  want_minima_ ? s.d_min : nullptr, s.d_flags, s.d_err, s.st,
                  n ? double(nidx) / double(n) : 0.0);
    BBMH_CUDA(cudaGetLastError());
    if (d_w_) {  // fused scoring on the device-resident codes (score.cu)
        BBMH_CUDA(cudaMemsetAsync(s.d_bad, 0xff, sizeof(unsigned long long), s.st));
        launch_score(s.d_codes, s.d_flags, n, f_.k, b_, d_w_, wdim_, s.d_scores, s.d_bad, s.st);
        BBMH_CUDA(cudaGetLastError());
        d2h(s.h_scores, s.d_scores, n * sizeof(double), s.st);
        d2h(s.h_bad, s.d_bad, sizeof(unsigned long long), s.st);
    }
    if (timed_) BBMH_CUDA(cudaEventRecord(s.ev1, s.st));
    if (n && cb_)
        d2h(s.h_codes, s.d_codes, n * cb_, s.st);
    if (want_minima_)
        d2h(s.h_min, s.d_min, n * f_.k * sizeof(uint64_t), s.st);
    d2h(s.h_flags, s.d_flags, n, s.st);
    d2h(s.h_err, s.d_err, sizeof(int), s.st);
    BBMH_CUDA(cudaEventRecord(s.done, s.st));
    s.busy = true;
}

ChunkResult Lane::finish(Slot& s) {
    BBMH_CUDA(cudaEventSynchronize(s.done));
    trace("lane: chunk done");
    s.busy = false;
    int herr;
    unsigned long long hbad = ~0ull;
    ChunkResult r;
    r.tag = s.job.tag;
    r.n = s.job.n;
    if (s.packed) {
        std::memcpy(&herr, s.h_blk + s.off_err, sizeof(int));
        std::memcpy(&hbad, s.h_blk + s.off_err + 8, sizeof(hbad));
        r.codes = s.job.codes_out ? s.job.codes_out : s.h_blk + s.off_codes;
        r.minima = nullptr;
        r.flags = s.h_blk + s.off_flags;
        r.scores = d_w_ ? reinterpret_cast<const double*>(s.h_blk + s.off_scores) : nullptr;
    } else {
        herr = *s.h_err;
        if (d_w_) hbad = *s.h_bad;
        r.codes = s.h_codes;
        r.minima = want_minima_ ? s.h_min : nullptr;
        r.flags = s.h_flags;
        r.scores = d_w_ ? s.h_scores : nullptr;
    }
    if (herr & 1)
        fail(Errc::InvalidArgument, "feature id out of range for the permutation universe");
    if (herr & 2) fail(Errc::InvalidArgument, "row_ptr must be non-decreasing");
    if (d_w_) {
        if (hbad != ~0ull) {  // predict_score (learner.cpp:515-517), first offender in order
            const uint64_t row = hbad >> 24;
            const uint32_t j = uint32_t(hbad & 0xffffff);
            const uint8_t* c = r.codes + row * cb_;
            uint32_t code = 0;
            for (uint32_t i = 0; i < b_; ++i) {
                const uint64_t pos = uint64_t(j) * b_ + i;
                code |= uint32_t((c[pos >> 3] >> (pos & 7)) & 1u) << i;
            }
            const uint32_t idx = uint32_t((uint64_t(j) << b_) + code);
            fail(Errc::DimensionExceeded,
                 "feature " + std::to_string(idx) + " >= dim " + std::to_string(wdim_));
        }
    }
    if (timed_) cudaEventElapsedTime(&r.kernel_ms, s.ev0, s.ev1);
    return r;
}

// ---- small pinned batches: zero-copy --------------------------------------
namespace {

// Zero-copy pays where the fixed per-call costs (H2D/D2H API calls) dominate:
// 2U batches up to ~500 webspam rows. Larger batches overlap chunk copies with
// kernels and the output memcpy in the chunked path (tools/zerocopy_probe.py,
// profiles/r10/zerocopy.jsonl); 4U is kernel-bound at every batch size.
constexpr uint64_t kZeroCopyMaxIds = 2ull << 20;

// Device address of page-locked host memory (UVA mapping), or null.
const void* mapped_device_ptr(const void* p) {
    if (!p) return nullptr;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// The kernel reads the caller's page-locked ids straight over PCIe (the TMA
// bulk copies take host addresses; repeated reads hit L2) and stores codes and
// flags into the slot's mapped pinned block, so a call is one launch and one
// synchronisation, with no H2D/D2H API calls and no staging copy of the ids.
// For small online batches those fixed costs dominate (profiles/r10: 2U k=500,
// batch 64: 79 -> 74 us; batch 256: 161 -> 131 us through the host API).
bool sketch_rows_zero_copy(const Family& f, int dev, const uint64_t* row_ptr,
                           const uint32_t* indices, uint64_t n, uint32_t b, uint8_t* codes,
                           uint8_t* flags) {
    const void* d_ids = mapped_device_ptr(indices);
    if (!d_ids) return false;
    DeviceGuard g(dev);
    const DeviceFamily& df = device_family(f, dev);
    Lane::Slot* s = acquire_slot(dev);
    struct Release {
        Lane::Slot* s;
        ~Release() { release_slot(s); }
    } rel{s};
    const size_t cb = packed_code_bytes(f.k, b);
    const size_t off_flags = align16((n + 1) * sizeof(uint64_t));
    const size_t off_codes = off_flags + n;
    const size_t need = off_codes + n * cb;
    if (need > s->cap_blk) {
        const uint64_t cap = std::max<uint64_t>(need, s->cap_blk + s->cap_blk / 2);
        if (s->d_blk) BBMH_CUDA(cudaFree(s->d_blk));
        if (s->h_blk) BBMH_CUDA(cudaFreeHost(s->h_blk));
        s->d_blk = nullptr;
        s->h_blk = nullptr;
        BBMH_CUDA(cudaMalloc(&s->d_blk, cap));
        BBMH_CUDA(cudaMallocHost(&s->h_blk, cap));
        s->cap_blk = cap;
    }
    uint8_t* h = s->h_blk;  // cudaMallocHost memory: the same address is valid on the device
    std::memcpy(h, row_ptr, (n + 1) * sizeof(uint64_t));
    // err: the kernel only flags permutation ids >= D (not this path) and a
    // decreasing row_ptr (rejected on the host before we get here)
    launch_sketch(df.kf, reinterpret_cast<const uint64_t*>(h), 0,
                  static_cast<const uint32_t*>(d_ids), n, b, h + off_codes, nullptr,
                  h + off_flags, s->d_err, s->st, n ? double(row_ptr[n] - row_ptr[0]) / double(n) : 0.0);
    BBMH_CUDA(cudaGetLastError());
    BBMH_CUDA(cudaStreamSynchronize(s->st));
    count_transfer((n + 1) * sizeof(uint64_t) + (row_ptr[n] - row_ptr[0]) * sizeof(uint32_t), n + n * cb);
    count(Counter::ZeroCopyCalls);
    if (codes) std::memcpy(codes, h + off_codes, n * cb);
    if (flags) std::memcpy(flags, h + off_flags, n);
    return true;
}

}  // namespace

// ---- host-buffer CSR entry -------------------------------------------------
void sketch_rows_host(const Family& f, const uint64_t* row_ptr, const uint32_t* indices,
                      uint64_t n, uint32_t b, uint8_t* codes, uint64_t* minima, uint8_t* flags,
                      const ScoreModel* score, double* scores) {
    if (n == 0) return;
    check_row_ptr(row_ptr, n);
    const size_t cb = packed_code_bytes(f.k, b);
    const bool pinned = is_pinned(indices);
    // (zero-copy reads the caller's buffer in whole 16-byte granules: only
    // when the first id starts one and the last id ends one, so nothing
    // outside the caller's data is touched)
    if (opt(Opt::ZeroCopy) && pinned && !minima && !score && f.scheme == Scheme::TwoU &&
        row_ptr[n] - row_ptr[0] <= kZeroCopyMaxIds &&
        ((uintptr_t)(indices + row_ptr[0]) & 15) == 0 &&
        ((uintptr_t)(indices + row_ptr[n]) & 15) == 0) {
        const std::vector<int> devs = pipeline_devices();
        if (devs.size() == 1 && sketch_rows_zero_copy(f, devs[0], row_ptr, indices, n, b, codes, flags))
            return;
    }

    // Mixing transfers: encoded chunks cost 8 B of host DRAM traffic per id
    // and 2 B of PCIe, raw ones 4 B of each. With the encode bound by host
    // DRAM and the link idle half the time, sending some chunks raw moves
    // more ids per second than either alone.
    // a page-locked output buffer takes the codes' D2H directly
    const bool codes_pinned = codes && !minima && is_pinned(codes) && is_pinned(codes + n * cb - 1);
    // chunk boundaries: <= chunk_docs rows, <= kChunkIdxCap ids (unless one row is larger)
    uint64_t cap_docs = chunk_docs_setting();
    if (minima) cap_docs = std::max<uint64_t>(1, std::min<uint64_t>(cap_docs, kChunkMinimaBytes / (8ull * f.k)));
    // A batch that is one chunk serialises H2D -> kernel -> D2H; splitting a
    // mid-sized batch into ~4 chunks (>= kMinSplitIds ids each) lets the
    // slots' streams overlap one chunk's copy with another's kernel.
    const uint64_t total_ids = row_ptr[n] - row_ptr[0];
    const uint64_t idx_cap =
        std::min<uint64_t>(chunk_idx_cap(), std::max<uint64_t>(kMinSplitIds, total_ids / 4));
    std::vector<uint64_t> bounds{0};
    for (uint64_t r = 0; r < n;) {
        uint64_t e = r + 1;
        while (e < n && e - r < cap_docs && row_ptr[e + 1] - row_ptr[r] <= idx_cap) ++e;
        bounds.push_back(e);
        r = e;
    }
    const uint64_t nchunks = bounds.size() - 1;
    const std::vector<int> devs = pipeline_devices();
    // GPUs fed from this host (lanes here times the processes of the job
    // that share it) split its DRAM and cores
    const uint64_t feeds = devs.size() * uint64_t(std::max<int64_t>(1, opt(Opt::HostSharers)));
    const int64_t raw_opt = opt(Opt::DeltaRawEvery);
    const uint64_t raw_every = raw_opt >= 0 ? uint64_t(raw_opt) : mixed_raw_every(feeds, nullptr);
    std::atomic<uint64_t> next{0};
    std::mutex err_mu;
    std::exception_ptr err;
    std::atomic<bool> abort{false};

    auto run_device = [&](int dev) {
        try {
            Lane lane(f, dev, b, minima != nullptr, score);
            lane.set_timed(false);
            // GPUs fed from this host (lanes here times the processes of the
            // job that share it) split its DRAM and cores: the 16-bit transfer
            // is used only where that budget says it moves ids faster.
            lane.set_delta16(delta16_budget_pays(feeds, nullptr, nullptr));
            auto done = [&](const ChunkResult& res) {
                const uint64_t r0 = bounds[res.tag];
                if (codes && res.codes != codes + r0 * cb) host_memcpy(codes + r0 * cb, res.codes, res.n * cb);
                if (scores) std::memcpy(scores + r0, res.scores, res.n * sizeof(double));
                if (minima) host_memcpy(minima + r0 * f.k, res.minima, res.n * f.k * 8);
                if (flags) std::memcpy(flags + r0, res.flags, res.n);
                trace("host: chunk copied out");
            };
            for (uint64_t c; !abort.load() && (c = next.fetch_add(1)) < nchunks;) {
                ChunkJob job;
                job.tag = c;
                job.row_ptr = row_ptr + bounds[c];
                job.index_base = row_ptr[bounds[c]];
                job.indices = indices + row_ptr[bounds[c]];
                job.n = bounds[c + 1] - bounds[c];
                job.pinned_input = pinned;
                if (codes_pinned) job.codes_out = codes + bounds[c] * cb;
                // every raw_every-th chunk crosses as 4-byte ids: its DMA needs
                // no host cores and runs while the others are encoded
                job.ids_as_is = raw_every && c % raw_every == raw_every - 1;
                lane.submit(job, done);
            }
            lane.drain(done);
        } catch (...) {
            std::lock_guard lk(err_mu);
            if (!err) err = std::current_exception();
            abort = true;
        }
    };
    if (devs.size() == 1) {
        run_device(devs[0]);
    } else {
        std::vector<std::thread> ts;
        for (int d : devs) ts.emplace_back(run_device, d);
        for (auto& t : ts) t.join();
    }
    if (err) std::rethrow_exception(err);
}

void sketch_rows_device(const Family& f, const uint64_t* d_row_ptr, uint64_t index_base,
                        const uint32_t* d_indices, uint64_t n, uint32_t b, uint8_t* d_codes,
                        uint64_t* d_minima, uint8_t* d_flags, cudaStream_t stream) {
    if (n == 0) return;
    int dev = 0;
    BBMH_CUDA(cudaGetDevice(&dev));
    const DeviceFamily& df = device_family(f, dev);
    // per-device scratch error word (the async API does not report it; ids
    // out of range in permutation mode are clamped to 0 inside the kernel)
    static std::mutex mu;
    static std::vector<int*> errs;
    int* d_err;
    {
        std::lock_guard lk(mu);
        if (size_t(dev) >= errs.size()) errs.resize(dev + 1, nullptr);
        if (!errs[dev]) BBMH_CUDA(cudaMalloc(&errs[dev], sizeof(int)));
        d_err = errs[dev];
    }
    launch_sketch(df.kf, d_row_ptr, index_base, d_indices, n, b, d_codes, d_minima, d_flags, d_err,
                  stream);
    BBMH_CUDA(cudaGetLastError());
}

}  // namespace bbmh
