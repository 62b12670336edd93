// options.hpp -- the library's tuning and test switches, in one table.
//
// The reference reads no environment variables. Here every
// switch has a default that is what the product runs; a process may override
// one with bbmh_ext_set_option(name, value) at any time (tests and tools do),
// and, for developer A/B runs, with BBMH_OPT_<NAME> in the environment, which
// is read once, when the table is first used. Nothing reads the environment
// on a launch or chunk path.
#pragma once

#include <cstdint>

namespace bbmh {

enum class Opt : int {
    Tile,           // ids per staged sketch item (0: per-shape default)
    SmemCap,        // cap one-warp wide-J 2U CTAs at 20 per SM (1) or not (0)
    CtasPerSm,      // cap on resident sketch CTAs per SM (0: occupancy limit)
    ShapeJ,         // force J functions per thread (0: choose_shape)
    ShapeTpb,       // force threads per CTA (0: choose_shape)
    Carveout,       // shared-memory carveout % for the sketch kernels (-1: driver default)
    DynamicDocs,    // small-k sketch kernel takes documents from a ticket counter (1) or round-robin (0)
    SplitSmallK,    // small-k lane-split kernel (1) or the persistent kernel (0)
    Uniform2U,      // 2U with 16 < k <= 544: coefficient-uniform kernel by row length (1), always (2), never (0)
    UniformSbDocs,  // uniform kernels: documents per super-block (0: 58 MB of ids, >= 3,072)
    Uniform4U,      // 4U-bit with 16 < k <= 1024: coefficient-uniform kernel by the persistent shape (1), always (2), never (0)
    PermTablewise,  // permutation schedule: -1 auto, 0 document-outer, 1 table-outer
    PermScratchMb,  // table-outer schedule: device scratch budget per pass group (MiB)
    GpuPermgen,     // build large permutation tables on the GPU (1) or the host (0)
    ForcePeerCopy,  // replicate device-built tables with cudaMemcpyPeer even on the same device
    GpuParse,       // parse LibSVM text on the GPU (1) or on host cores only (0)
    GpuParseBlock,  // GPU parser block size in bytes (0: default)
    ParsePriority,  // GPU parser streams at the device's highest stream priority (1) or default (0)
    DeviceIds,      // keep parsed ids on the parsing GPU (1) or go through the host (0)
    RangeShards,    // text ranges per lane for multi-lane LibSVM files (0: shared reader)
    TextLanes,      // loader lanes for LibSVM text files in all (at least one per GPU)
    ReadThreads,    // pread threads per text block
    Delta16,        // 16-bit id transfer: -1 where it pays, 0 never, 1 whenever possible
    DeltaRawEvery,  // every n-th chunk crosses as 4-byte ids (0: none, -1: from the host budget)
    HostSharers,    // GPU feeds sharing this host's DRAM, e.g. ranks per node (>= 1)
    HostDramGbs,    // host DRAM copy bandwidth, read + write GB/s (0: measure on first use)
    PcieGbs,        // host -> device link bandwidth per GPU, GB/s
    ZeroCopy,       // small pinned 2U batches read over the link without staging copies
    ChunkIds,       // ids per host-pipeline chunk (0: default)
    Trace,          // stage tracing to stderr
    kCount
};

int64_t opt(Opt o);
// false if `name` is unknown; `value` is stored as given (consumers clamp)
bool set_opt(const char* name, int64_t value);
bool get_opt(const char* name, int64_t* value);
// names in table order, for listing ("" past the end)
const char* opt_name(int i);

}  // namespace bbmh
