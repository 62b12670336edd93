// delta.hpp -- 2-byte transfer encoding of CSR ids for the host->device copy.
//
// From host buffers the 2U path is bound by the PCIe H2D copy of the ids
// (4 B per id at ~55 GB/s) for every k up to ~1,000; the kernel alone would
// take twice the ids per second. Ids within a row are sorted, so consecutive
// differences are small (mean D/nnz, ~4,500 at the webspam shape). Each id
// therefore travels as the 16-bit difference to the previous id of its row
// (the first id: to 0). A difference of 0 or >= 2^16 is sent as 0 (escape)
// and its 32-bit value goes to a side list, in order. The device rebuilds the
// ids with a per-row prefix sum (decode_delta16_kernel) into the buffer the
// sketch kernel reads. Differences are taken and summed mod 2^32, so the
// round trip is exact for any u32 input; unsorted or repeated ids only escape.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bbmh {

// Encodes the chunk's ids: rows r in [0, n) hold ids[row_ptr[r] - base,
// row_ptr[r+1] - base). Writes deltas[i] for every id, exc_ptr[r] (escapes
// before row r, n + 1 entries) and the escaped differences to exc. Uses the
// host pool. Returns false, with `exc` partly written, if there are more than
// exc_cap escapes (the caller then sends the ids as they are).
bool encode_delta16(const uint64_t* row_ptr, uint64_t n, uint64_t base, const uint32_t* ids,
                    uint16_t* deltas, uint32_t* exc_ptr, uint32_t* exc, uint64_t exc_cap,
                    uint64_t& nexc);

// Whether the encoding pays for a chunk: ids that are sorted and dense enough
// that nearly all differences fit 16 bits (estimated from a few rows).
bool delta16_worthwhile(const uint64_t* row_ptr, uint64_t n, uint64_t base, const uint32_t* ids);

// Device side: ids[row_ptr[r] - base + i] for every row (one warp per row).
void launch_decode_delta16(const uint64_t* row_ptr, uint64_t base, uint64_t n,
                           const uint16_t* deltas, const uint32_t* exc_ptr, const uint32_t* exc,
                           uint32_t* ids, cudaStream_t stream);

}  // namespace bbmh
