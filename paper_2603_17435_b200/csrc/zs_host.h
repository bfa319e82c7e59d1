// zs_host.h -- host helpers shared by the host encoder and the GPU encoder's driver code
// (internal to libzs.so; not part of the C ABI).
#pragma once
#include <cstdint>

#include "../../include/zs.h"

namespace zs {
// Alg. 1 line 3: start of the max-coverage window of 7 consecutive exponents (ties -> the
// smallest start); covered = elements inside it.
int window_start(const int64_t hist[256], int64_t* covered);
// Sizes of the encoding and the offsets array (n_blocktiles + 1 pairs, 16-B padded segments)
// from the per-BlockTile in-window counts (padding elements count as in-window).
void sizes_and_offsets(int64_t rows, int64_t cols, const uint32_t* hcnt, zs_sizes* s, uint64_t* offsets);
}  // namespace zs
