// Kernel argument blocks shared by host and device code.
#pragma once

#include <stddef.h>

namespace flx {

constexpr int kMaxRanks = 16;  // FLX_MAX_VIRTUAL_RANKS

enum RedOp { kSum = 0, kProd = 1, kMax = 2, kMin = 3 };

// n sources, ndst destinations, `bytes` per source: dst[d] = fold(src[0..n)).
// Used for the virtual-rank NVLink slice (n = ndst = N), the PCIe
// reduce-on-receive (src = staged copies) and the real-rank reduce phase.
struct FoldArgs {
  const char* src[kMaxRanks];
  char* dst[kMaxRanks];
  int n;
  int ndst;
  size_t bytes;
};

// AllGather data movement: for every source r copy `bytes` from src[r] to
// dst[d] + r*dst_stride for all d.  Byte-exact by construction.
struct FanoutArgs {
  const char* src[kMaxRanks];
  char* dst[kMaxRanks];
  int nsrc;
  int ndst;
  size_t bytes;       // per source
  size_t dst_stride;  // byte distance between consecutive sources' blocks in dst
};

// ReduceScatter rows: row y (blockIdx.y, one per destination rank) folds
// src[0..n) + y*src_stride into dst[y], `bytes` per row.
struct RowsArgs {
  const char* src[kMaxRanks];
  char* dst[kMaxRanks];
  int n;      // sources per row
  int nrows;  // destinations
  size_t bytes;
  size_t src_stride;
};

// AllToAll block transpose: y = r*n + q copies `bytes` from src[r] +
// q*src_stride to dst[q] + r*dst_stride.
struct XposeArgs {
  const char* src[kMaxRanks];
  char* dst[kMaxRanks];
  int n;
  size_t bytes;
  size_t src_stride;
  size_t dst_stride;
};

}  // namespace flx
