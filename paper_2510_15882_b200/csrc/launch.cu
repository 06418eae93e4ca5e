// Template dispatch for the data-plane kernels (see kernels.cuh).
#include <algorithm>
#include <atomic>

#include "internal.h"
#include "kernels.cuh"
#include "rank_launch.h"  // opt_in_dyn_smem

namespace flx {

std::atomic<unsigned long long> g_launches{0};

namespace {

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename T, int OP, int NMAX>
cudaError_t fold_vec(const FoldArgs& a, int grid, cudaStream_t s) {
  constexpr int kUnroll = NMAX <= 4 ? 2 : 1;
  fold_vec_kernel<T, OP, NMAX, kUnroll><<<grid, 512, 0, s>>>(a);
  return cudaGetLastError();
}

// FLX_TMA=1 selects the bulk-copy (cp.async.bulk + mbarrier) variants.  Off
// by default: with one 16 B vector per thread over a large grid the LDG
// kernels measure 1.04x (fold) and 0.95x (fan-out) of the copy peak, the TMA
// ones 0.91x / 0.84x (profiles/r1/*variants*.jsonl).
int tma_mode() {
  static const int mode = getenv("FLX_TMA") ? atoi(getenv("FLX_TMA")) : 0;
  return mode;
}
bool use_tma_fold() { return tma_mode() == 1; }
bool use_tma_fanout() { return tma_mode() == 1; }

template <typename T, int OP, int NMAX>
cudaError_t fold_tma(const FoldArgs& a, int grid, cudaStream_t s) {
  constexpr size_t smem = tma_fold_smem<NMAX>();
  static std::atomic<uint64_t> opted{0};  // per device: cliques may span several
  opt_in_dyn_smem(opted, {(const void*)fold_tma_kernel<T, OP, NMAX>}, (int)smem);
  fold_tma_kernel<T, OP, NMAX><<<grid, kTmaThreads, smem, s>>>(a);
  return cudaGetLastError();
}

template <typename T, int OP>
cudaError_t fold_typed(const FoldArgs& a, int grid, cudaStream_t s) {
  bool vec = true;
  for (int r = 0; r < a.n; ++r) vec = vec && aligned16(a.src[r]);
  for (int d = 0; d < a.ndst; ++d) vec = vec && aligned16(a.dst[d]);
  if (!vec) {
    fold_scalar_kernel<T, OP><<<grid, 512, 0, s>>>(a);
    return cudaGetLastError();
  }
  if (use_tma_fold() && a.n <= 8 && a.ndst <= kMaxRanks) {
    if (a.n <= 4) return fold_tma<T, OP, 4>(a, grid, s);
    return fold_tma<T, OP, 8>(a, grid, s);
  }
  const size_t nvec = a.bytes >> 4;
  if ((size_t)grid * 512 >= nvec) {  // uncapped: single pass, one vector per thread
    // (the grid covers nvec + 16 threads: the ragged tail's elements)
    // 1024-thread CTAs for up to 8 ranks of 2- and 4-byte types (64-bit and
    // 1-byte ones would spill under the 64-register cap of a 1024-thread CTA)
    constexpr int kT = (sizeof(T) == 2 || sizeof(T) == 4) ? 1024 : 512;
    const int width = a.n > a.ndst ? a.n : a.ndst;
    const int once = (int)((nvec + 16 + kT - 1) / kT);
    if (width <= 2) fold_once_kernel<T, OP, 2, kT><<<once, kT, 0, s>>>(a);
    else if (width <= 4) fold_once_kernel<T, OP, 4, kT><<<once, kT, 0, s>>>(a);
    else if (width <= 8) fold_once_kernel<T, OP, 8, kT><<<once, kT, 0, s>>>(a);
    else fold_once_kernel<T, OP, 16><<<(int)((nvec + 16 + 511) / 512), 512, 0, s>>>(a);
    return cudaGetLastError();
  }
  const int width = a.n > a.ndst ? a.n : a.ndst;
  if (width <= 2) return fold_vec<T, OP, 2>(a, grid, s);
  if (width <= 4) return fold_vec<T, OP, 4>(a, grid, s);
  if (width <= 8) return fold_vec<T, OP, 8>(a, grid, s);
  return fold_vec<T, OP, 16>(a, grid, s);
}

template <typename T>
cudaError_t fold_op(int op, const FoldArgs& a, int grid, cudaStream_t s) {
  switch (op) {
    case kSum: return fold_typed<T, kSum>(a, grid, s);
    case kProd: return fold_typed<T, kProd>(a, grid, s);
    case kMax: return fold_typed<T, kMax>(a, grid, s);
    case kMin: return fold_typed<T, kMin>(a, grid, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_fold(int dtype, int op, const FoldArgs& a, int grid, cudaStream_t s) {
  if (a.bytes == 0) return cudaSuccess;
  if (a.n < 1 || a.n > kMaxRanks || a.ndst < 1 || a.ndst > kMaxRanks || grid < 1)
    return cudaErrorInvalidValue;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  switch (dtype) {
    case flxInt8: return fold_op<int8_t>(op, a, grid, s);
    case flxUint8: return fold_op<uint8_t>(op, a, grid, s);
    case flxInt32: return fold_op<int32_t>(op, a, grid, s);
    case flxUint32: return fold_op<uint32_t>(op, a, grid, s);
    case flxInt64: return fold_op<int64_t>(op, a, grid, s);
    case flxUint64: return fold_op<uint64_t>(op, a, grid, s);
    case flxFloat16: return fold_op<__half>(op, a, grid, s);
    case flxFloat32: return fold_op<float>(op, a, grid, s);
    case flxFloat64: return fold_op<double>(op, a, grid, s);
    case flxBfloat16: return fold_op<__nv_bfloat16>(op, a, grid, s);
  }
  return cudaErrorInvalidValue;
}

namespace {

template <typename T, int OP>
cudaError_t rows_typed(const RowsArgs& a, int grid, cudaStream_t s) {
  bool vec = (a.src_stride & 15) == 0;
  for (int r = 0; r < a.n; ++r) vec = vec && aligned16(a.src[r]);
  for (int d = 0; d < a.nrows; ++d) vec = vec && aligned16(a.dst[d]);
  const dim3 g(grid, a.nrows);
  if (!vec)
    rows_scalar_kernel<T, OP><<<g, 512, 0, s>>>(a);
  else if (a.n <= 2)
    rows_vec_kernel<T, OP, 2><<<g, 512, 0, s>>>(a);
  else if (a.n <= 4)
    rows_vec_kernel<T, OP, 4><<<g, 512, 0, s>>>(a);
  else if (a.n <= 8)
    rows_vec_kernel<T, OP, 8><<<g, 512, 0, s>>>(a);
  else
    rows_vec_kernel<T, OP, 16><<<g, 512, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename T>
cudaError_t rows_op(int op, const RowsArgs& a, int grid, cudaStream_t s) {
  switch (op) {
    case kSum: return rows_typed<T, kSum>(a, grid, s);
    case kProd: return rows_typed<T, kProd>(a, grid, s);
    case kMax: return rows_typed<T, kMax>(a, grid, s);
    case kMin: return rows_typed<T, kMin>(a, grid, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_rows(int dtype, int op, const RowsArgs& a, int grid, cudaStream_t s) {
  if (a.bytes == 0) return cudaSuccess;
  if (a.n < 1 || a.n > kMaxRanks || a.nrows < 1 || a.nrows > kMaxRanks || grid < 1)
    return cudaErrorInvalidValue;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  switch (dtype) {
    case flxInt8: return rows_op<int8_t>(op, a, grid, s);
    case flxUint8: return rows_op<uint8_t>(op, a, grid, s);
    case flxInt32: return rows_op<int32_t>(op, a, grid, s);
    case flxUint32: return rows_op<uint32_t>(op, a, grid, s);
    case flxInt64: return rows_op<int64_t>(op, a, grid, s);
    case flxUint64: return rows_op<uint64_t>(op, a, grid, s);
    case flxFloat16: return rows_op<__half>(op, a, grid, s);
    case flxFloat32: return rows_op<float>(op, a, grid, s);
    case flxFloat64: return rows_op<double>(op, a, grid, s);
    case flxBfloat16: return rows_op<__nv_bfloat16>(op, a, grid, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_xpose(const XposeArgs& a, int grid, cudaStream_t s) {
  if (a.bytes == 0) return cudaSuccess;
  if (a.n < 1 || a.n > kMaxRanks || grid < 1) return cudaErrorInvalidValue;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  bool vec = (a.src_stride & 15) == 0 && (a.dst_stride & 15) == 0;
  for (int r = 0; r < a.n; ++r) vec = vec && aligned16(a.src[r]) && aligned16(a.dst[r]);
  const size_t need = ((a.bytes >> 4) + 2047) / 2048;  // single pass (4 vectors/thread)
  const unsigned gx = (unsigned)std::min<size_t>(std::max<size_t>(1, need), (size_t)grid);
  xpose_kernel<<<dim3(gx, a.n * a.n), 512, 0, s>>>(a, vec ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_fanout(const FanoutArgs& a, int grid, cudaStream_t s) {
  if (a.bytes == 0) return cudaSuccess;
  if (a.nsrc < 1 || a.nsrc > kMaxRanks || a.ndst < 1 || a.ndst > kMaxRanks || grid < 1)
    return cudaErrorInvalidValue;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  bool bases = true;  // every source and destination base 16 B aligned
  for (int r = 0; r < a.nsrc; ++r) bases = bases && aligned16(a.src[r]);
  for (int d = 0; d < a.ndst; ++d) bases = bases && aligned16(a.dst[d]);
  const bool vec = bases && (a.dst_stride & 15) == 0;
  const dim3 g(grid, a.nsrc);
  if (bases && !vec) {  // ragged per-rank blocks: aligned stores, funnel-shifted loads
    const unsigned bx = (unsigned)std::min<size_t>(((a.bytes >> 4) + 511) / 512 + 1, (size_t)grid);
    const dim3 gs(std::max(1u, bx), a.nsrc);
    // (a two-CTA destination split as in fanout_once measured slower here)
    if (a.ndst <= 2) fanout_shift_kernel<2, 1><<<gs, 512, 0, s>>>(a);
    else if (a.ndst <= 4) fanout_shift_kernel<4, 1><<<gs, 512, 0, s>>>(a);
    else if (a.ndst <= 8) fanout_shift_kernel<8, 1><<<gs, 512, 0, s>>>(a);
    else fanout_shift_kernel<16, 1><<<gs, 512, 0, s>>>(a);
    return cudaGetLastError();
  }
  if (vec && use_tma_fanout()) {
    constexpr size_t smem = (size_t)kTmaStages * kTmaTile * 4 + kTmaStages * sizeof(uint64_t);
    static std::atomic<uint64_t> opted{0};  // per device: cliques may span several
    opt_in_dyn_smem(opted, {(const void*)fanout_tma_kernel}, (int)smem);
    fanout_tma_kernel<<<dim3(grid * 3, a.nsrc), 32, smem, s>>>(a);
  } else if (!vec) {
    fanout_byte_kernel<<<g, 512, 0, s>>>(a);
  } else if ((size_t)grid * 512 >= (a.bytes >> 4)) {  // uncapped: single pass
    const unsigned bx = (unsigned)(((a.bytes >> 4) + 16 + 511) / 512);
    const dim3 once(bx, a.nsrc), twice(2 * bx, a.nsrc);
    if (a.ndst <= 2) fanout_once_kernel<2, 1><<<once, 512, 0, s>>>(a);
    else if (a.ndst <= 4) fanout_once_kernel<4, 2><<<twice, 512, 0, s>>>(a);
    else if (a.ndst <= 8) fanout_once_kernel<8, 2><<<twice, 512, 0, s>>>(a);
    else fanout_once_kernel<16, 2><<<twice, 512, 0, s>>>(a);
  } else if (a.ndst <= 2) {
    fanout_vec_kernel<2, 1><<<g, 512, 0, s>>>(a);
  } else if (a.ndst <= 4) {
    // UNR 1: one vector per thread per pass keeps registers low (the unrolled
    // <8,2> build needed 76, one CTA/SM, and ran 24% slower on the big grid)
    fanout_vec_kernel<4, 1><<<g, 512, 0, s>>>(a);
  } else if (a.ndst <= 8) {
    fanout_vec_kernel<8, 1><<<g, 512, 0, s>>>(a);
  } else {
    fanout_vec_kernel<16, 1><<<g, 512, 0, s>>>(a);
  }
  return cudaGetLastError();
}

// ncclAvg's second half: buf[i] = buf[i] / n on the caller's stream
// (accumulation type for 16-bit floats, C division for integers)
template <typename T>
__global__ void __launch_bounds__(512) div_kernel(T* buf, size_t count, int n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    using A = typename AccT<T>::type;
    buf[i] = from_acc<T>(to_acc<T>(buf[i]) / (A)n);
  }
}

template <typename T>
cudaError_t div_typed(void* buf, size_t count, int n, cudaStream_t s) {
  const int grid = (int)std::min<size_t>((count + 511) / 512, 148 * 8);
  div_kernel<T><<<std::max(grid, 1), 512, 0, s>>>(static_cast<T*>(buf), count, n);
  g_launches++;
  return cudaGetLastError();
}

cudaError_t launch_div(int dtype, void* buf, size_t count, int n, cudaStream_t s) {
  if (count == 0 || n == 1) return cudaSuccess;
  switch (dtype) {
    case flxInt8: return div_typed<int8_t>(buf, count, n, s);
    case flxUint8: return div_typed<uint8_t>(buf, count, n, s);
    case flxInt32: return div_typed<int32_t>(buf, count, n, s);
    case flxUint32: return div_typed<uint32_t>(buf, count, n, s);
    case flxInt64: return div_typed<int64_t>(buf, count, n, s);
    case flxUint64: return div_typed<uint64_t>(buf, count, n, s);
    case flxFloat16: return div_typed<__half>(buf, count, n, s);
    case flxFloat32: return div_typed<float>(buf, count, n, s);
    case flxFloat64: return div_typed<double>(buf, count, n, s);
    case flxBfloat16: return div_typed<__nv_bfloat16>(buf, count, n, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t preload_launch_cu() {
  return preload_module((const void*)fold_once_kernel<float, kSum, 8, 1024>);
}

}  // namespace flx
