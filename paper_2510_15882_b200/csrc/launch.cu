// Template dispatch for the data-plane kernels (see kernels.cuh).
#include <atomic>

#include "internal.h"
#include "kernels.cuh"

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

template <typename T, int OP>
cudaError_t fold_typed(const FoldArgs& a, int grid, cudaStream_t s) {
  bool vec = true;
  for (int r = 0; r < a.n; ++r) vec = vec && aligned16(a.src[r]);
  for (int d = 0; d < a.ndst; ++d) vec = vec && aligned16(a.dst[d]);
  if (!vec) {
    fold_scalar_kernel<T, OP><<<grid, 512, 0, s>>>(a);
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

cudaError_t launch_fanout(const FanoutArgs& a, int grid, cudaStream_t s) {
  if (a.bytes == 0) return cudaSuccess;
  if (a.nsrc < 1 || a.nsrc > kMaxRanks || a.ndst < 1 || a.ndst > kMaxRanks || grid < 1)
    return cudaErrorInvalidValue;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  bool vec = (a.dst_stride & 15) == 0;
  for (int r = 0; r < a.nsrc; ++r) vec = vec && aligned16(a.src[r]);
  for (int d = 0; d < a.ndst; ++d) vec = vec && aligned16(a.dst[d]);
  const dim3 g(grid, a.nsrc);
  if (!vec) {
    fanout_byte_kernel<<<g, 512, 0, s>>>(a);
  } else if (a.ndst <= 2) {
    fanout_vec_kernel<2, 2><<<g, 512, 0, s>>>(a);
  } else if (a.ndst <= 4) {
    fanout_vec_kernel<4, 2><<<g, 512, 0, s>>>(a);
  } else if (a.ndst <= 8) {
    fanout_vec_kernel<8, 2><<<g, 512, 0, s>>>(a);
  } else {
    fanout_vec_kernel<16, 1><<<g, 512, 0, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace flx
