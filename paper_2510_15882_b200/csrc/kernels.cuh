// Device side of the FlexLink data plane (sm_100a).
//
// All collective arithmetic funnels through ONE fold rule so that every path
// (NVLink kernel, PCIe reduce-on-receive, real or virtual ranks) produces the
// same bits: for each element, acc = x[0]; acc = op(acc, x[r]) for r = 1..N-1
// in rank order, accumulated in AccT<T> (fp32 for fp16/bf16, the native type
// otherwise, integers wrapping), rounded once to T.  oracle/flx_oracle.c
// restates exactly this rule on the CPU.
//
// The kernels are HBM/link-bound streaming loops: 128-bit vector loads on the
// non-coherent path with L1 no-allocate, all N sources in flight before the
// fold, 128-bit stores, grid sized to the SM count.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <type_traits>

#include "args.h"

namespace flx {


// ---------------------------------------------------------------- numerics
template <typename T> struct AccT { using type = T; };
template <> struct AccT<__half> { using type = float; };
template <> struct AccT<__nv_bfloat16> { using type = float; };

template <typename T>
__device__ __forceinline__ typename AccT<T>::type to_acc(T v) { return v; }
template <>
__device__ __forceinline__ float to_acc<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_acc<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}

template <typename T>
__device__ __forceinline__ T from_acc(typename AccT<T>::type v) { return v; }
template <>
__device__ __forceinline__ __half from_acc<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// Binary operator on the accumulator type.  Integers wrap (computed in the
// unsigned twin so signed overflow is defined); max/min are plain compares so
// the result for NaN / signed zero is a fixed function of the fold order.
template <int OP, typename A>
__device__ __forceinline__ A apply_op(A a, A b) {
  if constexpr (std::is_integral<A>::value) {
    using U = typename std::make_unsigned<A>::type;
    if constexpr (OP == kSum) return (A)(U)((U)a + (U)b);
    if constexpr (OP == kProd) return (A)(U)((U)a * (U)b);
  } else {
    if constexpr (OP == kSum) return a + b;
    if constexpr (OP == kProd) return a * b;
  }
  if constexpr (OP == kMax) return (b > a) ? b : a;
  if constexpr (OP == kMin) return (b < a) ? b : a;
}

// ------------------------------------------------------------- memory ops
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

template <typename T, int OP>
__device__ __forceinline__ void fold_into(typename AccT<T>::type* acc, const uint4& word) {
  constexpr int kVec = 16 / sizeof(T);
  const T* x = reinterpret_cast<const T*>(&word);
#pragma unroll
  for (int j = 0; j < kVec; ++j) acc[j] = apply_op<OP>(acc[j], to_acc<T>(x[j]));
}

template <typename T>
__device__ __forceinline__ void load_acc(typename AccT<T>::type* acc, const uint4& word) {
  constexpr int kVec = 16 / sizeof(T);
  const T* x = reinterpret_cast<const T*>(&word);
#pragma unroll
  for (int j = 0; j < kVec; ++j) acc[j] = to_acc<T>(x[j]);
}

template <typename T>
__device__ __forceinline__ uint4 pack_acc(const typename AccT<T>::type* acc) {
  constexpr int kVec = 16 / sizeof(T);
  uint4 out;
  T* y = reinterpret_cast<T*>(&out);
#pragma unroll
  for (int j = 0; j < kVec; ++j) y[j] = from_acc<T>(acc[j]);
  return out;
}

// ------------------------------------------------------------ fold kernel
// n sources, ndst destinations, `bytes` per source.  dst[d] = fold(src[0..n)).
// Used for the virtual-rank NVLink slice (n = ndst = N), the PCIe
// reduce-on-receive (src = staged copies), and the real-rank reduce phase.


template <typename T, int OP, int NMAX, int UNR>
__global__ void __launch_bounds__(512) fold_vec_kernel(const FoldArgs a) {
  using A = typename AccT<T>::type;
  constexpr int kVec = 16 / sizeof(T);
  const size_t nvec = a.bytes >> 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;

  for (; v + (UNR - 1) * stride < nvec; v += UNR * stride) {
    uint4 in[UNR][NMAX];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int r = 0; r < NMAX; ++r)
        if (r < a.n) in[u][r] = ld_stream(a.src[r] + ((v + u * stride) << 4));
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      A acc[kVec];
      load_acc<T>(acc, in[u][0]);
#pragma unroll
      for (int r = 1; r < NMAX; ++r)
        if (r < a.n) fold_into<T, OP>(acc, in[u][r]);
      const uint4 out = pack_acc<T>(acc);
#pragma unroll
      for (int d = 0; d < NMAX; ++d)
        if (d < a.ndst) st_stream(a.dst[d] + ((v + u * stride) << 4), out);
    }
  }
  for (; v < nvec; v += stride) {
    uint4 in[NMAX];
#pragma unroll
    for (int r = 0; r < NMAX; ++r)
      if (r < a.n) in[r] = ld_stream(a.src[r] + (v << 4));
    A acc[kVec];
    load_acc<T>(acc, in[0]);
#pragma unroll
    for (int r = 1; r < NMAX; ++r)
      if (r < a.n) fold_into<T, OP>(acc, in[r]);
    const uint4 out = pack_acc<T>(acc);
#pragma unroll
    for (int d = 0; d < NMAX; ++d)
      if (d < a.ndst) st_stream(a.dst[d] + (v << 4), out);
  }
  // ragged tail: fewer than 16 bytes of whole elements
  if (blockIdx.x == 0) {
    const size_t base = nvec << 4;
    const size_t tail = (a.bytes - base) / sizeof(T);
    if (threadIdx.x < tail) {
      const size_t off = base + threadIdx.x * sizeof(T);
      A acc = to_acc<T>(*reinterpret_cast<const T*>(a.src[0] + off));
      for (int r = 1; r < a.n; ++r)
        acc = apply_op<OP>(acc, to_acc<T>(*reinterpret_cast<const T*>(a.src[r] + off)));
      const T out = from_acc<T>(acc);
      for (int d = 0; d < a.ndst; ++d) *reinterpret_cast<T*>(a.dst[d] + off) = out;
    }
  }
  (void)kVec;
}

// Element-at-a-time fallback for buffers that are not 16-byte aligned.
template <typename T, int OP>
__global__ void __launch_bounds__(512) fold_scalar_kernel(const FoldArgs a) {
  using A = typename AccT<T>::type;
  const size_t count = a.bytes / sizeof(T);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    A acc = to_acc<T>(reinterpret_cast<const T*>(a.src[0])[i]);
    for (int r = 1; r < a.n; ++r)
      acc = apply_op<OP>(acc, to_acc<T>(reinterpret_cast<const T*>(a.src[r])[i]));
    const T out = from_acc<T>(acc);
    for (int d = 0; d < a.ndst; ++d) reinterpret_cast<T*>(a.dst[d])[i] = out;
  }
}

// ---------------------------------------------------------- fanout kernel
// AllGather data movement: for every source r (blockIdx.y) copy `bytes` from
// src[r] to dst[d] + r*dst_stride for all d.  Byte-exact by construction.


template <int NMAX, int UNR>
__global__ void __launch_bounds__(512) fanout_vec_kernel(const FanoutArgs a) {
  const int r = blockIdx.y;
  const char* src = a.src[r];
  const size_t shift = (size_t)r * a.dst_stride;
  const size_t nvec = a.bytes >> 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; v + (UNR - 1) * stride < nvec; v += UNR * stride) {
    uint4 w[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) w[u] = ld_stream(src + ((v + u * stride) << 4));
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int d = 0; d < NMAX; ++d)
        if (d < a.ndst) st_stream(a.dst[d] + shift + ((v + u * stride) << 4), w[u]);
  }
  for (; v < nvec; v += stride) {
    const uint4 w = ld_stream(src + (v << 4));
#pragma unroll
    for (int d = 0; d < NMAX; ++d)
      if (d < a.ndst) st_stream(a.dst[d] + shift + (v << 4), w);
  }
  if (blockIdx.x == 0) {
    const size_t base = nvec << 4;
    const size_t i = base + threadIdx.x;
    if (i < a.bytes) {
      const char b = src[i];
      for (int d = 0; d < a.ndst; ++d) a.dst[d][shift + i] = b;
    }
  }
}

static __global__ void __launch_bounds__(512) fanout_byte_kernel(const FanoutArgs a) {
  const int r = blockIdx.y;
  const size_t shift = (size_t)r * a.dst_stride;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.bytes; i += stride) {
    const char b = a.src[r][i];
    for (int d = 0; d < a.ndst; ++d) a.dst[d][shift + i] = b;
  }
}

}  // namespace flx
