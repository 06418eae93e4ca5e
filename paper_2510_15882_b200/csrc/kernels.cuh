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

// The 16 B at p when all of them lie inside the source (avail >= 16); else only
// the first `avail` bytes, loaded one by one, the rest zero — a shifted window's
// last vector must not read past the end of its source buffer.
__device__ __forceinline__ uint4 ld_vec_clamped(const char* p, size_t avail, bool coherent) {
  if (avail >= 16) {
    if (!coherent) return ld_stream(p);
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
  }
  uint32_t w[4] = {0, 0, 0, 0};
  for (size_t i = 0; i < avail; ++i) {
    const uint32_t b = coherent ? (uint8_t)*(volatile const char*)(p + i) : (uint8_t)p[i];
    w[i >> 2] |= b << (8 * (i & 3));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
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

// Single-pass form: exactly one 16 B vector per thread, grid covers the slice.
// No loop-invariant address hoisting, so few registers (high occupancy) and
// CTA turnover instead of a grid-stride tail: the uncapped default.  THREADS =
// 1024 for up to 8 ranks: each CTA streams 16 KiB runs of every source and
// destination, +1.4 % over 512-thread CTAs at 8 x 256 MiB (6.85 vs 6.75 TB/s,
// profiles/r2/fold_occupancy.jsonl — more CTAs per SM or more vectors per
// thread do not help)
template <typename T, int OP, int NMAX, int THREADS = 512>
__global__ void __launch_bounds__(THREADS) fold_once_kernel(const FoldArgs a) {
  using A = typename AccT<T>::type;
  constexpr int kVec = 16 / sizeof(T);
  const size_t nvec = a.bytes >> 4;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nvec) {
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
  } else {  // ragged tail (< 16 B): the first threads past the last vector
    // (the launcher sizes the grid for nvec + 16 threads)
    const size_t base = nvec << 4;
    const size_t j = v - nvec;
    const size_t i = base + j * sizeof(T);
    if (j < (a.bytes - base) / sizeof(T)) {
      A acc = to_acc<T>(*reinterpret_cast<const T*>(a.src[0] + i));
      for (int r = 1; r < a.n; ++r)
        acc = apply_op<OP>(acc, to_acc<T>(*reinterpret_cast<const T*>(a.src[r] + i)));
      const T out = from_acc<T>(acc);
      for (int d = 0; d < a.ndst; ++d) *reinterpret_cast<T*>(a.dst[d] + i) = out;
    }
  }
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

// ------------------------------------------------- ReduceScatter rows
// Row y = blockIdx.y: dst[y] = fold_q(src[q] + y*src_stride), same fold rule.
template <typename T, int OP, int NMAX>
__global__ void __launch_bounds__(512) rows_vec_kernel(const RowsArgs a) {
  using A = typename AccT<T>::type;
  constexpr int kVec = 16 / sizeof(T);
  const size_t shift = (size_t)blockIdx.y * a.src_stride;
  char* dst = a.dst[blockIdx.y];
  const size_t nvec = a.bytes >> 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    uint4 in[NMAX];
#pragma unroll
    for (int r = 0; r < NMAX; ++r)
      if (r < a.n) in[r] = ld_stream(a.src[r] + shift + (v << 4));
    A acc[kVec];
    load_acc<T>(acc, in[0]);
#pragma unroll
    for (int r = 1; r < NMAX; ++r)
      if (r < a.n) fold_into<T, OP>(acc, in[r]);
    st_stream(dst + (v << 4), pack_acc<T>(acc));
  }
  if (blockIdx.x == 0) {
    const size_t base = nvec << 4;
    const size_t tail = (a.bytes - base) / sizeof(T);
    if (threadIdx.x < tail) {
      const size_t off = base + threadIdx.x * sizeof(T);
      A acc = to_acc<T>(*reinterpret_cast<const T*>(a.src[0] + shift + off));
      for (int r = 1; r < a.n; ++r)
        acc = apply_op<OP>(acc, to_acc<T>(*reinterpret_cast<const T*>(a.src[r] + shift + off)));
      *reinterpret_cast<T*>(dst + off) = from_acc<T>(acc);
    }
  }
  (void)kVec;
}

template <typename T, int OP>
__global__ void __launch_bounds__(512) rows_scalar_kernel(const RowsArgs a) {
  using A = typename AccT<T>::type;
  const size_t shift = (size_t)blockIdx.y * a.src_stride;
  T* dst = reinterpret_cast<T*>(a.dst[blockIdx.y]);
  const size_t count = a.bytes / sizeof(T);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    A acc = to_acc<T>(reinterpret_cast<const T*>(a.src[0] + shift)[i]);
    for (int r = 1; r < a.n; ++r)
      acc = apply_op<OP>(acc, to_acc<T>(reinterpret_cast<const T*>(a.src[r] + shift)[i]));
    dst[i] = from_acc<T>(acc);
  }
}

// ------------------------------------------------- TMA bulk-copy variants
// 1-D bulk copies (cp.async.bulk) stage each source's tile in shared memory
// behind an mbarrier (complete_tx), the CTA folds smem -> smem, and the
// result tile leaves through N bulk stores (smem -> global) without touching
// registers again.  S-stage ring; one CTA of kTmaThreads per SM.
constexpr int kTmaTile = 4096;    // bytes per source per stage
constexpr int kTmaStages = 4;
constexpr int kTmaThreads = 256;  // kTmaThreads * 16 B == kTmaTile

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem, const void* gmem, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem),
               "r"(smem_u32(smem)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int NMAX>
constexpr size_t tma_fold_smem() {
  return (size_t)kTmaStages * NMAX * kTmaTile + 2 * kTmaTile + kTmaStages * sizeof(uint64_t);
}

// Requires 16 B aligned src/dst; a.bytes may be ragged (tail < 16 B folded
// element-wise by CTA 0).
template <typename T, int OP, int NMAX>
__global__ void __launch_bounds__(kTmaThreads, 1) fold_tma_kernel(const FoldArgs a) {
  using A = typename AccT<T>::type;
  constexpr int kVec = 16 / sizeof(T);
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* in = smem;                                         // [S][NMAX][tile]
  unsigned char* out = smem + (size_t)kTmaStages * NMAX * kTmaTile;  // [2][tile]
  uint64_t* full = reinterpret_cast<uint64_t*>(out + 2 * kTmaTile);  // [S]
  const int n = a.n;
  const size_t body = a.bytes & ~(size_t)15;
  const size_t ntiles = (body + kTmaTile - 1) / kTmaTile;
  auto tile_bytes = [&](size_t t) -> uint32_t {
    return (uint32_t)min((size_t)kTmaTile, body - t * kTmaTile);
  };
  auto issue = [&](size_t t, int s) {
    const uint32_t len = tile_bytes(t);
    mbar_expect_tx(&full[s], len * n);
    for (int r = 0; r < n; ++r)
      bulk_load(in + ((size_t)s * NMAX + r) * kTmaTile, a.src[r] + t * kTmaTile, len, &full[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t first = blockIdx.x;
  if (threadIdx.x == 0)
    for (int s = 0; s < kTmaStages; ++s) {
      const size_t t = first + (size_t)s * gridDim.x;
      if (t < ntiles) issue(t, s);
    }
  uint32_t iter = 0;
  for (size_t t = first; t < ntiles; t += gridDim.x, ++iter) {
    const int s = iter % kTmaStages;
    const uint32_t parity = (iter / kTmaStages) & 1;
    const uint32_t len = tile_bytes(t);
    unsigned char* o = out + (iter & 1) * kTmaTile;
    if (threadIdx.x == 0) bulk_wait_read<1>();  // out[iter&1] free (store of iter-2 read)
    mbar_wait(&full[s], parity);
    __syncthreads();
    const uint32_t off = threadIdx.x * 16;
    if (off < len) {
      const unsigned char* base = in + (size_t)s * NMAX * kTmaTile + off;
      A acc[kVec];
      load_acc<T>(acc, *reinterpret_cast<const uint4*>(base));
#pragma unroll
      for (int r = 1; r < NMAX; ++r)
        if (r < n) fold_into<T, OP>(acc, *reinterpret_cast<const uint4*>(base + (size_t)r * kTmaTile));
      *reinterpret_cast<uint4*>(o + off) = pack_acc<T>(acc);
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int d = 0; d < a.ndst; ++d) bulk_store(a.dst[d] + t * kTmaTile, o, len);
      bulk_commit();
      const size_t nxt = t + (size_t)kTmaStages * gridDim.x;
      if (nxt < ntiles) issue(nxt, s);  // slot s fully consumed (barrier above)
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
  if (blockIdx.x == 0) {  // ragged tail (< 16 B)
    const size_t tail = (a.bytes - body) / sizeof(T);
    if (threadIdx.x < tail) {
      const size_t offb = body + threadIdx.x * sizeof(T);
      A acc = to_acc<T>(*reinterpret_cast<const T*>(a.src[0] + offb));
      for (int r = 1; r < n; ++r)
        acc = apply_op<OP>(acc, to_acc<T>(*reinterpret_cast<const T*>(a.src[r] + offb)));
      const T v = from_acc<T>(acc);
      for (int d = 0; d < a.ndst; ++d) *reinterpret_cast<T*>(a.dst[d] + offb) = v;
    }
  }
}

// AllGather fan-out with bulk copies: tile of source r (blockIdx.y) lands in
// smem once, then goes out to every destination by bulk stores.
static __global__ void __launch_bounds__(32, 1) fanout_tma_kernel(const FanoutArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kTmaStages * kTmaTile * 4);
  constexpr int kBig = kTmaTile * 4;  // 16 KB tiles: one smem slot per stage
  const int r = blockIdx.y;
  const char* src = a.src[r];
  const size_t shift = (size_t)r * a.dst_stride;
  const size_t body = a.bytes & ~(size_t)15;
  const size_t ntiles = (body + kBig - 1) / kBig;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kTmaStages; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto len_of = [&](size_t t) { return (uint32_t)min((size_t)kBig, body - t * kBig); };
  for (int s = 0; s < kTmaStages; ++s) {
    const size_t t = blockIdx.x + (size_t)s * gridDim.x;
    if (t < ntiles) {
      mbar_expect_tx(&full[s], len_of(t));
      bulk_load(smem + (size_t)s * kBig, src + t * kBig, len_of(t), &full[s]);
    }
  }
  uint32_t iter = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++iter) {
    const int s = iter % kTmaStages;
    mbar_wait(&full[s], (iter / kTmaStages) & 1);
    for (int d = 0; d < a.ndst; ++d) bulk_store(a.dst[d] + shift + t * kBig, smem + (size_t)s * kBig, len_of(t));
    bulk_commit();
    const size_t nxt = t + (size_t)kTmaStages * gridDim.x;
    if (nxt < ntiles) {
      bulk_wait_read<0>();  // slot s read by the stores just issued
      mbar_expect_tx(&full[s], len_of(nxt));
      bulk_load(smem + (size_t)s * kBig, src + nxt * kBig, len_of(nxt), &full[s]);
    }
  }
  bulk_wait_all();
  if (blockIdx.x == 0)
    for (size_t i = body; i < a.bytes; ++i)
      for (int d = 0; d < a.ndst; ++d) a.dst[d][shift + i] = src[i];
}

// Single-pass fan-out: one vector (or, past the last vector, one tail byte)
// per thread; blockIdx.y = source.  G adjacent CTAs read the same source span
// and each stores to its 1/G of the destinations (the repeated reads hit L2;
// G=2 halves the stores per thread: 0.379 vs 0.392 ms for 8 x 32 MiB,
// profiles/r1/fanout_ceiling.jsonl).  The launcher sizes x for G * (nvec + 16).
template <int NMAX, int G>
__global__ void __launch_bounds__(512) fanout_once_kernel(const FanoutArgs a) {
  constexpr int kPer = (NMAX + G - 1) / G;
  const int r = blockIdx.y;
  const int d0 = (int)(blockIdx.x % G) * kPer;
  const size_t nvec = a.bytes >> 4;
  const size_t v = (size_t)(blockIdx.x / G) * blockDim.x + threadIdx.x;
  const size_t shift = (size_t)r * a.dst_stride;
  if (v < nvec) {
    const uint4 w = ld_stream(a.src[r] + (v << 4));
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (d0 + k < a.ndst) st_stream(a.dst[d0 + k] + shift + (v << 4), w);
  } else {
    const size_t i = (nvec << 4) + (v - nvec);
    if (i < a.bytes) {
      const char b = a.src[r][i];
      for (int k = 0; k < kPer; ++k)
        if (d0 + k < a.ndst) a.dst[d0 + k][shift + i] = b;
    }
  }
}

// AllToAll transpose copy, blockIdx.y = r*n + q; one vector (or, past the
// last vector, one tail byte) per thread; byte loop when misaligned.
static __global__ void __launch_bounds__(512) xpose_kernel(const XposeArgs a, int vec) {
  const int r = blockIdx.y / a.n, q = blockIdx.y % a.n;
  const char* src = a.src[r] + (size_t)q * a.src_stride;
  char* dst = a.dst[q] + (size_t)r * a.dst_stride;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    // 4 vectors per thread, all loads before the stores (a bare 16 B copy per
    // thread left the AllToAll at 0.85 of the copy peak)
    const size_t nvec = a.bytes >> 4;
    size_t v = (size_t)blockIdx.x * blockDim.x * 4 + threadIdx.x;
    const size_t step4 = stride * 4;
    for (; v + 3 * blockDim.x < nvec; v += step4) {
      uint4 w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = ld_stream(src + ((v + u * blockDim.x) << 4));
#pragma unroll
      for (int u = 0; u < 4; ++u) st_stream(dst + ((v + u * blockDim.x) << 4), w[u]);
    }
    for (; v < nvec; v += blockDim.x) st_stream(dst + (v << 4), ld_stream(src + (v << 4)));
    for (size_t i = (nvec << 4) + t; i < a.bytes; i += stride) dst[i] = src[i];
  } else {
    for (size_t i = t; i < a.bytes; i += stride) dst[i] = src[i];
  }
}

// AllGather fan-out when every source and destination BASE is 16 B aligned
// but the rank-block stride is not (a ragged per-rank count: block r lands at
// dst[d] + r*dst_stride, misaligned by m = r*dst_stride mod 16, the same for
// every d).  Each thread writes one ALIGNED 16 B destination vector: the h =
// (16-m) mod 16 bytes before the first aligned destination boundary are the
// head, so destination vector j takes source bytes [h+16j, h+16j+16), i.e.
// the aligned source vectors j and j+1 funnel-shifted by h bytes.  The
// second load only happens when h != 0, and then it starts inside the
// source (h+16j+15 < bytes), so it never leaves the allocation's last
// 16 B granule.  Head and tail bytes (< 32 per source) are copied bytewise.
// Reads each source ~once from DRAM (the neighbouring vector hits L1/L2);
// replaces the byte-per-thread fallback (fanout_byte_kernel) for this case.
template <int Q>
__device__ __forceinline__ uint4 shift_window(const uint4& x, const uint4& y, uint32_t sh) {
  const uint32_t w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
  return make_uint4(__funnelshift_r(w[Q], w[Q + 1], sh), __funnelshift_r(w[Q + 1], w[Q + 2], sh),
                    __funnelshift_r(w[Q + 2], w[Q + 3], sh), __funnelshift_r(w[Q + 3], w[Q + 4], sh));
}

__device__ __forceinline__ uint4 shift_bytes(const uint4& x, const uint4& y, uint32_t h) {
  const uint32_t sh = (h & 3) * 8;
  switch (h >> 2) {  // uniform per (block, source): no divergence
    case 0: return shift_window<0>(x, y, sh);
    case 1: return shift_window<1>(x, y, sh);
    case 2: return shift_window<2>(x, y, sh);
    default: return shift_window<3>(x, y, sh);
  }
}

// G adjacent CTAs read the same source span and each stores to its 1/G of the
// destinations (fanout_once_kernel's split); the launcher uses G = 1 — with the
// shuffled window G = 2 measured 0.437 vs 0.414 ms (8 x 32 MiB+3 bf16).
template <int NMAX, int G>
__global__ void __launch_bounds__(512) fanout_shift_kernel(const FanoutArgs a) {
  constexpr int kPer = (NMAX + G - 1) / G;
  const int d0 = (int)(blockIdx.x % G) * kPer;
  const size_t blk = blockIdx.x / G, nblk = gridDim.x / G;
  const int r = blockIdx.y;
  const char* src = a.src[r];
  const size_t shift = (size_t)r * a.dst_stride;
  const uint32_t m = (uint32_t)(shift & 15);
  const size_t h = (16 - m) & 15;  // head bytes before the first aligned destination
  const size_t body = a.bytes > h ? (a.bytes - h) >> 4 : 0;
  const size_t stride = nblk * blockDim.x;
  // consecutive lanes hold consecutive source vectors: the window's second
  // vector comes from lane+1 by shuffle (one global load per output vector;
  // lane 31 and the warp's last active lane load theirs), not a second load
  // through L2.  The loop trip count is warp-uniform (stride is a multiple of
  // 32 and so is the warp's first j), so every lane reaches the shuffles.
  const uint32_t lane = threadIdx.x & 31;
  const size_t warp_j0 = blk * blockDim.x + (threadIdx.x & ~31u);
  for (size_t base = warp_j0; base < body; base += stride) {
    const size_t j = base + lane;
    const bool live = j < body;
    const uint4 x = live ? ld_stream(src + (j << 4)) : make_uint4(0, 0, 0, 0);
    uint4 out = x;
    if (h) {
      uint4 y;
      y.x = __shfl_down_sync(0xffffffffu, x.x, 1);
      y.y = __shfl_down_sync(0xffffffffu, x.y, 1);
      y.z = __shfl_down_sync(0xffffffffu, x.z, 1);
      y.w = __shfl_down_sync(0xffffffffu, x.w, 1);
      if (live && (lane == 31 || j + 1 == body))
        y = ld_vec_clamped(src + ((j + 1) << 4), a.bytes - ((j + 1) << 4), false);
      out = shift_bytes(x, y, (uint32_t)h);
    }
    if (live) {
#pragma unroll
      for (int k = 0; k < kPer; ++k)
        if (d0 + k < a.ndst) st_stream(a.dst[d0 + k] + shift + h + (j << 4), out);
    }
  }
  if (blockIdx.x == 0) {  // head [0, h) and tail [h + 16*body, bytes), every destination
    const size_t tail0 = h + (body << 4);
    const size_t nh = a.bytes < h ? a.bytes : h;
    const size_t i = threadIdx.x < nh ? threadIdx.x : tail0 + (threadIdx.x - nh);
    if ((threadIdx.x < nh || i < a.bytes) && threadIdx.x < 64) {
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
