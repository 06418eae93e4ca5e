// NVLink-SHARP (NVLS) AllReduce: the NVSwitch reduces.  Every rank's message
// sits in a buffer bound to one multicast object; rank r asks the switch for
// the sum of every rank's copy of chunk r (multimem.ld_reduce on the multicast
// address) and writes the result back to every rank at once (multimem.st).
// Per GPU and direction that moves ~S instead of the two-shot's 2(N-1)/N·S,
// so the switch-side reduction lifts the ceiling above the per-link two-shot
// (PAPER.md:176 — the paper's NVLink leg is NCCL, which runs NVLS on
// NVSwitch systems).
//
// Per call, CTA b of rank r (same grid on every rank):
//   1 stage    copy part b of every chunk of my send into my UC buffer (local)
//   2 barrier  red.release.sys +1 on the MULTICAST arrive word b (lands on every
//              rank), then wait until MY copy of it reached N * epoch
//   3 reduce   for part b of chunk r: ld_reduce(mc) -> st(mc): every rank's UC
//              buffer now holds the reduced part
//   4 barrier  the same on the second word: every rank's stores of part b landed
//   5 land     copy part b of every chunk from my UC buffer into recv
// Reuse of the UC buffer by the next call is safe: a peer's step-3 loads of my
// chunk finish before its step-4 arrival, which precedes my step 5 and so my
// next step 1; its next step-3 stores into my buffer wait for my next step-2
// arrival, which follows my step 5.
//
// (nvls_allgather_kernel below: the same buffer, one multicast store per slice.)
//
// The reduction order inside the switch is unspecified: results equal the
// fixed-order fold for integer-valued data and are within 1 ulp of the output
// dtype otherwise (bf16/fp16 accumulate in fp32: .acc::f32).  Capability-gated
// (flxNvlsProbe / FLX_NVLS=1); absent where multicast objects cannot be made.
#pragma once

#include "kernels.cuh"

namespace flx {

constexpr int kNvlsCtas = 64;
constexpr size_t kNvlsFlagBytes = 4096;  // [arrive1][arrive2][64 CTAs] at the buffer head

struct NvlsArgs {
  const char* send;
  char* recv;
  char* uc;         // my buffer (unicast mapping), data after kNvlsFlagBytes
  char* mc;         // the multicast mapping of the same offsets
  uint32_t* state;  // per-CTA epoch counters, private device memory [kNvlsCtas]
  int rank, nranks;
  size_t bytes;     // message bytes per rank (a multiple of 16 * nranks for the vector path)
  uint32_t* abort_word;
  long long spin_limit;
  char* peers[kMaxRanks];  // FLX_NVLS_EMULATE only: every rank's buffer (unicast, one GPU)
};

// data other ranks wrote during this kernel: bypass L1
__device__ __forceinline__ uint4 ld_cg_nvls(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void mm_red_add_release(uint32_t* mc_word, uint32_t v) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc_word), "r"(v)
               : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename T>
__device__ __forceinline__ uint4 mm_ld_reduce_sum(const char* mc);

template <>
__device__ __forceinline__ uint4 mm_ld_reduce_sum<float>(const char* mc) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}

template <>
__device__ __forceinline__ uint4 mm_ld_reduce_sum<__nv_bfloat16>(const char* mc) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}

template <>
__device__ __forceinline__ uint4 mm_ld_reduce_sum<__half>(const char* mc) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}

__device__ __forceinline__ void mm_st(char* mc, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// The three multicast operations the kernels use, on byte offset `o` of the
// data area (after kNvlsFlagBytes) or arrive word `word`.
#ifdef FLX_NVLS_EMULATE
// tools/nvls_emulate.cu: every rank on ONE GPU (cooperative launch) and each
// multimem operation replaced by its unicast equivalent over every rank's
// buffer — the reduction in rank order (the switch's order is unspecified).
// It runs this file's partitioning, epochs, barriers and staging on a GPU that
// is in no multicast fabric; the multimem instructions themselves need one.
__device__ __forceinline__ void nvls_arrive(const NvlsArgs& a, size_t word) {
  for (int q = 0; q < a.nranks; ++q)
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(
                     reinterpret_cast<uint32_t*>(a.peers[q]) + word),
                 "r"(1u)
                 : "memory");
}
template <typename T>
__device__ __forceinline__ uint4 nvls_reduce(const NvlsArgs& a, size_t o) {
  typename AccT<T>::type acc[16 / sizeof(T)];
  load_acc<T>(acc, ld_cg_nvls(a.peers[0] + kNvlsFlagBytes + o));
  for (int q = 1; q < a.nranks; ++q)
    fold_into<T, kSum>(acc, ld_cg_nvls(a.peers[q] + kNvlsFlagBytes + o));
  return pack_acc<T>(acc);
}
__device__ __forceinline__ void nvls_store(const NvlsArgs& a, size_t o, const uint4& v) {
  for (int q = 0; q < a.nranks; ++q)
    *reinterpret_cast<uint4*>(a.peers[q] + kNvlsFlagBytes + o) = v;
}
#else
__device__ __forceinline__ void nvls_arrive(const NvlsArgs& a, size_t word) {
  mm_red_add_release(reinterpret_cast<uint32_t*>(a.mc) + word, 1u);
}
template <typename T>
__device__ __forceinline__ uint4 nvls_reduce(const NvlsArgs& a, size_t o) {
  return mm_ld_reduce_sum<T>(a.mc + kNvlsFlagBytes + o);
}
__device__ __forceinline__ void nvls_store(const NvlsArgs& a, size_t o, const uint4& v) {
  mm_st(a.mc + kNvlsFlagBytes + o, v);
}
#endif

// CTA-wide NVLS barrier on word `w` (CTA b's arrive word of one kind): +1 on
// every rank through the multicast mapping, then wait for my copy to reach
// target.  false: timed out / aborted.
__device__ __forceinline__ bool nvls_barrier(const NvlsArgs& a, size_t word, uint32_t target) {
  __shared__ int ok;
  __syncthreads();  // this CTA's prior stores (incl. multimem.st) before the release
  if (threadIdx.x == 0) {
    nvls_arrive(a, word);
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(a.uc) + word;
    const long long t0 = clock64();
    int good = 1;
    uint32_t spins = 0;
    while ((int)(ld_acquire_sys_u32(mine) - target) < 0) {
      if ((++spins & 4095) == 0 &&
          (*(volatile uint32_t*)a.abort_word || clock64() - t0 > a.spin_limit)) {
        atomicExch(a.abort_word, 1u);
        good = 0;
        break;
      }
    }
    ok = good;
  }
  __syncthreads();
  return ok;
}

template <typename T>
__device__ __forceinline__ void nvls_allreduce_body(const NvlsArgs& a) {
  const int b = blockIdx.x, nb = gridDim.x, r = a.rank, n = a.nranks;
  const uint32_t e = a.state[b] + 1;  // this CTA's call epoch (identical on every rank)
  const size_t chunk = a.bytes / n;   // 16 B multiple (host guarantees)
  const size_t part = (((chunk + nb - 1) / nb) + 15) & ~(size_t)15;  // covers the chunk
  const size_t lo = min(chunk, (size_t)b * part), hi = min(chunk, lo + part);
  char* ucd = a.uc + kNvlsFlagBytes;
  // 1 stage my message (part b of every chunk) into the multicast-bound buffer
  for (int c = 0; c < n; ++c)
    for (size_t v = lo + 16 * threadIdx.x; v < hi; v += 16 * blockDim.x) {
      const size_t o = (size_t)c * chunk + v;
      *reinterpret_cast<uint4*>(ucd + o) = ld_stream(a.send + o);
    }
  if (!nvls_barrier(a, b, (uint32_t)n * e)) return;
  // 3 the switch sums part b of chunk r over every rank and writes it back to all
  for (size_t v = lo + 16 * threadIdx.x; v < hi; v += 16 * blockDim.x) {
    const size_t o = (size_t)r * chunk + v;
    nvls_store(a, o, nvls_reduce<T>(a, o));
  }
  if (!nvls_barrier(a, kNvlsCtas + b, (uint32_t)n * e)) return;
  // 5 land every reduced chunk (part b) in recv
  for (int c = 0; c < n; ++c)
    for (size_t v = lo + 16 * threadIdx.x; v < hi; v += 16 * blockDim.x) {
      const size_t o = (size_t)c * chunk + v;
      *reinterpret_cast<uint4*>(a.recv + o) = ld_cg_nvls(ucd + o);
    }
  if (threadIdx.x == 0) a.state[b] = e;
}

template <typename T>
__global__ void __launch_bounds__(512, 2) nvls_allreduce_kernel(const __grid_constant__ NvlsArgs a) {
  nvls_allreduce_body<T>(a);
}

// NVLS AllGather: one multimem.st puts my slice into EVERY rank's buffer (the
// switch replicates it), so each GPU sends its S bytes once instead of N-1
// times.  a.bytes = per-rank send bytes (16 B multiple); the buffer holds N
// blocks; recv block c at c * a.stride.  Per call, CTA b:
//   1 store part b of my slice to block r of every rank's buffer (multicast)
//   2 barrier: every rank's part b landed everywhere
//   3 land part b of every block from my buffer into recv
//   4 barrier: every rank finished landing before anyone's next call stores
static __device__ __forceinline__ void nvls_allgather_body(const NvlsArgs& a, size_t stride) {
  const int b = blockIdx.x, nb = gridDim.x, r = a.rank, n = a.nranks;
  const uint32_t e = a.state[b] + 1;
  const size_t part = (((a.bytes + nb - 1) / nb) + 15) & ~(size_t)15;  // covers the slice
  const size_t lo = min(a.bytes, (size_t)b * part), hi = min(a.bytes, lo + part);
  char* ucd = a.uc + kNvlsFlagBytes;
  for (size_t v = lo + 16 * threadIdx.x; v < hi; v += 16 * blockDim.x)
    nvls_store(a, (size_t)r * a.bytes + v, ld_stream(a.send + v));
  if (!nvls_barrier(a, b, (uint32_t)n * e)) return;
  for (int c = 0; c < n; ++c)
    for (size_t v = lo + 16 * threadIdx.x; v < hi; v += 16 * blockDim.x)
      *reinterpret_cast<uint4*>(a.recv + (size_t)c * stride + v) =
          ld_cg_nvls(ucd + (size_t)c * a.bytes + v);
  if (!nvls_barrier(a, kNvlsCtas + b, (uint32_t)n * e)) return;
  if (threadIdx.x == 0) a.state[b] = e;
}

template <int UNUSED = 0>
__global__ void __launch_bounds__(512, 2) nvls_allgather_kernel(const __grid_constant__ NvlsArgs a,
                                                                 size_t stride) {
  nvls_allgather_body(a, stride);
}

#ifdef FLX_NVLS_EMULATE
// every rank's CTAs in one cooperative grid (blockIdx.y = rank)
struct NvlsLoopArgs {
  NvlsArgs r[kMaxRanks];
};
template <typename T>
__global__ void __launch_bounds__(512, 2) nvls_allreduce_loop_kernel(const __grid_constant__ NvlsLoopArgs la) {
  nvls_allreduce_body<T>(la.r[blockIdx.y]);
}
__global__ void __launch_bounds__(512, 2) nvls_allgather_loop_kernel(const __grid_constant__ NvlsLoopArgs la,
                                                                      size_t stride) {
  nvls_allgather_body(la.r[blockIdx.y], stride);
}
#endif

}  // namespace flx
