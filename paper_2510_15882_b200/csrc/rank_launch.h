// Launchers of the reducing rank kernels (AllReduce / ReduceScatter), one
// translation unit per dtype group (rank_launch_*.cu) so the 160 template
// instantiations compile in parallel.  `scatter` selects ReduceScatter;
// `loop` the cooperative loopback form (args = LoopbackArgs) instead of the
// per-GPU kernel (args = RankArgs).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <initializer_list>

namespace flx {

// Opt kernels into `bytes` of dynamic shared memory (the rank kernels'
// bulk-copy ring) on the CURRENT device, once per call site and device:
// cudaFuncSetAttribute binds to the current device's context, so a process
// that launches on several devices needs it on each.
inline void opt_in_dyn_smem(std::atomic<uint64_t>& done, std::initializer_list<const void*> fns,
                            int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  for (const void* f : fns) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done.fetch_or(bit, std::memory_order_acq_rel);
}

cudaError_t rank_reduce_i8(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                           int n, cudaStream_t s);
cudaError_t rank_reduce_i32(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                            int n, cudaStream_t s);
cudaError_t rank_reduce_i64(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                            int n, cudaStream_t s);
cudaError_t rank_reduce_f16(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                            int n, cudaStream_t s);
cudaError_t rank_reduce_f32(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                            int n, cudaStream_t s);
cudaError_t rank_reduce_f64(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                            int n, cudaStream_t s);
// each rank_launch_*.cu loads its module (see preload_module in internal.h)
cudaError_t preload_rank_i8();
cudaError_t preload_rank_i32();
cudaError_t preload_rank_i64();
cudaError_t preload_rank_f16();
cudaError_t preload_rank_f32();
cudaError_t preload_rank_f64();
// CTAs of the loopback AllReduce kernel that fit one SM (co-residency bound)
int loopback_blocks_per_sm();

}  // namespace flx
