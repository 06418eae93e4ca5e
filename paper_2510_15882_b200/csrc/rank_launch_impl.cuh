#pragma once
// Shared by the rank_launch_*.cu units: the per-(T, op) launch of the reducing
// rank kernels, per GPU or cooperatively in loopback.
#include "rank_kernels.cuh"
#include "rank_launch.h"

namespace flx {

template <typename T, int OP>
cudaError_t rank_reduce_t(bool scatter, bool loop, const void* args, int nctas, int nranks,
                          cudaStream_t s) {
  // the bulk-copy ring (RankArgs::bulk) is dynamic shared memory
  static std::atomic<uint64_t> opted{0};
  opt_in_dyn_smem(opted, {(const void*)loopback_allreduce_kernel<T, OP>,
                          (const void*)rank_allreduce_kernel<T, OP>,
                          (const void*)loopback_reducescatter_kernel<T, OP>,
                          (const void*)rank_reducescatter_kernel<T, OP>},
                  (int)kRankDynSmem);
  const int bulk = loop ? static_cast<const LoopbackArgs*>(args)->r[0].bulk
                        : static_cast<const RankArgs*>(args)->bulk;
  const size_t dyn = bulk ? kRankDynSmem : 0;
  if (loop) {
    const void* fn = scatter ? (const void*)loopback_reducescatter_kernel<T, OP>
                             : (const void*)loopback_allreduce_kernel<T, OP>;
    void* params[] = {const_cast<void*>(args)};
    return cudaLaunchCooperativeKernel(fn, dim3(nctas, nranks), dim3(512), params, dyn, s);
  }
  const RankArgs& a = *static_cast<const RankArgs*>(args);
  if (scatter)
    rank_reducescatter_kernel<T, OP><<<nctas, 512, dyn, s>>>(a);
  else
    rank_allreduce_kernel<T, OP><<<nctas, 512, dyn, s>>>(a);
  return cudaGetLastError();
}

template <typename T>
cudaError_t rank_reduce_typed(int op, bool scatter, bool loop, const void* a, int nctas, int n,
                              cudaStream_t s) {
  switch (op) {
    case kSum: return rank_reduce_t<T, kSum>(scatter, loop, a, nctas, n, s);
    case kProd: return rank_reduce_t<T, kProd>(scatter, loop, a, nctas, n, s);
    case kMax: return rank_reduce_t<T, kMax>(scatter, loop, a, nctas, n, s);
    case kMin: return rank_reduce_t<T, kMin>(scatter, loop, a, nctas, n, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace flx
