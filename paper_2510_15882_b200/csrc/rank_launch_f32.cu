// Reducing rank kernels for float (see rank_launch.h).
#include "../../include/flexlink.h"
#include "internal.h"
#include "rank_launch_impl.cuh"

namespace flx {

cudaError_t rank_reduce_f32(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                           int n, cudaStream_t s) {
  switch (dtype) {
    case flxFloat32: return rank_reduce_typed<float>(op, scatter, loop, a, nctas, n, s);
  }
  return cudaErrorInvalidValue;
}

int loopback_blocks_per_sm() {
  int per_sm = 1;
  cudaFuncSetAttribute(loopback_allreduce_kernel<float, kSum>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRankDynSmem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, loopback_allreduce_kernel<float, kSum>,
                                                    512, kRankDynSmem) != cudaSuccess)
    return 1;
  return per_sm > 0 ? per_sm : 1;
}

cudaError_t preload_rank_f32() {
  return preload_module((const void*)rank_allreduce_kernel<float, kSum>);
}

}  // namespace flx
