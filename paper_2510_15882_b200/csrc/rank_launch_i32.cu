// Reducing rank kernels for int32_t, uint32_t (see rank_launch.h).
#include "../../include/flexlink.h"
#include "internal.h"
#include "rank_launch_impl.cuh"

namespace flx {

cudaError_t rank_reduce_i32(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                           int n, cudaStream_t s) {
  switch (dtype) {
    case flxInt32: return rank_reduce_typed<int32_t>(op, scatter, loop, a, nctas, n, s);
    case flxUint32: return rank_reduce_typed<uint32_t>(op, scatter, loop, a, nctas, n, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t preload_rank_i32() {
  return preload_module((const void*)rank_allreduce_kernel<int32_t, kSum>);
}

}  // namespace flx
