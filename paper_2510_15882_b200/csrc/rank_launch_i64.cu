// Reducing rank kernels for int64_t, uint64_t (see rank_launch.h).
#include "../../include/flexlink.h"
#include "internal.h"
#include "rank_launch_impl.cuh"

namespace flx {

cudaError_t rank_reduce_i64(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                           int n, cudaStream_t s) {
  switch (dtype) {
    case flxInt64: return rank_reduce_typed<int64_t>(op, scatter, loop, a, nctas, n, s);
    case flxUint64: return rank_reduce_typed<uint64_t>(op, scatter, loop, a, nctas, n, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t preload_rank_i64() {
  return preload_module((const void*)rank_allreduce_kernel<int64_t, kSum>);
}

}  // namespace flx
