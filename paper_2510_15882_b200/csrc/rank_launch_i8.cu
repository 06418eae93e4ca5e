// Reducing rank kernels for int8_t, uint8_t (see rank_launch.h).
#include "../../include/flexlink.h"
#include "internal.h"
#include "rank_launch_impl.cuh"

namespace flx {

cudaError_t rank_reduce_i8(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                           int n, cudaStream_t s) {
  switch (dtype) {
    case flxInt8: return rank_reduce_typed<int8_t>(op, scatter, loop, a, nctas, n, s);
    case flxUint8: return rank_reduce_typed<uint8_t>(op, scatter, loop, a, nctas, n, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t preload_rank_i8() {
  return preload_module((const void*)rank_allreduce_kernel<int8_t, kSum>);
}

}  // namespace flx
