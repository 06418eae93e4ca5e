// Reducing rank kernels for __half, __nv_bfloat16 (see rank_launch.h).
#include "../../include/flexlink.h"
#include "internal.h"
#include "rank_launch_impl.cuh"

namespace flx {

cudaError_t rank_reduce_f16(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                           int n, cudaStream_t s) {
  switch (dtype) {
    case flxFloat16: return rank_reduce_typed<__half>(op, scatter, loop, a, nctas, n, s);
    case flxBfloat16: return rank_reduce_typed<__nv_bfloat16>(op, scatter, loop, a, nctas, n, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t preload_rank_f16() {
  return preload_module((const void*)rank_allreduce_kernel<__half, kSum>);
}

}  // namespace flx
