// Reducing rank kernels for double (see rank_launch.h).
#include "../../include/flexlink.h"
#include "internal.h"
#include "rank_launch_impl.cuh"

namespace flx {

cudaError_t rank_reduce_f64(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                           int n, cudaStream_t s) {
  switch (dtype) {
    case flxFloat64: return rank_reduce_typed<double>(op, scatter, loop, a, nctas, n, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t preload_rank_f64() {
  return preload_module((const void*)rank_allreduce_kernel<double, kSum>);
}

}  // namespace flx
