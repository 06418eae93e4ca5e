// Reducing rank kernels for double (see rank_launch.h).
#include "../../include/flexlink.h"
#include "rank_launch_impl.cuh"

namespace flx {

cudaError_t rank_reduce_f64(int dtype, int op, bool scatter, bool loop, const void* a, int nctas,
                           int n, cudaStream_t s) {
  switch (dtype) {
    case flxFloat64: return rank_reduce_typed<double>(op, scatter, loop, a, nctas, n, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace flx
