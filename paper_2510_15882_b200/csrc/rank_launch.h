// Launchers of the reducing rank kernels (AllReduce / ReduceScatter), one
// translation unit per dtype group (rank_launch_*.cu) so the 160 template
// instantiations compile in parallel.  `scatter` selects ReduceScatter;
// `loop` the cooperative loopback form (args = LoopbackArgs) instead of the
// per-GPU kernel (args = RankArgs).
#pragma once

#include <cuda_runtime.h>

namespace flx {

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
// CTAs of the loopback AllReduce kernel that fit one SM (co-residency bound)
int loopback_blocks_per_sm();

}  // namespace flx
