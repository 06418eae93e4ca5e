// Phase timeline of the multi-rank AllReduce kernel in loopback (all ranks on
// one GPU, cooperative launch), from %globaltimer stamps at the protocol's
// phase boundaries (FLX_PHASE hooks in rank_kernels.cuh).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/rank_phases tools/rank_phases.cu
//   tools/bin/rank_phases [bytes_per_rank] [nranks] [nctas] [oneshot 0/1]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

__device__ unsigned long long g_t[16][128][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define FLX_PHASE(i) \
  if (threadIdx.x == 0) g_t[blockIdx.y][blockIdx.x][i] = gtimer();

#include "../paper_2510_15882_b200/csrc/rank_kernels.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

using namespace flx;

int main(int argc, char** argv) {
  const size_t bytes = argc > 1 ? strtoull(argv[1], nullptr, 0) : 4096;
  const int n = argc > 2 ? atoi(argv[2]) : 8;
  const int nctas = argc > 3 ? atoi(argv[3]) : 1;
  const int oneshot = argc > 4 ? atoi(argv[4]) : 0;
  const size_t slot = 64u << 20, small = 4u << 20;  // small: one-shot parts up to 64 KiB per CTA
  LoopbackArgs la;
  memset(&la, 0, sizeof(la));
  char* scratch[kMaxRanks];
  uint32_t* flags[kMaxRanks];
  for (int r = 0; r < n; ++r) {
    CK(cudaMalloc(&scratch[r], slot * (n + 1) + 2 * n * small));
    CK(cudaMalloc(&flags[r], (kFlagWords + kStateWords) * 4));
    CK(cudaMemset(flags[r], 0, (kFlagWords + kStateWords) * 4));
  }
  uint32_t* abort_word;
  CK(cudaHostAlloc(&abort_word, 64, cudaHostAllocMapped));
  *abort_word = 0;
  uint32_t* abort_dev;
  CK(cudaHostGetDevicePointer(&abort_dev, abort_word, 0));
  for (int r = 0; r < n; ++r) {
    RankArgs& a = la.r[r];
    char *s, *d;
    CK(cudaMalloc(&s, bytes));
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemset(s, 0, bytes));
    a.send = s;
    a.recv = d;
    for (int p = 0; p < n; ++p) {
      a.scratch[p] = scratch[p];
      a.flags[p] = flags[p];
    }
    a.rank = r;
    a.nranks = n;
    a.bytes = bytes;
    a.rank_stride = bytes;
    a.slot = slot;
    a.small_slot = small;
    a.oneshot = oneshot;
    a.ll = 0;  // the LL area is not allocated here
    a.bulk = 0;  // register copies: launched without the bulk ring's dynamic smem
    a.abort_word = abort_dev;
    a.spin_limit = 20000000000ll;
  }
  void* params[] = {&la};
  const void* fn = (const void*)loopback_allreduce_kernel<float, kSum>;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 50;
  for (int i = 0; i < 5; ++i)
    CK(cudaLaunchCooperativeKernel(fn, dim3(nctas, n), dim3(512), params, 0, 0));
  CK(cudaEventRecord(e0));
  for (int i = 0; i < iters; ++i)
    CK(cudaLaunchCooperativeKernel(fn, dim3(nctas, n), dim3(512), params, 0, 0));
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  static unsigned long long t[16][128][8];
  CK(cudaMemcpyFromSymbol(t, g_t, sizeof(t)));
  unsigned long long t0 = ~0ull;
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < nctas; ++c) t0 = t[r][c][0] < t0 ? t[r][c][0] : t0;
  double avg[7] = {0}, mx[7] = {0};
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < nctas; ++c)
      for (int i = 0; i < 7; ++i) {
        const double v = (double)(t[r][c][i] - t0) / 1e3;
        avg[i] += v / (n * nctas);
        mx[i] = v > mx[i] ? v : mx[i];
      }
  if (oneshot) avg[5] = avg[6] = mx[5] = mx[6] = 0;
  printf("{\"oneshot\": %d, \"bytes\": %zu, \"nranks\": %d, \"nctas\": %d, \"us_per_launch\": %.2f, "
         "\"phase_avg_us\": [%.2f, %.2f, %.2f, %.2f, %.2f, %.2f, %.2f], "
         "\"phase_max_us\": [%.2f, %.2f, %.2f, %.2f, %.2f, %.2f, %.2f], "
         "\"phases\": \"%s\"}\n",
         oneshot, bytes, n, nctas, ms * 1e3 / iters, avg[0], avg[1], avg[2], avg[3], avg[4], avg[5], avg[6],
         mx[0], mx[1], mx[2], mx[3], mx[4], mx[5], mx[6],
         oneshot ? "entry, setup, pushed+signalled, arrive waited, folded"
                 : "entry, kFree waited, pushed+signalled, arrive waited, folded+signalled, "
                   "ready waited, pulled+signalled");
  return 0;
}
