// Per-round phase timeline of the multi-rank two-shot AllReduce in loopback
// (all ranks on one GPU, cooperative launch), from %globaltimer stamps at every
// phase boundary of every round (FLX_PHASE hooks in rank_kernels.cuh).  Reports
// how much of the call's time rank 0's CTAs spend moving data between ranks
// (push / pull) while some of its CTAs fold — with staggered rounds the folds
// of half the CTAs overlap the other half's transfers.  Build both ways:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFLX_STAGGER=1 \
//        -o tools/bin/rank_timeline tools/rank_timeline.cu
//   tools/bin/rank_timeline [bytes_per_rank] [nranks] [nctas] [bulk]
// (bulk = 1: copy phases as TMA bulk copies, RankArgs::bulk, the library default)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

constexpr int kEv = 64;
__device__ unsigned long long g_ev[16][64][kEv];  // (phase << 56) | globaltimer ns
__device__ int g_n[16][64];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define FLX_PHASE(i)                                                                  \
  if (threadIdx.x == 0) {                                                             \
    const int j_ = g_n[blockIdx.y][blockIdx.x]++;                                     \
    if (j_ < kEv) g_ev[blockIdx.y][blockIdx.x][j_] = ((unsigned long long)(i) << 56) | \
                                                      (gtimer() & ((1ull << 56) - 1)); \
  }

#include "../paper_2510_15882_b200/csrc/rank_kernels.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

using namespace flx;

int main(int argc, char** argv) {
  const size_t bytes = argc > 1 ? strtoull(argv[1], nullptr, 0) : (256ull << 20);
  const int n = argc > 2 ? atoi(argv[2]) : 8;
  const int nctas = argc > 3 ? atoi(argv[3]) : 32;
  const int bulk = argc > 4 ? atoi(argv[4]) : 0;
  const size_t slot = 64u << 20, small = 1u << 20;
  LoopbackArgs la;
  memset(&la, 0, sizeof(la));
  for (int r = 0; r < n; ++r) {
    char* sc;
    uint32_t* fl;
    CK(cudaMalloc(&sc, slot * (n + 1) + 2 * n * small));
    CK(cudaMalloc(&fl, (kFlagWords + kStateWords) * 4));
    CK(cudaMemset(fl, 0, (kFlagWords + kStateWords) * 4));
    for (int q = 0; q < n; ++q) {
      la.r[q].scratch[r] = sc;
      la.r[q].flags[r] = fl;
    }
  }
  uint32_t *abort_word, *abort_dev;
  CK(cudaHostAlloc(&abort_word, 64, cudaHostAllocMapped));
  *abort_word = 0;
  CK(cudaHostGetDevicePointer(&abort_dev, abort_word, 0));
  for (int r = 0; r < n; ++r) {
    RankArgs& a = la.r[r];
    char *s, *d;
    CK(cudaMalloc(&s, bytes));
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemset(s, 0, bytes));
    a.send = s;
    a.recv = d;
    a.rank = r;
    a.nranks = n;
    a.bytes = bytes;
    a.rank_stride = bytes;
    a.slot = slot;
    a.small_slot = small;
    a.oneshot = 0;
    a.ll = 0;
    a.bulk = bulk;
    a.abort_word = abort_dev;
    a.spin_limit = 20000000000ll;
  }
  void* params[] = {&la};
  const void* fn = (const void*)loopback_allreduce_kernel<float, kSum>;
  const size_t dyn = bulk ? kRankDynSmem : 0;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRankDynSmem));
  for (int i = 0; i < 4; ++i)
    CK(cudaLaunchCooperativeKernel(fn, dim3(nctas, n), dim3(512), params, dyn, 0));
  CK(cudaDeviceSynchronize());
  int zero[16][64] = {};
  CK(cudaMemcpyToSymbol(g_n, zero, sizeof(zero)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  CK(cudaEventRecord(e0));
  CK(cudaLaunchCooperativeKernel(fn, dim3(nctas, n), dim3(512), params, dyn, 0));
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  static unsigned long long ev[16][64][kEv];
  static int cnt[16][64];
  CK(cudaMemcpyFromSymbol(ev, g_ev, sizeof(ev)));
  CK(cudaMemcpyFromSymbol(cnt, g_n, sizeof(cnt)));
  // rank 0's CTAs: intervals [phase 1 -> 2] push, [3 -> 4] fold, [5 -> 6] pull
  struct Iv { double a, b; int kind; };  // kind 0 transfer, 1 fold
  std::vector<Iv> iv;
  double t0 = 1e30, t1 = 0;
  int rounds = 0;
  for (int c = 0; c < nctas; ++c) {
    double last[8];
    for (int j = 0; j < std::min(cnt[0][c], kEv); ++j) {
      const int ph = (int)(ev[0][c][j] >> 56);
      const double t = (double)(ev[0][c][j] & ((1ull << 56) - 1)) / 1e3;
      t0 = std::min(t0, t);
      t1 = std::max(t1, t);
      last[ph] = t;
      if (ph == 2) iv.push_back({last[1], t, 0});
      if (ph == 4) iv.push_back({last[3], t, 1});
      if (ph == 6) {
        iv.push_back({last[5], t, 0});
        if (c == 0) ++rounds;
      }
    }
  }
  // sweep: time with >= 1 CTA transferring, and with some CTA folding while
  // another transfers (the overlap staggering buys)
  std::vector<std::pair<double, int>> pts;
  for (auto& x : iv) {
    pts.push_back({x.a, x.kind == 0 ? 1 : 100});
    pts.push_back({x.b, x.kind == 0 ? -1 : -100});
  }
  std::sort(pts.begin(), pts.end());
  int xfer = 0, fold = 0;
  double covered = 0, overlap = 0, only_fold = 0, prev = t0;
  for (auto& p : pts) {
    const double dt = p.first - prev;
    if (xfer > 0) covered += dt;
    if (xfer > 0 && fold > 0) overlap += dt;
    if (xfer == 0 && fold > 0) only_fold += dt;
    prev = p.first;
    if (p.second == 1 || p.second == -1) xfer += p.second;
    else fold += p.second / 100;
  }
  const double span = t1 - t0;
  printf("{\"bulk\": %d, \"stagger\": %d, \"bytes\": %zu, \"nranks\": %d, \"nctas\": %d, \"rounds_cta0\": %d, "
         "\"us_per_launch\": %.1f, \"span_us\": %.1f, \"transfer_coverage\": %.3f, "
         "\"fold_overlapping_transfers\": %.3f, \"fold_only\": %.3f}\n",
         bulk, FLX_STAGGER, bytes, n, nctas, rounds, ms * 1e3, span, covered / span, overlap / span,
         only_fold / span);
  return 0;
}
