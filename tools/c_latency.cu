// Host cost of one 8-virtual-rank collective issued from C (no Python):
// flxGroupCollective vs GroupStart + 8 calls + GroupEnd, tiny messages.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/c_latency tools/c_latency.cu \
//          -Iinclude -Lpaper_2510_15882_b200 -lflexlink -Xlinker -rpath=$PWD/paper_2510_15882_b200
#include <chrono>
#include <cstdio>

#include "flexlink.h"

int main() {
  const int n = 8;
  const size_t count = 1024;
  flxComm_t comms[n];
  int devs[n] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (flxCommInitAll(comms, n, devs) != flxSuccess) { printf("init: %s\n", flxGetLastError()); return 1; }
  void *s[n], *r[n];
  for (int i = 0; i < n; ++i) { cudaMalloc(&s[i], count * 4); cudaMalloc(&r[i], count * 4); }
  cudaStream_t st; cudaStreamCreate(&st);
  for (int mode = 0; mode < 2; ++mode) {
    for (int w = 0; w < 100; ++w) flxGroupCollective(flxCollAllReduce, comms, n, s, r, count, flxFloat32, flxSum, st);
    cudaStreamSynchronize(st);
    const int iters = 2000;
    auto t0 = std::chrono::steady_clock::now();
    for (int it = 0; it < iters; ++it) {
      if (mode == 0) {
        flxGroupCollective(flxCollAllReduce, comms, n, s, r, count, flxFloat32, flxSum, st);
      } else {
        flxGroupStart();
        for (int i = 0; i < n; ++i) flxAllReduce(s[i], r[i], count, flxFloat32, flxSum, comms[i], st);
        flxGroupEnd();
      }
    }
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    auto t2 = std::chrono::steady_clock::now();
    printf("{\"mode\": \"%s\", \"host_us_per_call\": %.2f, \"total_us_per_call\": %.2f}\n",
           mode == 0 ? "flxGroupCollective" : "GroupStart+8+GroupEnd",
           std::chrono::duration<double, std::micro>(t1 - t0).count() / iters,
           std::chrono::duration<double, std::micro>(t2 - t0).count() / iters);
  }
  return 0;
}
