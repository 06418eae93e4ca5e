// Flag round-trip latency between two CTAs of one kernel (the loopback
// engine's signalling primitive), by memory scope and flavour.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/flag_pingpong tools/flag_pingpong.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

template <int MODE>
__device__ __forceinline__ void put(uint32_t* p, uint32_t v) {
  if (MODE == 0) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else if (MODE == 1) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else if (MODE == 2) { __threadfence_system(); *(volatile uint32_t*)p = v; }
  else asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <int MODE>
__device__ __forceinline__ uint32_t get(const uint32_t* p) {
  uint32_t v;
  if (MODE == 0) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else if (MODE == 1) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else if (MODE == 2) v = *(volatile const uint32_t*)p;
  else asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int MODE>
__global__ void pingpong(uint32_t* a, uint32_t* b, int iters) {
  if (threadIdx.x != 0) return;
  for (int i = 1; i <= iters; ++i) {
    if (blockIdx.x == 0) {
      put<MODE>(a, i);
      while ((int)(get<MODE>(b) - i) < 0) {}
    } else {
      while ((int)(get<MODE>(a) - i) < 0) {}
      put<MODE>(b, i);
    }
  }
}

template <int MODE>
float run(uint32_t* a, uint32_t* b, int iters) {
  cudaMemset(a, 0, 4); cudaMemset(b, 0, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  pingpong<MODE><<<2, 32>>>(a, b, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / iters;
}

// fan-out signal cost: 14 flags per round (the AllReduce phase-2 signal),
// CTA 0 signals, CTA 1 waits on the last flag and answers on one flag.
// WAYS: 0 = 14 lanes each st.release.sys; 1 = lane 0 fence.sys then 14
// relaxed stores; 2 = lane 0 fence.sys, __syncwarp, 14 lanes relaxed store
template <int WAYS>
__global__ void fanout_signal(uint32_t* flags, uint32_t* back, int iters) {
  const int lane = threadIdx.x;
  for (int i = 1; i <= iters; ++i) {
    if (blockIdx.x == 0) {
      __syncthreads();
      if (WAYS == 0) {
        if (lane < 14) put<0>(flags + lane * 64, i);
      } else if (WAYS == 1) {
        if (lane == 0) {
          asm volatile("fence.acq_rel.sys;" ::: "memory");
          for (int k = 0; k < 14; ++k) put<3>(flags + k * 64, i);
        }
      } else {
        if (lane == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
        __syncwarp();
        if (lane < 14) put<3>(flags + lane * 64, i);
      }
      if (lane == 0) while ((int)(get<0>(back) - i) < 0) {}
      __syncthreads();
    } else if (lane == 0) {
      while ((int)(get<0>(flags + 13 * 64) - i) < 0) {}
      put<0>(back, i);
    }
  }
}

template <int WAYS>
float run_fan(uint32_t* flags, uint32_t* back, int iters) {
  cudaMemset(flags, 0, 14 * 64 * 4); cudaMemset(back, 0, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fanout_signal<WAYS><<<2, 32>>>(flags, back, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / iters;
}

int main() {
  uint32_t* d; cudaMalloc(&d, 4096);
  uint32_t *a = d, *b = d + 256;  // different 1 KiB lines
  const int iters = 20000;
  const char* names[4] = {"st.release.sys / ld.acquire.sys", "st.release.gpu / ld.acquire.gpu",
                          "threadfence_system + volatile", "relaxed.sys (no ordering)"};
  float us[4] = {run<0>(a, b, iters), run<1>(a, b, iters), run<2>(a, b, iters), run<3>(a, b, iters)};
  for (int m = 0; m < 4; ++m)
    printf("{\"flags\": \"device\", \"mode\": \"%s\", \"round_trip_us\": %.3f}\n", names[m], us[m]);
  uint32_t* fl; cudaMalloc(&fl, 64 * 1024);
  const char* ways[3] = {"14 lanes st.release.sys", "lane0 fence.sys + 14 relaxed stores",
                         "lane0 fence.sys, syncwarp, 14 lanes relaxed"};
  const float fu[3] = {run_fan<0>(fl, fl + 8192, iters), run_fan<1>(fl, fl + 8192, iters),
                       run_fan<2>(fl, fl + 8192, iters)};
  for (int m = 0; m < 3; ++m)
    printf("{\"flags\": \"device\", \"signal14\": \"%s\", \"round_trip_us\": %.3f}\n", ways[m], fu[m]);
  // a release.sys store while this CTA has outstanding writes to host-mapped memory
  uint32_t* h; cudaHostAlloc(&h, 4096, cudaHostAllocMapped);
  uint32_t* hd; cudaHostGetDevicePointer(&hd, h, 0);
  const float hu = run<0>(hd, hd + 256, 2000);
  printf("{\"flags\": \"host-mapped\", \"mode\": \"%s\", \"round_trip_us\": %.3f}\n", names[0], hu);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
