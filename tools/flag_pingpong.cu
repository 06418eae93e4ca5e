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

// cost of a satisfied 7-flag wait (flags already >= target), per call:
// W 0: 7 lanes ld.acquire.sys; 1: 7 lanes ld.relaxed.sys, then each of those
// lanes fence.acq_rel.sys; 2: lane 0 loads 7 flags relaxed, one fence;
// 3: 7 lanes relaxed, __syncwarp, lane 0 fence (not a formal acquire)
template <int W>
__global__ void satisfied_wait(const uint32_t* flags, int iters, uint32_t* out) {
  const int lane = threadIdx.x;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (W == 0) {
      if (lane < 7) acc += get<0>(flags + lane * 64);
    } else if (W == 1) {
      if (lane < 7) {
        acc += get<3>(flags + lane * 64);
        asm volatile("fence.acq_rel.sys;" ::: "memory");
      }
    } else if (W == 2) {
      if (lane == 0) {
        uint32_t v[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) v[k] = get<3>(flags + k * 64);
#pragma unroll
        for (int k = 0; k < 7; ++k) acc += v[k];
        asm volatile("fence.acq_rel.sys;" ::: "memory");
      }
    } else {
      if (lane < 7) acc += get<3>(flags + lane * 64);
      __syncwarp();
      if (lane == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
    __syncwarp();
  }
  if (acc == 0xdeadbeef) *out = acc;
}

template <int W>
float run_wait(const uint32_t* flags, uint32_t* out, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  satisfied_wait<W><<<1, 32>>>(flags, iters, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / iters;
}

// cost of a 7-flag release signal right after the CTA wrote `kb` KiB of data
// (W 0: 7 lanes st.release.sys; 1: bar, lane 0 fence.sys, syncwarp, 7 lanes relaxed)
template <int W>
__global__ void __launch_bounds__(512) signal_after_writes(uint32_t* flags, uint4* data, int kb, int iters) {
  for (int i = 1; i <= iters; ++i) {
    for (int v = threadIdx.x; v < kb * 64; v += blockDim.x) data[v] = make_uint4(i, i, i, i);
    __syncthreads();
    if (W == 0) {
      if (threadIdx.x < 7) put<0>(flags + threadIdx.x * 64, i);
    } else {
      if (threadIdx.x == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
      __syncwarp();
      if (threadIdx.x < 7) put<3>(flags + threadIdx.x * 64, i);
    }
    __syncthreads();
  }
}

template <int W>
float run_sig(uint32_t* flags, uint4* data, int kb, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  signal_after_writes<W><<<1, 512>>>(flags, data, kb, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / iters;
}

#define CK_SET(p) cudaMemset(p, 1, 64 * 1024)

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
  CK_SET(fl);
  const char* wn[4] = {"7 lanes ld.acquire.sys", "7 lanes relaxed + per-lane fence.sys",
                       "lane 0: 7 relaxed loads + 1 fence.sys", "7 lanes relaxed, lane 0 fence.sys"};
  const float wu[4] = {run_wait<0>(fl, fl + 8000, 2000), run_wait<1>(fl, fl + 8000, 2000),
                       run_wait<2>(fl, fl + 8000, 2000), run_wait<3>(fl, fl + 8000, 2000)};
  for (int m = 0; m < 4; ++m)
    printf("{\"satisfied_wait7\": \"%s\", \"us\": %.3f}\n", wn[m], wu[m]);
  uint4* data; cudaMalloc(&data, 1 << 20);
  for (int kb : {0, 4, 64}) {
    printf("{\"signal7_after_kib\": %d, \"7 lanes st.release.sys_us\": %.3f, \"one fence + relaxed_us\": %.3f}\n",
           kb, run_sig<0>(fl, data, kb, 2000), run_sig<1>(fl, data, kb, 2000));
  }
  // a release.sys store while this CTA has outstanding writes to host-mapped memory
  uint32_t* h; cudaHostAlloc(&h, 4096, cudaHostAllocMapped);
  uint32_t* hd; cudaHostGetDevicePointer(&hd, h, 0);
  const float hu = run<0>(hd, hd + 256, 2000);
  printf("{\"flags\": \"host-mapped\", \"mode\": \"%s\", \"round_trip_us\": %.3f}\n", names[0], hu);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
