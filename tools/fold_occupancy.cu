// Occupancy / bytes-in-flight sweep of the single-pass virtual-rank fold
// (8 x 256 MiB fp32 sum, 8 outputs — config 1's kernel shape): CTAs per SM
// forced by __launch_bounds__ min-blocks, vectors per thread per source, and
// the store order.  Complements tools/fold_bench.cu (launch shapes, hints).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/fold_occupancy tools/fold_occupancy.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int N = 8;
struct Args { const float4* src[N]; float4* dst[N]; size_t nvec; };

__device__ __forceinline__ float4 ld(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st(float4* p, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// V vectors per thread per source, V*THREADS consecutive vectors per CTA
template <int THREADS, int MINB, int V>
__global__ void __launch_bounds__(THREADS, MINB) once(const Args a) {
  const size_t base = (size_t)blockIdx.x * THREADS * V + threadIdx.x;
  float4 acc[V];
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const size_t v = base + (size_t)u * THREADS;
    if (v < a.nvec) {
      float4 in[N];
#pragma unroll
      for (int r = 0; r < N; ++r) in[r] = ld(a.src[r] + v);
      acc[u] = in[0];
#pragma unroll
      for (int r = 1; r < N; ++r) {
        acc[u].x += in[r].x; acc[u].y += in[r].y; acc[u].z += in[r].z; acc[u].w += in[r].w;
      }
    }
  }
#pragma unroll
  for (int d = 0; d < N; ++d)
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const size_t v = base + (size_t)u * THREADS;
      if (v < a.nvec) st(a.dst[d] + v, acc[u]);
    }
}

int main() {
  const size_t bytes = 256ull << 20, nvec = bytes / 16;
  Args a{};
  for (int r = 0; r < N; ++r) {
    CK(cudaMalloc((void**)&a.src[r], bytes));
    CK(cudaMalloc((void**)&a.dst[r], bytes));
    CK(cudaMemset((void*)a.src[r], r + 1, bytes));
  }
  a.nvec = nvec;
  const double alg = 2.0 * N * bytes;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 20;
  };
  auto report = [&](const char* name, const void* fn, int threads, float ms) {
    cudaFuncAttributes at{};
    cudaFuncGetAttributes(&at, fn);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
    printf("{\"variant\": \"%s\", \"regs\": %d, \"local_bytes\": %zu, \"ctas_per_sm\": %d, "
           "\"ms\": %.4f, \"GBps\": %.1f}\n",
           name, at.numRegs, at.localSizeBytes, per_sm, ms, alg / (ms * 1e-3) / 1e9);
  };
#define RUN(T, M, V)                                                                          \
  {                                                                                           \
    const unsigned grid = (unsigned)((nvec + (size_t)T * V - 1) / ((size_t)T * V));           \
    float ms = timeit([&] { once<T, M, V><<<grid, T>>>(a); });                                \
    report(#T "x" #M "/SM v" #V, (const void*)once<T, M, V>, T, ms);                          \
  }
  for (int rep = 0; rep < 2; ++rep) {  // two passes, interleaved, to see the noise
  RUN(1024, 1, 1)
  RUN(512, 1, 1)  // the library's fold_once shape (46 regs -> 2 CTAs/SM)
  RUN(1024, 1, 2)
  RUN(768, 1, 1)
  }
  RUN(512, 2, 1)
  RUN(512, 3, 1)
  RUN(512, 4, 1)
  RUN(256, 6, 1)
  RUN(256, 8, 1)
  RUN(512, 1, 2)
  RUN(512, 2, 2)
  RUN(256, 4, 2)
  RUN(1024, 1, 1)
  RUN(1024, 2, 1)
  CK(cudaGetLastError());
  return 0;
}
