// Can SMs pull host memory over PCIe faster than the copy engines?  Reads
// 8 x 256 MiB of pinned host memory three ways: cudaMemcpyAsync H2D (copy
// engine), a kernel reading the mapped host pointers into HBM, and a kernel
// folding the 8 host buffers straight into one device result (a fused
// H2D + AllReduce for the e2e case).  One JSON line each.
#include <cuda_runtime.h>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void pull(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

struct Srcs { const float4* s[8]; };
__global__ void fold8(Srcs a, float4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 acc = a.s[0][i];
#pragma unroll
    for (int r = 1; r < 8; ++r) {
      const float4 v = a.s[r][i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    dst[i] = acc;
  }
}

int main() {
  const size_t per = 256ull << 20, n = 8;
  char* h[8];
  char* d[8];
  for (int r = 0; r < 8; ++r) {
    CK(cudaHostAlloc(&h[r], per, cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaMalloc(&d[r], per));
  }
  float4* out;
  CK(cudaMalloc(&out, per));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  // copy engine
  for (int it = 0; it < 2; ++it) {
    CK(cudaEventRecord(a));
    for (int r = 0; r < 8; ++r) CK(cudaMemcpyAsync(d[r], h[r], per, cudaMemcpyHostToDevice));
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
  }
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"how\": \"copy engine\", \"ms\": %.3f, \"GBps\": %.2f}\n", ms, n * per / ms / 1e6);
  for (int grid : {148, 296, 592, 1184}) {
    for (int it = 0; it < 2; ++it) {
      CK(cudaEventRecord(a));
      for (int r = 0; r < 8; ++r) pull<<<grid, 512>>>((const uint4*)h[r], (uint4*)d[r], per / 16);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"how\": \"SM pull\", \"grid\": %d, \"ms\": %.3f, \"GBps\": %.2f}\n", grid, ms, n * per / ms / 1e6);
  }
  Srcs s;
  for (int r = 0; r < 8; ++r) s.s[r] = (const float4*)h[r];
  for (int grid : {148, 296, 592, 1184}) {
    for (int it = 0; it < 2; ++it) {
      CK(cudaEventRecord(a));
      fold8<<<grid, 512>>>(s, out, per / 16);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"how\": \"SM fold of host buffers\", \"grid\": %d, \"ms\": %.3f, \"GBps_read\": %.2f}\n", grid, ms,
           n * per / ms / 1e6);
  }
  return 0;
}
