#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void push(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
int main() {
  const size_t per = 256ull << 20;
  char *h, *d;
  CK(cudaHostAlloc(&h, per, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaMalloc(&d, per));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for (int it = 0; it < 2; ++it) { cudaEventRecord(a); for (int r = 0; r < 8; ++r) cudaMemcpyAsync(h, d, per, cudaMemcpyDeviceToHost); cudaEventRecord(b); cudaEventSynchronize(b); }
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"how\": \"copy engine D2H\", \"GBps\": %.2f}\n", 8 * per / ms / 1e6);
  for (int grid : {4, 8, 16, 32, 64, 148}) {
    for (int it = 0; it < 2; ++it) { cudaEventRecord(a); for (int r = 0; r < 8; ++r) push<<<grid, 512>>>((const uint4*)d, (uint4*)h, per / 16); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"how\": \"SM writes to host\", \"grid\": %d, \"GBps\": %.2f}\n", grid, 8 * per / ms / 1e6);
  }
  return 0;
}
