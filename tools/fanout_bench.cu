// Stand-alone variant sweep for the virtual-rank AllGather fan-out
// (8 ranks x 32 MiB bf16 send -> 8 x 256 MiB gathered): each source block is
// read once and written to 8 destinations.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/fanout_bench tools/fanout_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int N = 8;
struct Args { const uint4* src[N]; uint4* dst[N]; size_t nvec; size_t stride_vec; };

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
template <int CS>
__device__ __forceinline__ void stv(uint4* p, uint4 v) {
  if (CS) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// blockIdx.y = source; grid-stride over vectors
template <int UNR, int CS>
__global__ void __launch_bounds__(512) fan(const Args a) {
  const int r = blockIdx.y;
  const uint4* src = a.src[r];
  const size_t shift = (size_t)r * a.stride_vec;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; v + (UNR - 1) * stride < a.nvec; v += UNR * stride) {
    uint4 w[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) w[u] = ldnc(src + v + u * stride);
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int d = 0; d < N; ++d) stv<CS>(a.dst[d] + shift + v + u * stride, w[u]);
  }
  for (; v < a.nvec; v += stride) {
    uint4 w = ldnc(src + v);
#pragma unroll
    for (int d = 0; d < N; ++d) stv<CS>(a.dst[d] + shift + v, w);
  }
}

// destination-major: blockIdx.y = destination d, each CTA copies a span of the
// gathered output (all sources) into dst[d]: reads N x, writes 1 x per CTA.
__global__ void __launch_bounds__(512) fan_dst(const Args a) {
  uint4* dst = a.dst[blockIdx.y];
  const size_t total = a.nvec * N;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += stride) {
    const size_t r = v / a.nvec, i = v - r * a.nvec;
    stv<0>(dst + r * a.stride_vec + i, ldnc(a.src[r] + i));
  }
}

// destination groups: G adjacent CTAs read the same source span (the repeats
// hit L2) and each writes N/G of the destinations: fewer stores per thread.
template <int G>
__global__ void __launch_bounds__(512) fan_split(const Args a) {
  const int r = blockIdx.y;
  const int g = blockIdx.x % G;
  const size_t v = (size_t)(blockIdx.x / G) * blockDim.x + threadIdx.x;
  if (v >= a.nvec) return;
  const uint4 w = ldnc(a.src[r] + v);
  const size_t shift = (size_t)r * a.stride_vec;
#pragma unroll
  for (int d = g * (N / G); d < (g + 1) * (N / G); ++d) stv<0>(a.dst[d] + shift + v, w);
}

__global__ void __launch_bounds__(512) write_only(const Args a) {
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < a.nvec * N) stv<0>(a.dst[blockIdx.y] + v, make_uint4(v, v, v, v));
}

__global__ void fill_random(uint32_t* p, size_t n, uint32_t seed) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = x;
  }
}

template <typename K>
float timeit(K launch, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) launch();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main(int argc, char**) {
  const size_t in_bytes = 32ull << 20, nvec = in_bytes / 16;
  Args a; a.nvec = nvec; a.stride_vec = nvec;
  for (int r = 0; r < N; ++r) {
    uint4 *s, *d; CK(cudaMalloc(&s, in_bytes)); CK(cudaMalloc(&d, in_bytes * N));
    CK(cudaMemset(s, r + 1, in_bytes)); a.src[r] = s; a.dst[r] = d;
  }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const bool random_data = argc > 1;
  if (random_data)
    for (int r = 0; r < N; ++r) fill_random<<<4 * sms, 256>>>((uint32_t*)a.src[r], in_bytes / 4, 77 + r);
  CK(cudaDeviceSynchronize());
  printf("{\"data\": \"%s\"}\n", random_data ? "random" : "memset");
  const double alg = (double)(N + N * N) * in_bytes;
  auto rep = [&](const char* name, float ms) { printf("{\"variant\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f}\n", name, ms, alg / (ms * 1e-3) / 1e9); };
  rep("persistent sm/8 per src, unr2", timeit([&] { fan<2, 0><<<dim3(sms / N, N), 512>>>(a); }, 20));
  rep("persistent 2sm/8 per src, unr2", timeit([&] { fan<2, 0><<<dim3(2 * sms / N, N), 512>>>(a); }, 20));
  rep("1 vec/thread many CTAs", timeit([&] { fan<1, 0><<<dim3((unsigned)((nvec + 511) / 512), N), 512>>>(a); }, 20));
  rep("1 vec/thread many CTAs st.cs", timeit([&] { fan<1, 1><<<dim3((unsigned)((nvec + 511) / 512), N), 512>>>(a); }, 20));
  rep("2 vec/thread many CTAs", timeit([&] { fan<2, 0><<<dim3((unsigned)((nvec + 1023) / 1024), N), 512>>>(a); }, 20));
  rep("dst-major sm/8 per dst", timeit([&] { fan_dst<<<dim3(sms / N * 2, N), 512>>>(a); }, 20));
  rep("dst-major many", timeit([&] { fan_dst<<<dim3((unsigned)((nvec * N + 511) / 512 / 4), N), 512>>>(a); }, 20));
  const unsigned nb = (unsigned)((nvec + 511) / 512);
  rep("split dst x2 (L2 re-read)", timeit([&] { fan_split<2><<<dim3(nb * 2, N), 512>>>(a); }, 20));
  rep("split dst x4 (L2 re-read)", timeit([&] { fan_split<4><<<dim3(nb * 4, N), 512>>>(a); }, 20));
  rep("split dst x8 (L2 re-read)", timeit([&] { fan_split<8><<<dim3(nb * 8, N), 512>>>(a); }, 20));
  // ceilings: the fan-out is 8/9 writes, so the HBM write-only rate bounds it
  const double wbytes = (double)N * N * in_bytes;
  auto rep_w = [&](const char* name, float ms) { printf("{\"variant\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f}\n", name, ms, wbytes / (ms * 1e-3) / 1e9); };
  rep_w("ceiling: cudaMemsetAsync of the 8 outputs (write only)",
        timeit([&] { for (int d = 0; d < N; ++d) cudaMemsetAsync(a.dst[d], 0, in_bytes * N); }, 20));
  rep_w("ceiling: store-only kernel, 1 vec/thread",
        timeit([&] { write_only<<<dim3((unsigned)((nvec * N + 511) / 512), N), 512>>>(a); }, 20));
  return 0;
}
