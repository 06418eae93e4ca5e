// Stand-alone variant sweep for the virtual-rank fold (8 x 256 MiB fp32 sum):
// launch shape, unroll and cache-hint variants of the same streaming loop, plus
// a plain copy for the roofline reference.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/fold_bench tools/fold_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int N = 8;
struct Args { const float4* src[N]; float4* dst[N]; size_t nvec; };

template <int LD>  // 0: nc.L1::no_allocate  1: + L2::256B prefetch  2: plain ld.global
__device__ __forceinline__ float4 ld(const float4* p) {
  float4 v;
  if (LD == 0)
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else if (LD == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else
    v = *p;
  return v;
}
template <int ST>  // 0: L1::no_allocate  1: .cs  2: plain
__device__ __forceinline__ void st(float4* p, float4 v) {
  if (ST == 0)
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  else if (ST == 1)
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  else
    *p = v;
}

template <int THREADS, int UNR, int LD, int ST>
__global__ void __launch_bounds__(THREADS) fold(const Args a) {
  const size_t stride = (size_t)gridDim.x * THREADS;
  size_t v = (size_t)blockIdx.x * THREADS + threadIdx.x;
  for (; v + (UNR - 1) * stride < a.nvec; v += UNR * stride) {
    float4 in[UNR][N];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int r = 0; r < N; ++r) in[u][r] = ld<LD>(a.src[r] + v + u * stride);
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      float4 acc = in[u][0];
#pragma unroll
      for (int r = 1; r < N; ++r) { acc.x += in[u][r].x; acc.y += in[u][r].y; acc.z += in[u][r].z; acc.w += in[u][r].w; }
#pragma unroll
      for (int d = 0; d < N; ++d) st<ST>(a.dst[d] + v + u * stride, acc);
    }
  }
  for (; v < a.nvec; v += stride) {
    float4 acc = ld<LD>(a.src[0] + v);
#pragma unroll
    for (int r = 1; r < N; ++r) { float4 x = ld<LD>(a.src[r] + v); acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w; }
#pragma unroll
    for (int d = 0; d < N; ++d) st<ST>(a.dst[d] + v, acc);
  }
}

// G adjacent CTAs fold the same span (repeat reads from L2); each stores N/G dsts
template <int G>
__global__ void __launch_bounds__(512) fold_split(const Args a) {
  const int g = blockIdx.x % G;
  const size_t v = (size_t)(blockIdx.x / G) * 512 + threadIdx.x;
  if (v >= a.nvec) return;
  float4 in[N];
#pragma unroll
  for (int r = 0; r < N; ++r) in[r] = ld<0>(a.src[r] + v);
  float4 acc = in[0];
#pragma unroll
  for (int r = 1; r < N; ++r) { acc.x += in[r].x; acc.y += in[r].y; acc.z += in[r].z; acc.w += in[r].w; }
#pragma unroll
  for (int d = g * (N / G); d < (g + 1) * (N / G); ++d) st<0>(a.dst[d] + v, acc);
}

// single-pass fold with L2 eviction-priority hints (createpolicy):
// LP/SP: 0 none, 1 evict_first, 2 evict_last, 3 evict_unchanged (loads) / no hint
template <int LP, int SP>
__global__ void __launch_bounds__(512) fold_policy(const Args a) {
  const size_t v = (size_t)blockIdx.x * 512 + threadIdx.x;
  if (v >= a.nvec) return;
  uint64_t lpol = 0, spol = 0;
  if (LP == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(lpol));
  if (LP == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(lpol));
  if (LP == 3) asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(lpol));
  if (SP == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(spol));
  if (SP == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(spol));
  float4 in[N];
#pragma unroll
  for (int r = 0; r < N; ++r) {
    const float4* p = a.src[r] + v;
    if (LP == 0) in[r] = ld<0>(p);
    else asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                      : "=f"(in[r].x), "=f"(in[r].y), "=f"(in[r].z), "=f"(in[r].w) : "l"(p), "l"(lpol));
  }
  float4 acc = in[0];
#pragma unroll
  for (int r = 1; r < N; ++r) { acc.x += in[r].x; acc.y += in[r].y; acc.z += in[r].z; acc.w += in[r].w; }
#pragma unroll
  for (int d = 0; d < N; ++d) {
    float4* p = a.dst[d] + v;
    if (SP == 0) st<0>(p, acc);
    else asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                      :: "l"(p), "f"(acc.x), "f"(acc.y), "f"(acc.z), "f"(acc.w), "l"(spol) : "memory");
  }
}

// ceilings: read-only (8 inputs, one flag store if impossible) and store-only
__global__ void __launch_bounds__(512) read_only(const Args a, float* sink) {
  const size_t v = (size_t)blockIdx.x * 512 + threadIdx.x;
  if (v >= a.nvec) return;
  float s = 0.f;
#pragma unroll
  for (int r = 0; r < N; ++r) { float4 x = ld<0>(a.src[r] + v); s += x.x + x.y + x.z + x.w; }
  if (s == -1.2345f) *sink = s;
}
__global__ void __launch_bounds__(512) store_only(const Args a) {
  const size_t v = (size_t)blockIdx.x * 512 + threadIdx.x;
  if (v >= a.nvec) return;
  const float4 x = make_float4(v, v, v, v);
#pragma unroll
  for (int d = 0; d < N; ++d) st<0>(a.dst[d] + v, x);
}

__global__ void copyk(const float4* __restrict__ s, float4* __restrict__ d, size_t nvec) {
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += (size_t)gridDim.x * blockDim.x) d[v] = s[v];
}

__global__ void fill_random(uint32_t* p, size_t n, uint32_t seed) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = (x & 0x7fffff) | 0x3f800000u;  // finite floats in [1,2)
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
  const size_t bytes = 256ull << 20, nvec = bytes / 16;
  Args a; a.nvec = nvec;
  for (int r = 0; r < N; ++r) {
    float4 *s, *d; CK(cudaMalloc(&s, bytes)); CK(cudaMalloc(&d, bytes));
    CK(cudaMemset(s, 0, bytes)); a.src[r] = s; a.dst[r] = d;
  }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const bool random_data = argc > 1;
  if (random_data)
    for (int r = 0; r < N; ++r) fill_random<<<4 * sms, 256>>>((uint32_t*)a.src[r], bytes / 4, 77 + r);
  CK(cudaDeviceSynchronize());
  printf("{\"data\": \"%s\"}\n", random_data ? "random" : "memset");
  const double alg = 2.0 * N * bytes;
  auto report = [&](const char* name, float ms) { printf("{\"variant\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f}\n", name, ms, alg / (ms * 1e-3) / 1e9); };
  report("512x1/SM unr1 nc/noalloc (current)", timeit([&] { fold<512, 1, 0, 0><<<sms, 512>>>(a); }, 20));
  report("256x2/SM unr1", timeit([&] { fold<256, 1, 0, 0><<<2 * sms, 256>>>(a); }, 20));
  report("256x4/SM unr1", timeit([&] { fold<256, 1, 0, 0><<<4 * sms, 256>>>(a); }, 20));
  report("1024x1/SM unr1", timeit([&] { fold<1024, 1, 0, 0><<<sms, 1024>>>(a); }, 20));
  report("512x1/SM unr2", timeit([&] { fold<512, 2, 0, 0><<<sms, 512>>>(a); }, 20));
  report("256x1/SM unr2", timeit([&] { fold<256, 2, 0, 0><<<sms, 256>>>(a); }, 20));
  report("512x1/SM L2::256B", timeit([&] { fold<512, 1, 1, 0><<<sms, 512>>>(a); }, 20));
  report("512x1/SM st.cs", timeit([&] { fold<512, 1, 0, 1><<<sms, 512>>>(a); }, 20));
  report("512x1/SM plain ld/st", timeit([&] { fold<512, 1, 2, 2><<<sms, 512>>>(a); }, 20));
  report("512x2/SM unr1", timeit([&] { fold<512, 1, 0, 0><<<2 * sms, 512>>>(a); }, 20));
  report("128x8/SM unr1", timeit([&] { fold<128, 1, 0, 0><<<8 * sms, 128>>>(a); }, 20));
  report("512 x many (nvec/512 CTAs)", timeit([&] { fold<512, 1, 0, 0><<<(unsigned)((nvec + 511) / 512), 512>>>(a); }, 20));
  const unsigned nb = (unsigned)((nvec + 511) / 512);
  report("policy: none (single pass)", timeit([&] { fold_policy<0, 0><<<nb, 512>>>(a); }, 20));
  report("policy: loads evict_first", timeit([&] { fold_policy<1, 0><<<nb, 512>>>(a); }, 20));
  report("policy: loads evict_unchanged", timeit([&] { fold_policy<3, 0><<<nb, 512>>>(a); }, 20));
  report("policy: stores evict_first", timeit([&] { fold_policy<0, 1><<<nb, 512>>>(a); }, 20));
  report("policy: stores evict_last", timeit([&] { fold_policy<0, 2><<<nb, 512>>>(a); }, 20));
  report("policy: loads evict_first, stores evict_last", timeit([&] { fold_policy<1, 2><<<nb, 512>>>(a); }, 20));
  report("policy: loads evict_first, stores evict_first", timeit([&] { fold_policy<1, 1><<<nb, 512>>>(a); }, 20));
  report("split dst x2 (L2 re-read)", timeit([&] { fold_split<2><<<nb * 2, 512>>>(a); }, 20));
  report("split dst x4 (L2 re-read)", timeit([&] { fold_split<4><<<nb * 4, 512>>>(a); }, 20));
  float* sink; CK(cudaMalloc(&sink, 4));
  const float rms = timeit([&] { read_only<<<nb, 512>>>(a, sink); }, 20);
  printf("{\"variant\": \"ceiling: read-only 8 x 256 MiB\", \"ms\": %.4f, \"GBps\": %.1f}\n", rms, N * (double)bytes / (rms * 1e-3) / 1e9);
  const float wms = timeit([&] { store_only<<<nb, 512>>>(a); }, 20);
  printf("{\"variant\": \"ceiling: store-only 8 x 256 MiB\", \"ms\": %.4f, \"GBps\": %.1f}\n", wms, N * (double)bytes / (wms * 1e-3) / 1e9);
  printf("{\"variant\": \"ceiling: read-only + store-only times\", \"ms\": %.4f, \"GBps\": %.1f}\n", rms + wms, alg / ((rms + wms) * 1e-3) / 1e9);
  float cms = timeit([&] { for (int r = 0; r < N; ++r) copyk<<<4 * sms, 256>>>(a.src[r], a.dst[r], nvec); }, 10);
  printf("{\"variant\": \"copy 8 x 256 MiB (reference)\", \"ms\": %.4f, \"GBps\": %.1f}\n", cms, alg / (cms * 1e-3) / 1e9);
  return 0;
}
