// Probe NVLink-SHARP multicast on this box: attribute, granularity, a
// 1-device multicast object bound to local memory, and a kernel that uses
// multimem.ld_reduce / multimem.st on it.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>

#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("{\"step\": \"%s\", \"error\": \"%s\"}\n", #x, s); return 1; } } while (0)

__global__ void mm(float* mc, float* out, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * i + 3 < n) {
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc + 4 * i) : "memory");
    reinterpret_cast<float4*>(out)[i] = v;
    v.x += 1.f; v.y += 1.f; v.z += 1.f; v.w += 1.f;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(mc + 4 * i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  }
}

int main() {
  CU(cuInit(0));
  CUdevice dev; CU(cuDeviceGet(&dev, 0));
  CUcontext ctx; CU(cuDevicePrimaryCtxRetain(&ctx, dev)); CU(cuCtxSetCurrent(ctx));
  int mcs = 0, fabric = 0;
  CU(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  cuDeviceGetAttribute(&fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("{\"multicast_supported\": %d, \"fabric_handles\": %d}\n", mcs, fabric);
  if (!mcs) return 0;
  const size_t want = 64ull << 20;
  CUmulticastObjectProp mp; memset(&mp, 0, sizeof(mp));
  mp.numDevices = 1; mp.size = want; mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0, gmin = 0;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CU(cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  printf("{\"granularity\": %zu, \"min_granularity\": %zu}\n", gran, gmin);
  // which (numDevices, handle type, size) combinations create?
  const unsigned long long types[3] = {0, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                       CU_MEM_HANDLE_TYPE_FABRIC};
  for (int nd = 1; nd <= 2; ++nd)
    for (int t = 0; t < 3; ++t)
      for (int sz = 0; sz < 2; ++sz) {
        CUmulticastObjectProp q; memset(&q, 0, sizeof(q));
        q.numDevices = nd; q.handleTypes = types[t]; q.size = sz ? gran : gmin;
        CUmemGenericAllocationHandle h;
        CUresult r = cuMulticastCreate(&h, &q);
        const char* s; cuGetErrorString(r, &s);
        printf("{\"numDevices\": %d, \"handleType\": %llu, \"size\": %zu, \"create\": \"%s\"}\n", nd,
               types[t], (size_t)q.size, s);
        if (r == CUDA_SUCCESS) cuMemRelease(h);
      }
  mp.handleTypes = 0;
  const size_t size = (want + gmin - 1) / gmin * gmin; mp.size = size;
  gran = gmin;
  CUmemGenericAllocationHandle mc; CU(cuMulticastCreate(&mc, &mp));
  CU(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp ap; memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t ugran = 0; CU(cuMemGetAllocationGranularity(&ugran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CUmemGenericAllocationHandle mem; CU(cuMemCreate(&mem, size, &ap, 0));
  CU(cuMulticastBindMem(mc, 0, mem, 0, size, 0));
  CUdeviceptr uc, mcva;
  CU(cuMemAddressReserve(&uc, size, ugran, 0, 0)); CU(cuMemMap(uc, size, 0, mem, 0));
  CU(cuMemAddressReserve(&mcva, size, gran, 0, 0)); CU(cuMemMap(mcva, size, 0, mc, 0));
  CUmemAccessDesc acc; acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE; acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU(cuMemSetAccess(uc, size, &acc, 1)); CU(cuMemSetAccess(mcva, size, &acc, 1));
  const size_t n = size / 4;
  float* h = new float[n];
  for (size_t i = 0; i < n; ++i) h[i] = (float)(i % 1000);
  cudaMemcpy((void*)uc, h, size, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, size);
  mm<<<(unsigned)((n / 4 + 255) / 256), 256>>>((float*)mcva, out, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"kernel\": \"%s\"}\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  float* o = new float[n]; float* u = new float[n];
  cudaMemcpy(o, out, size, cudaMemcpyDeviceToHost);
  cudaMemcpy(u, (void*)uc, size, cudaMemcpyDeviceToHost);
  size_t bad_ld = 0, bad_st = 0;
  for (size_t i = 0; i < n; ++i) { if (o[i] != h[i]) ++bad_ld; if (u[i] != h[i] + 1.f) ++bad_st; }
  printf("{\"ld_reduce_mismatch\": %zu, \"st_mismatch\": %zu, \"n\": %zu}\n", bad_ld, bad_st, n);
  // timing: ld_reduce+st over the multicast mapping vs plain
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int it = 0; it < 20; ++it) mm<<<(unsigned)((n / 4 + 255) / 256), 256>>>((float*)mcva, out, n);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("{\"mm_kernel_ms\": %.4f, \"GBps_rw\": %.1f}\n", ms / 20, 3.0 * size / (ms / 20 * 1e-3) / 1e9);
  return 0;
}
