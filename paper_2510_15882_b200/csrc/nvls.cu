// NVLink-SHARP multicast setup and the NVLS AllReduce launch.
//
// Multi-rank: rank 0 creates a multicast object spanning the world's GPUs
// with a FABRIC handle type and publishes the 64-byte fabric handle in the
// bootstrap header (a plain byte copy through the shared segment — no file
// descriptor passing); every rank imports it, adds its device, and once every
// device is added binds its own buffer and maps both the unicast and the
// multicast view.  Each step is a counted rendezvous in which failures are
// counted too, so every rank ends with the same verdict: NVLS on everywhere or
// nowhere (with the reason).  Driver entry points are resolved at run time
// (no -lcuda), as for the stream memory operations.
//
// flxNvlsProbe runs the same machinery for ONE device and the kernel on it
// (ld_reduce over a single rank is the identity): the capability check the
// GPU tests gate on, and the reason text where it is absent.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "args.h"
#include "internal.h"
#include "nvls.h"
#include "nvls_kernels.cuh"

namespace flx {

namespace {

struct Drv {
  decltype(&cuMulticastCreate) mc_create = nullptr;
  decltype(&cuMulticastGetGranularity) mc_gran = nullptr;
  decltype(&cuMulticastAddDevice) mc_add = nullptr;
  decltype(&cuMulticastBindMem) mc_bind = nullptr;
  decltype(&cuMulticastUnbind) mc_unbind = nullptr;
  decltype(&cuMemCreate) mem_create = nullptr;
  decltype(&cuMemRelease) mem_release = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemGetAllocationGranularity) alloc_gran = nullptr;
  decltype(&cuMemExportToShareableHandle) export_h = nullptr;
  decltype(&cuMemImportFromShareableHandle) import_h = nullptr;
  decltype(&cuDeviceGetAttribute) attr = nullptr;
  decltype(&cuGetErrorString) err = nullptr;
  bool ok = false;
};

template <typename F>
bool resolve(const char* name, F* out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return false;
  *out = reinterpret_cast<F>(fn);
  return true;
}

const Drv& drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = resolve("cuMulticastCreate", &d.mc_create) &&
           resolve("cuMulticastGetGranularity", &d.mc_gran) &&
           resolve("cuMulticastAddDevice", &d.mc_add) &&
           resolve("cuMulticastBindMem", &d.mc_bind) &&
           resolve("cuMulticastUnbind", &d.mc_unbind) && resolve("cuMemCreate", &d.mem_create) &&
           resolve("cuMemRelease", &d.mem_release) &&
           resolve("cuMemAddressReserve", &d.reserve) &&
           resolve("cuMemAddressFree", &d.addr_free) && resolve("cuMemMap", &d.map) &&
           resolve("cuMemUnmap", &d.unmap) && resolve("cuMemSetAccess", &d.set_access) &&
           resolve("cuMemGetAllocationGranularity", &d.alloc_gran) &&
           resolve("cuMemExportToShareableHandle", &d.export_h) &&
           resolve("cuMemImportFromShareableHandle", &d.import_h) &&
           resolve("cuDeviceGetAttribute", &d.attr) && resolve("cuGetErrorString", &d.err);
  });
  return d;
}

// false + reason when r is not CUDA_SUCCESS
bool check(CUresult r, const char* what, NvlsBuffer* nb) {
  if (r == CUDA_SUCCESS) return true;
  const char* s = "unknown";
  if (drv().err) drv().err(r, &s);
  snprintf(nb->why, sizeof(nb->why), "%s: %s", what, s);
  return false;
}

template <typename F>
bool wait_for(F pred, double seconds) {
  const auto t0 = std::chrono::steady_clock::now();
  while (!pred()) {
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > seconds)
      return false;
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  return true;
}

// multicast capability of the device + the object's properties and granularity
bool mc_props(NvlsBuffer* nb, int device, int ndev, size_t data_bytes, bool fabric,
              CUmulticastObjectProp* prop) {
  const Drv& d = drv();
  if (!d.ok) {
    snprintf(nb->why, sizeof(nb->why), "driver lacks the multicast / VMM entry points");
    return false;
  }
  int mcs = 0;
  if (!check(d.attr(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, device),
             "cuDeviceGetAttribute(MULTICAST_SUPPORTED)", nb))
    return false;
  if (!mcs) {
    snprintf(nb->why, sizeof(nb->why), "device %d reports no multicast support", device);
    return false;
  }
  memset(prop, 0, sizeof(*prop));
  prop->numDevices = ndev;
  prop->handleTypes = fabric ? CU_MEM_HANDLE_TYPE_FABRIC : 0;
  prop->size = kNvlsFlagBytes + data_bytes;
  size_t gran = 0;
  if (!check(d.mc_gran(&gran, prop, CU_MULTICAST_GRANULARITY_MINIMUM),
             "cuMulticastGetGranularity", nb))
    return false;
  prop->size = (prop->size + gran - 1) / gran * gran;
  nb->size = prop->size;
  nb->capacity = prop->size - kNvlsFlagBytes;
  nb->device = device;
  return true;
}

// bind my physical buffer to the multicast object and map both views
bool bind_and_map(NvlsBuffer* nb) {
  const Drv& d = drv();
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = nb->device;
  size_t ugran = 0;
  if (!check(d.alloc_gran(&ugran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
             "cuMemGetAllocationGranularity", nb))
    return false;
  const size_t size = (nb->size + ugran - 1) / ugran * ugran;
  if (size != nb->size) {
    snprintf(nb->why, sizeof(nb->why), "multicast size %zu not a multiple of the %zu B page",
             nb->size, ugran);
    return false;
  }
  if (!check(d.mem_create(&nb->mem, nb->size, &ap, 0), "cuMemCreate", nb)) return false;
  if (!check(d.mc_bind(nb->mc, 0, nb->mem, 0, nb->size, 0), "cuMulticastBindMem", nb))
    return false;
  nb->bound = true;
  CUmemAccessDesc acc;
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = nb->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (!check(d.reserve(&nb->uc, nb->size, ugran, 0, 0), "cuMemAddressReserve(uc)", nb) ||
      !check(d.map(nb->uc, nb->size, 0, nb->mem, 0), "cuMemMap(uc)", nb))
    return false;
  nb->uc_mapped = true;
  if (!check(d.set_access(nb->uc, nb->size, &acc, 1), "cuMemSetAccess(uc)", nb)) return false;
  if (!check(d.reserve(&nb->mcva, nb->size, ugran, 0, 0), "cuMemAddressReserve(mc)", nb) ||
      !check(d.map(nb->mcva, nb->size, 0, nb->mc, 0), "cuMemMap(mc)", nb))
    return false;
  nb->mc_mapped = true;
  if (!check(d.set_access(nb->mcva, nb->size, &acc, 1), "cuMemSetAccess(mc)", nb)) return false;
  // arrive words start at zero before any peer can add to them (the bound
  // rendezvous follows); per-CTA epochs likewise
  if (cudaMemset(reinterpret_cast<void*>(nb->uc), 0, kNvlsFlagBytes) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&nb->state), kNvlsCtas * 4) != cudaSuccess ||
      cudaMemset(nb->state, 0, kNvlsCtas * 4) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    snprintf(nb->why, sizeof(nb->why), "zeroing the NVLS flags failed");
    return false;
  }
  return true;
}

}  // namespace

bool nvls_dtype_ok(int dtype) {
  return dtype == flxFloat32 || dtype == flxBfloat16 || dtype == flxFloat16;
}

void nvls_free(NvlsBuffer* nb) {
  const Drv& d = drv();
  if (!d.ok) return;
  cudaSetDevice(nb->device);
  if (nb->state) cudaFree(nb->state);
  if (nb->mc_mapped) d.unmap(nb->mcva, nb->size);
  if (nb->mcva) d.addr_free(nb->mcva, nb->size);
  if (nb->uc_mapped) d.unmap(nb->uc, nb->size);
  if (nb->uc) d.addr_free(nb->uc, nb->size);
  if (nb->bound) d.mc_unbind(nb->mc, nb->device, 0, nb->size);
  if (nb->mem) d.mem_release(nb->mem);
  if (nb->mc) d.mem_release(nb->mc);
  const char* why = "released";
  *nb = NvlsBuffer();
  snprintf(nb->why, sizeof(nb->why), "%s", why);
}

void nvls_setup_rank(NvlsBuffer* nb, NvlsBoot* boot, int rank, int nranks, int device,
                     size_t data_bytes, double timeout_s) {
  const Drv& d = drv();
  CUmulticastObjectProp prop;
  bool mine = mc_props(nb, device, nranks, data_bytes, true, &prop);
  // 1 rank 0 creates and publishes the fabric handle
  if (rank == 0) {
    bool ok = mine && check(d.mc_create(&nb->mc, &prop), "cuMulticastCreate", nb) &&
              check(d.export_h(&boot->handle, nb->mc, CU_MEM_HANDLE_TYPE_FABRIC, 0),
                    "cuMemExportToShareableHandle(FABRIC)", nb);
    if (!ok) snprintf(boot->why, sizeof(boot->why), "rank 0: %s", nb->why);
    __atomic_store_n(&boot->state, ok ? 1 : -1, __ATOMIC_RELEASE);
    mine = ok;
  } else {
    if (!wait_for([&] { return __atomic_load_n(&boot->state, __ATOMIC_ACQUIRE) != 0; },
                  timeout_s)) {
      snprintf(nb->why, sizeof(nb->why), "rank 0 never published the multicast handle");
      mine = false;
    } else if (__atomic_load_n(&boot->state, __ATOMIC_ACQUIRE) < 0) {
      snprintf(nb->why, sizeof(nb->why), "%s", boot->why);
      mine = false;
    } else if (mine) {
      mine = check(d.import_h(&nb->mc, &boot->handle, CU_MEM_HANDLE_TYPE_FABRIC),
                   "cuMemImportFromShareableHandle(FABRIC)", nb);
    }
  }
  // 2 every device joins (counted whether it succeeded or not)
  if (mine) mine = check(d.mc_add(nb->mc, device), "cuMulticastAddDevice", nb);
  nb->added = mine;
  __atomic_fetch_add(&boot->added, 1, __ATOMIC_ACQ_REL);
  if (!wait_for([&] { return __atomic_load_n(&boot->added, __ATOMIC_ACQUIRE) >= nranks; },
                timeout_s)) {
    snprintf(nb->why, sizeof(nb->why), "not every rank reached cuMulticastAddDevice");
    mine = false;
  }
  // 3 bind + map my buffer, then agree
  if (mine) mine = bind_and_map(nb);
  __atomic_store_n(&boot->ok[rank], mine ? 1 : -1, __ATOMIC_RELEASE);
  __atomic_fetch_add(&boot->bound, 1, __ATOMIC_ACQ_REL);
  bool all = wait_for([&] { return __atomic_load_n(&boot->bound, __ATOMIC_ACQUIRE) >= nranks; },
                      timeout_s);
  for (int p = 0; all && p < nranks; ++p)
    if (__atomic_load_n(&boot->ok[p], __ATOMIC_ACQUIRE) != 1) {
      if (mine) snprintf(nb->why, sizeof(nb->why), "rank %d could not join the multicast buffer", p);
      all = false;
    }
  if (!all) {
    nvls_free(nb);
    return;
  }
  nb->on = true;
  snprintf(nb->why, sizeof(nb->why), "on: %zu MiB multicast buffer over %d GPUs",
           nb->capacity >> 20, nranks);
}

cudaError_t launch_nvls_allgather(const void* args, size_t stride, int nctas, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  nvls_allgather_kernel<0><<<nctas, 512, 0, s>>>(*static_cast<const NvlsArgs*>(args), stride);
  return cudaGetLastError();
}

cudaError_t launch_nvls_allreduce(int dtype, const void* args, int nctas, cudaStream_t s) {
  const NvlsArgs& a = *static_cast<const NvlsArgs*>(args);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  switch (dtype) {
    case flxFloat32: nvls_allreduce_kernel<float><<<nctas, 512, 0, s>>>(a); break;
    case flxBfloat16: nvls_allreduce_kernel<__nv_bfloat16><<<nctas, 512, 0, s>>>(a); break;
    case flxFloat16: nvls_allreduce_kernel<__half><<<nctas, 512, 0, s>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t preload_nvls_cu() {
  return preload_module((const void*)nvls_allgather_kernel<0>);
}

}  // namespace flx

using namespace flx;

extern "C" {

// Can this device make a multicast object and run the NVLS kernel on it?  A
// one-device object (ld_reduce over one rank returns the data itself) checked
// end to end: *available = 1 and reason "ok: ..." or 0 and why not.
flxResult_t flxNvlsProbe(int device, int* available, char* reason, size_t reason_len) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  if (!available) return fail(flxInvalidArgument, "null available");
  *available = 0;
  NvlsBuffer nb;
  auto say = [&](const char* s) {
    if (reason && reason_len) snprintf(reason, reason_len, "%s", s);
  };
  if (cudaSetDevice(device) != cudaSuccess) {
    say("cudaSetDevice failed");
    return flxSuccess;
  }
  CUmulticastObjectProp prop;
  const size_t bytes = 1 << 20;
  bool ok = mc_props(&nb, device, 1, bytes, false, &prop) &&
            check(drv().mc_create(&nb.mc, &prop), "cuMulticastCreate (1 device)", &nb) &&
            check(drv().mc_add(nb.mc, device), "cuMulticastAddDevice", &nb) && bind_and_map(&nb);
  if (ok) {
    char *src = nullptr, *dst = nullptr;
    uint32_t* abort_word = nullptr;
    ok = cudaMalloc(&src, bytes) == cudaSuccess && cudaMalloc(&dst, bytes) == cudaSuccess &&
         cudaMalloc(&abort_word, 4) == cudaSuccess && cudaMemset(abort_word, 0, 4) == cudaSuccess;
    if (ok) {
      std::vector<float> h(bytes / 4), back(bytes / 4);
      for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 977) - 400.f;
      cudaMemcpy(src, h.data(), bytes, cudaMemcpyHostToDevice);
      NvlsArgs a{src, dst, reinterpret_cast<char*>(nb.uc), reinterpret_cast<char*>(nb.mcva),
                 nb.state, 0, 1, bytes, abort_word, (long long)2e9};
      ok = launch_nvls_allreduce(flxFloat32, &a, 8, 0) == cudaSuccess &&
           cudaDeviceSynchronize() == cudaSuccess;
      if (ok) {
        cudaMemcpy(back.data(), dst, bytes, cudaMemcpyDeviceToHost);
        ok = memcmp(back.data(), h.data(), bytes) == 0;
        if (!ok) snprintf(nb.why, sizeof(nb.why), "NVLS AllReduce result mismatch on one device");
      }
      if (ok) {  // and the AllGather kernel (one rank: a copy through the multicast store)
        cudaMemset(dst, 0, bytes);
        ok = launch_nvls_allgather(&a, bytes, 8, 0) == cudaSuccess &&
             cudaDeviceSynchronize() == cudaSuccess;
        if (ok) {
          cudaMemcpy(back.data(), dst, bytes, cudaMemcpyDeviceToHost);
          ok = memcmp(back.data(), h.data(), bytes) == 0;
          if (!ok) snprintf(nb.why, sizeof(nb.why), "NVLS AllGather result mismatch on one device");
        }
      }
      if (!ok && !strstr(nb.why, "mismatch")) {
        snprintf(nb.why, sizeof(nb.why), "NVLS kernel failed: %s",
                 cudaGetErrorString(cudaGetLastError()));
      }
    }
    if (src) cudaFree(src);
    if (dst) cudaFree(dst);
    if (abort_word) cudaFree(abort_word);
    if (ok) snprintf(nb.why, sizeof(nb.why), "ok: multicast object + NVLS AllReduce and AllGather kernels");
  }
  say(nb.why);
  *available = ok ? 1 : 0;
  nvls_free(&nb);
  return flxSuccess;
}

}  // extern "C"
