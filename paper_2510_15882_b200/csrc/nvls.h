// NVLink-SHARP multicast buffers for the NVLS AllReduce (nvls_kernels.cuh).
#pragma once

#include <cuda.h>

#include "args.h"
#include "internal.h"

namespace flx {

// Rendezvous block inside the multi-rank bootstrap header (world.cu).
struct NvlsBoot {
  int state;   // 0 pending, 1 rank 0 published the multicast handle, -1 failed
  int added;   // ranks past cuMulticastAddDevice (succeeded or not)
  int bound;   // ranks past binding + mapping (succeeded or not)
  int pad;
  int ok[kMaxRanks];  // 1 = this rank's buffer is bound and mapped
  CUmemFabricHandle handle;
  char why[128];
};

struct NvlsBuffer {
  bool on = false;
  char why[192] = "not attempted (FLX_NVLS=1 enables the NVLS AllReduce on multi-GPU worlds)";
  int device = 0;
  size_t size = 0;      // bytes mapped (flags + data)
  size_t capacity = 0;  // data bytes per call round
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  CUdeviceptr uc = 0, mcva = 0;
  bool added = false, bound = false, uc_mapped = false, mc_mapped = false;
  uint32_t* state = nullptr;  // device, per-CTA epochs
};

// Multi-rank setup through the bootstrap header; never fails the world:
// on any error `nb->on` stays false (identically on every rank) with the reason.
void nvls_setup_rank(NvlsBuffer* nb, NvlsBoot* boot, int rank, int nranks, int device,
                     size_t data_bytes, double timeout_s);
void nvls_free(NvlsBuffer* nb);
cudaError_t launch_nvls_allreduce(int dtype, const void* args, int nctas, cudaStream_t s);
cudaError_t launch_nvls_allgather(const void* args, size_t stride, int nctas, cudaStream_t s);
bool nvls_dtype_ok(int dtype);

}  // namespace flx
