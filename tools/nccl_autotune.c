/*
 * An NCCL-only program (nccl.h names, no FlexLink call at all) whose
 * AllReduce gets striped by the in-library balancer: 8 ranks on one GPU
 * through ncclCommInitAll (virtual ranks), a 64 MiB fp32 AllReduce issued in
 * ncclGroupStart/End, repeated.  The NVLink-path kernel is capped through the
 * environment (FLX_NVLINK_CTAS, BASELINE config 4's H800-like link ratio), so
 * the two-stage balancer inside libflexlink finds real PCIe headroom.
 *
 * Passes (prints "ok") when every result is exact and the last call put bytes
 * on the PCIe path — i.e. Stage 1 ran inside the library and kept a striped
 * split without the program ever calling flxSetShares.  The only FlexLink
 * symbol it touches is flxGetPathBytes, to observe the outcome.
 *
 *   gcc -std=c11 -Iinclude -I/usr/local/cuda/include tools/nccl_autotune.c \
 *       -Lpaper_2510_15882_b200 -lflexlink_nccl -lflexlink -lcudart ...
 */
#define _POSIX_C_SOURCE 200809L
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>

#include "flexlink.h"

#define N 8
#define COUNT (16u << 20) /* floats per rank: 64 MiB */
#define CALLS 120

static float value(int rank, size_t i) { return (float)((i * (rank + 3)) % 251) - 100.f; }

int main(void) {
  if (!getenv("FLX_NVLINK_CTAS")) setenv("FLX_NVLINK_CTAS", "2", 1);
  int devs[N] = {0};
  ncclComm_t comms[N];
  if (ncclCommInitAll(comms, N, devs) != ncclSuccess) {
    printf("init failed: %s\n", ncclGetLastError(NULL));
    return 1;
  }
  float* send[N];
  float* recv[N];
  float* h = (float*)malloc(COUNT * sizeof(float));
  for (int r = 0; r < N; ++r) {
    if (cudaMalloc((void**)&send[r], COUNT * sizeof(float)) != cudaSuccess) return 2;
    if (cudaMalloc((void**)&recv[r], COUNT * sizeof(float)) != cudaSuccess) return 2;
    for (size_t i = 0; i < COUNT; ++i) h[i] = value(r, i);
    cudaMemcpy(send[r], h, COUNT * sizeof(float), cudaMemcpyHostToDevice);
  }
  cudaStream_t s;
  cudaStreamCreate(&s);
  size_t pcie_calls = 0;
  for (int it = 0; it < CALLS; ++it) {
    if (ncclGroupStart() != ncclSuccess) return 3;
    for (int r = 0; r < N; ++r)
      if (ncclAllReduce(send[r], recv[r], COUNT, ncclFloat32, ncclSum, comms[r], s) != ncclSuccess) {
        printf("allreduce failed: %s\n", ncclGetLastError(comms[r]));
        return 4;
      }
    if (ncclGroupEnd() != ncclSuccess) {
      printf("group failed: %s\n", ncclGetLastError(NULL));
      return 5;
    }
    size_t bytes[3];
    flxGetPathBytes((flxComm_t)comms[0], bytes);
    pcie_calls += bytes[1] > 0;
  }
  cudaStreamSynchronize(s);
  size_t bytes[3];
  flxGetPathBytes((flxComm_t)comms[0], bytes);
  long bad = 0;
  for (int r = 0; r < N; ++r) {
    cudaMemcpy(h, recv[r], COUNT * sizeof(float), cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < COUNT; ++i) {
      float want = 0.f;
      for (int q = 0; q < N; ++q) want += value(q, i);
      bad += h[i] != want;
    }
  }
  printf("last call: nvlink %zu B, pcie %zu B; %zu of %d calls striped; %ld mismatches\n",
         bytes[0], bytes[1], pcie_calls, CALLS, bad);
  for (int r = 0; r < N; ++r) ncclCommDestroy(comms[r]);
  if (bad) return 6;
  if (bytes[1] == 0) return 7;
  printf("ok\n");
  return 0;
}
