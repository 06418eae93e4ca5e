/*
 * An unmodified-NCCL-style C program driving FlexLink through the NCCL names
 * (libflexlink_nccl.so) across two real processes: ncclGetUniqueId, fork,
 * ncclCommInitRank, ncclAllReduce / ncclAllGather / ncclReduceScatter,
 * ncclCommDestroy.  The only FlexLink-specific call is flxSetShares, which
 * puts every byte on the host-staged PCIe path: both processes share one GPU
 * here (FLX_ALLOW_SHARED_GPU), and the PCIe path runs only copy engines and
 * stream memory ops, so neither process's kernels spin on the other's.
 *
 *   gcc -std=c11 -I/usr/local/cuda/include -Iinclude tools/nccl_two_process.c \
 *       -Lpaper_2510_15882_b200 -lflexlink_nccl -lflexlink -L/usr/local/cuda/lib64 \
 *       -lcudart -Wl,-rpath,... -o tools/bin/nccl_two_process [config]
 * With "config" the communicators come from ncclCommInitRankConfig (non-blocking
 * flag, maxCTAs = 16), as frameworks such as PyTorch's ProcessGroupNCCL create
 * them.  Exit code 0 and "ok" when every result is exact on both ranks.
 */
#define _POSIX_C_SOURCE 200809L
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/wait.h>
#include <unistd.h>

#include "flexlink.h"

#define N 2
#define COUNT (1 << 18) /* floats per rank: a multiple of the alignment, all on PCIe */

static float value(int rank, size_t i) { return (float)((i * (rank + 3)) % 251) - 100.f; }

static int use_config = 0;

static int run(int rank, ncclUniqueId id) {
  if (cudaSetDevice(0) != cudaSuccess) return 10;
  ncclComm_t comm;
  if (use_config) {
    ncclConfig_t config = NCCL_CONFIG_INITIALIZER;
    config.blocking = 0;
    config.maxCTAs = 16;
    if (ncclCommInitRankConfig(&comm, N, id, rank, &config) != ncclSuccess) return 14;
    ncclResult_t async = ncclInProgress;
    if (ncclCommGetAsyncError(comm, &async) != ncclSuccess || async != ncclSuccess) return 15;
  } else if (ncclCommInitRank(&comm, N, id, rank) != ncclSuccess) {
    return 11;
  }
  const int pcie_only[3] = {0, 1000, 0};
  for (int op = flxCollAllReduce; op <= flxCollReduceScatter; ++op)
    if (flxSetShares((flxComm_t)comm, (flxCollOp_t)op, FLX_BUCKET_ALL, pcie_only) != flxSuccess)
      return 12;
  const size_t bytes = (size_t)N * COUNT * sizeof(float);
  float* h = (float*)malloc(bytes);
  float *send, *recv;
  if (cudaMalloc((void**)&send, bytes) != cudaSuccess) return 13;
  if (cudaMalloc((void**)&recv, bytes) != cudaSuccess) return 13;
  for (size_t i = 0; i < (size_t)N * COUNT; ++i) h[i] = value(rank, i);
  cudaMemcpy(send, h, bytes, cudaMemcpyHostToDevice);
  cudaStream_t s;
  cudaStreamCreate(&s);
  int bad = 0;
  for (int it = 0; it < 3; ++it) {
    /* AllReduce of the first COUNT elements */
    if (ncclAllReduce(send, recv, COUNT, ncclFloat32, ncclSum, comm, s) != ncclSuccess) return 20;
    cudaStreamSynchronize(s);
    cudaMemcpy(h, recv, COUNT * sizeof(float), cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < COUNT; ++i) bad += h[i] != value(0, i) + value(1, i);
    /* AllGather of the first COUNT elements */
    if (ncclAllGather(send, recv, COUNT, ncclFloat32, comm, s) != ncclSuccess) return 21;
    cudaStreamSynchronize(s);
    cudaMemcpy(h, recv, bytes, cudaMemcpyDeviceToHost);
    for (int r = 0; r < N; ++r)
      for (size_t i = 0; i < COUNT; ++i) bad += h[r * COUNT + i] != value(r, i);
    /* ReduceScatter of N blocks of COUNT */
    if (ncclReduceScatter(send, recv, COUNT, ncclFloat32, ncclSum, comm, s) != ncclSuccess)
      return 22;
    cudaStreamSynchronize(s);
    cudaMemcpy(h, recv, COUNT * sizeof(float), cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < COUNT; ++i) {
      const size_t g = (size_t)rank * COUNT + i;
      bad += h[i] != value(0, g) + value(1, g);
    }
    for (size_t i = 0; i < (size_t)N * COUNT; ++i) h[i] = value(rank, i);  /* restore */
  }
  if (ncclCommFinalize(comm) != ncclSuccess) return 29;
  if (ncclCommDestroy(comm) != ncclSuccess) return 30;
  free(h);
  return bad ? 40 : 0;
}

int main(int argc, char** argv) {
  use_config = argc > 1 && argv[1][0] == 'c';
  if (use_config) {  /* a config not set up by NCCL_CONFIG_INITIALIZER is refused */
    ncclConfig_t raw;
    memset(&raw, 0, sizeof(raw));
    ncclComm_t c = NULL;
    ncclUniqueId any;
    memset(&any, 0, sizeof(any));
    if (ncclCommInitRankConfig(&c, N, any, 0, &raw) != ncclInvalidArgument) return 4;
  }
  setenv("FLX_ALLOW_SHARED_GPU", "1", 1);
  setenv("FLX_SLOT_MB", "1", 1);
  setenv("FLX_PCIE_STAGE_MB", "8", 1);
  setenv("FLX_BOOT_TIMEOUT", "60", 1);
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return 1;  /* before fork: no CUDA yet */
  const pid_t child = fork();
  if (child < 0) return 2;
  if (child == 0) _exit(run(1, id));
  const int mine = run(0, id);
  int status = 0;
  waitpid(child, &status, 0);
  const int theirs = WIFEXITED(status) ? WEXITSTATUS(status) : 99;
  if (mine || theirs) {
    printf("rank0 %d rank1 %d\n", mine, theirs);
    return 3;
  }
  printf("ok\n");
  return 0;
}
