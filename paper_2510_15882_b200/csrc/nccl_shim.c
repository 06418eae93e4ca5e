/*
 * libflexlink_nccl.so — NCCL-symbol front end for libflexlink.so.
 *
 * Compiled against the system /usr/include/nccl.h (NCCL 2.27.3, the version
 * the paper benchmarked), so the compiler itself checks that
 * every entry point below has NCCL's exact signature.  An application linked
 * against NCCL can be pointed at FlexLink for the calls below with
 * LD_PRELOAD=libflexlink_nccl.so (or by linking this library first); the
 * type values (ncclDataType_t, ncclRedOp_t, ncclResult_t, the 128-byte
 * ncclUniqueId) are identical to flexlink.h's, so arguments pass through
 * unchanged.
 *
 * A FlexLink communicator is not an ncclComm: every entry point below that
 * takes a communicator checks FlexLink's magic word (flxComm validation) and
 * rejects a real ncclComm_t with ncclInvalidArgument instead of dereferencing
 * it.  The NCCL calls FlexLink does not implement but that take a
 * communicator (Send, Recv, CommShrink, DevCommCreate,
 * buffer/window registration, PreMulSum ops) are DEFINED here and return
 * ncclInvalidUsage: without them a preloaded process would hand a FlexLink
 * communicator to the real libnccl, which would dereference it as its own
 * struct.  ncclCommInitRankConfig / ncclCommInitRankScalable (the init
 * frameworks such as PyTorch's ProcessGroupNCCL use) create FlexLink
 * communicators, honouring the config fields that map (below).  Calls without
 * a communicator that FlexLink does not provide (ncclMemAlloc/Free — plain
 * device memory from NCCL's allocator works with FlexLink's collectives —,
 * ncclGroupSimulateEnd, the pncl* profiling aliases) are not defined and
 * resolve to NCCL if it is loaded.
 */
#include <nccl.h>
#include <string.h>

#include "../../include/flexlink.h"

_Static_assert(sizeof(ncclUniqueId) == sizeof(flxUniqueId), "unique id size");
_Static_assert((int)ncclFloat32 == (int)flxFloat32 && (int)ncclBfloat16 == (int)flxBfloat16,
               "datatype codes");
_Static_assert((int)ncclSum == (int)flxSum && (int)ncclMin == (int)flxMin, "reduction codes");
_Static_assert((int)ncclAvg == FLX_OP_AVG, "average");
_Static_assert((int)ncclInvalidUsage == (int)flxInvalidUsage, "result codes");
_Static_assert(NCCL_SPLIT_NOCOLOR == FLX_SPLIT_NOCOLOR, "split no-color");

/* The NCCL API level this shim implements (the nccl.h it is compiled against),
 * not FlexLink's own version (flxGetVersion): callers such as PyTorch's
 * ProcessGroupNCCL pick their init path and feature set from it. */
ncclResult_t ncclGetVersion(int* version) {
  if (!version) return ncclInvalidArgument;
  *version = NCCL_VERSION_CODE;
  return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t result) {
  return flxGetErrorString((flxResult_t)result);
}

const char* ncclGetLastError(ncclComm_t comm) {
  (void)comm;
  return flxGetLastError();
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* uniqueId) {
  return (ncclResult_t)flxGetUniqueId((flxUniqueId*)uniqueId);
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId commId, int rank) {
  flxUniqueId id;
  memcpy(&id, &commId, sizeof(id));
  return (ncclResult_t)flxCommInitRank((flxComm_t*)comm, nranks, id, rank);
}

/* NCCL's config (nccl.h ncclConfig_t), where it maps onto FlexLink: maxCTAs caps
 * the NVLink-path kernel grid (flxSetNvlinkCtas, 1..64; NCCL also requires the
 * same config on every rank); blocking = 0 is satisfied by the blocking init (a
 * later ncclCommGetAsyncError reports ncclSuccess, never ncclInProgress).
 * cgaClusterSize, minCTAs, netName, splitShare, trafficClass, commName,
 * collnetEnable, CTAPolicy, shrinkShare and nvlsCTAs have no FlexLink meaning
 * (FLX_NVLS selects the NVLS path).  A config not set up with
 * NCCL_CONFIG_INITIALIZER is refused, as NCCL refuses it. */
static ncclResult_t init_with_config(ncclComm_t* comm, int nranks, ncclUniqueId commId, int rank,
                                     const ncclConfig_t* config) {
  if (config && config->magic != 0xcafebeef) {
    flxSetLastError("ncclConfig_t was not initialised with NCCL_CONFIG_INITIALIZER");
    return ncclInvalidArgument;
  }
  ncclResult_t r = ncclCommInitRank(comm, nranks, commId, rank);
  if (r != ncclSuccess || !config) return r;
  if (config->maxCTAs != NCCL_CONFIG_UNDEF_INT && config->maxCTAs > 0) {
    const int ctas = config->maxCTAs < 64 ? config->maxCTAs : 64;
    r = (ncclResult_t)flxSetNvlinkCtas((flxComm_t)*comm, ctas);
    if (r != ncclSuccess) {
      flxCommDestroy((flxComm_t)*comm);
      *comm = NULL;
    }
  }
  return r;
}

ncclResult_t ncclCommInitRankConfig(ncclComm_t* comm, int nranks, ncclUniqueId commId, int rank,
                                    ncclConfig_t* config) {
  return init_with_config(comm, nranks, commId, rank, config);
}

/* Several unique ids (one per bootstrap root in NCCL); every rank receives the
 * same array, so the first id names the FlexLink world identically everywhere. */
ncclResult_t ncclCommInitRankScalable(ncclComm_t* newcomm, int nranks, int myrank, int nId,
                                      ncclUniqueId* commIds, ncclConfig_t* config) {
  if (nId < 1 || !commIds) {
    flxSetLastError("ncclCommInitRankScalable needs at least one unique id");
    return ncclInvalidArgument;
  }
  return init_with_config(newcomm, nranks, commIds[0], myrank, config);
}

ncclResult_t ncclCommInitAll(ncclComm_t* comm, int ndev, const int* devlist) {
  return (ncclResult_t)flxCommInitAll((flxComm_t*)comm, ndev, devlist);
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  return (ncclResult_t)flxCommDestroy((flxComm_t)comm);
}

ncclResult_t ncclCommCount(const ncclComm_t comm, int* count) {
  return (ncclResult_t)flxCommCount((flxComm_t)comm, count);
}

ncclResult_t ncclCommCuDevice(const ncclComm_t comm, int* device) {
  return (ncclResult_t)flxCommCuDevice((flxComm_t)comm, device);
}

ncclResult_t ncclCommUserRank(const ncclComm_t comm, int* rank) {
  return (ncclResult_t)flxCommUserRank((flxComm_t)comm, rank);
}

ncclResult_t ncclAllReduce(const void* sendbuff, void* recvbuff, size_t count,
                           ncclDataType_t datatype, ncclRedOp_t op, ncclComm_t comm,
                           cudaStream_t stream) {
  if ((int)op > (int)ncclAvg) return ncclInvalidArgument; /* PreMulSum ops */
  return (ncclResult_t)flxAllReduce(sendbuff, recvbuff, count, (flxDataType_t)datatype,
                                    (flxRedOp_t)op, (flxComm_t)comm, stream);
}

ncclResult_t ncclAllGather(const void* sendbuff, void* recvbuff, size_t sendcount,
                           ncclDataType_t datatype, ncclComm_t comm, cudaStream_t stream) {
  return (ncclResult_t)flxAllGather(sendbuff, recvbuff, sendcount, (flxDataType_t)datatype,
                                    (flxComm_t)comm, stream);
}

ncclResult_t ncclReduceScatter(const void* sendbuff, void* recvbuff, size_t recvcount,
                               ncclDataType_t datatype, ncclRedOp_t op, ncclComm_t comm,
                               cudaStream_t stream) {
  if ((int)op > (int)ncclAvg) return ncclInvalidArgument; /* PreMulSum ops */
  return (ncclResult_t)flxReduceScatter(sendbuff, recvbuff, recvcount, (flxDataType_t)datatype,
                                        (flxRedOp_t)op, (flxComm_t)comm, stream);
}

/* NCCL 2.28 added ncclAlltoAll / ncclGather / ncclScatter and the device
 * communicator calls; PyTorch built against 2.28 (the bundled libnccl) imports
 * ncclAlltoAll for all_to_all_single and ncclDevCommCreate/Destroy.  The shim
 * compiles against the system nccl.h (2.27.3), so it declares them here with
 * 2.28's signatures (device-communicator types as opaque pointers) — defined,
 * so a preloaded process never hands a FlexLink communicator to libnccl. */
#if NCCL_VERSION_CODE < 22800
ncclResult_t ncclAlltoAll(const void* sendbuff, void* recvbuff, size_t count,
                          ncclDataType_t datatype, ncclComm_t comm, cudaStream_t stream);
ncclResult_t ncclGather(const void* sendbuff, void* recvbuff, size_t count,
                        ncclDataType_t datatype, int root, ncclComm_t comm, cudaStream_t stream);
ncclResult_t ncclScatter(const void* sendbuff, void* recvbuff, size_t count,
                         ncclDataType_t datatype, int root, ncclComm_t comm, cudaStream_t stream);
ncclResult_t ncclDevCommCreate(ncclComm_t comm, const void* reqs, void* outDevComm);
ncclResult_t ncclDevCommDestroy(ncclComm_t comm, const void* devComm);
#endif

/* ncclAlltoAll: block j of sendbuff to rank j, block i of recvbuff from rank i —
 * exactly flxAllToAll (striped per block) */
ncclResult_t ncclAlltoAll(const void* sendbuff, void* recvbuff, size_t count,
                          ncclDataType_t datatype, ncclComm_t comm, cudaStream_t stream) {
  return (ncclResult_t)flxAllToAll(sendbuff, recvbuff, count, (flxDataType_t)datatype,
                                   (flxComm_t)comm, stream);
}

ncclResult_t ncclCommFinalize(ncclComm_t comm) {
  return (ncclResult_t)flxCommFinalize((flxComm_t)comm);
}

ncclResult_t ncclCommAbort(ncclComm_t comm) { return (ncclResult_t)flxCommAbort((flxComm_t)comm); }

ncclResult_t ncclCommGetAsyncError(ncclComm_t comm, ncclResult_t* asyncError) {
  flxResult_t e = flxSuccess;
  const flxResult_t rc = flxCommGetAsyncError((flxComm_t)comm, &e);
  if (rc == flxSuccess && asyncError) *asyncError = (ncclResult_t)e;
  return (ncclResult_t)rc;
}

ncclResult_t ncclGroupStart(void) { return (ncclResult_t)flxGroupStart(); }

ncclResult_t ncclGroupEnd(void) { return (ncclResult_t)flxGroupEnd(); }

/* ---- NCCL calls that take a communicator but are not FlexLink collectives.
 * Refused loudly (ncclInvalidUsage; ncclGetLastError says why) instead of
 * falling through to libnccl with a FlexLink handle. */
static ncclResult_t unsupported(ncclComm_t comm, const char* what) {
  int n = 0;
  /* flxCommCount validates the handle (magic word) and records the error */
  if (flxCommCount((flxComm_t)comm, &n) != flxSuccess) return ncclInvalidArgument;
  flxSetLastError(what);
  return ncclInvalidUsage;
}

ncclResult_t ncclReduce(const void* sendbuff, void* recvbuff, size_t count,
                        ncclDataType_t datatype, ncclRedOp_t op, int root, ncclComm_t comm,
                        cudaStream_t stream) {
  if ((int)op > (int)ncclAvg) return ncclInvalidArgument; /* PreMulSum ops */
  return (ncclResult_t)flxReduce(sendbuff, recvbuff, count, (flxDataType_t)datatype,
                                 (flxRedOp_t)op, root, (flxComm_t)comm, stream);
}

/* ncclBroadcast / ncclBcast: FlexLink's bit-exact broadcast (flxBroadcast) */
ncclResult_t ncclBcast(void* buff, size_t count, ncclDataType_t datatype, int root,
                       ncclComm_t comm, cudaStream_t stream) {
  return (ncclResult_t)flxBroadcast(buff, buff, count, (flxDataType_t)datatype, root,
                                    (flxComm_t)comm, stream);
}

ncclResult_t ncclBroadcast(const void* sendbuff, void* recvbuff, size_t count,
                           ncclDataType_t datatype, int root, ncclComm_t comm,
                           cudaStream_t stream) {
  return (ncclResult_t)flxBroadcast(sendbuff, recvbuff, count, (flxDataType_t)datatype, root,
                                    (flxComm_t)comm, stream);
}

ncclResult_t ncclGather(const void* sendbuff, void* recvbuff, size_t count,
                        ncclDataType_t datatype, int root, ncclComm_t comm, cudaStream_t stream) {
  return (ncclResult_t)flxGather(sendbuff, recvbuff, count, (flxDataType_t)datatype, root,
                                 (flxComm_t)comm, stream);
}

ncclResult_t ncclScatter(const void* sendbuff, void* recvbuff, size_t count,
                         ncclDataType_t datatype, int root, ncclComm_t comm, cudaStream_t stream) {
  return (ncclResult_t)flxScatter(sendbuff, recvbuff, count, (flxDataType_t)datatype, root,
                                  (flxComm_t)comm, stream);
}

ncclResult_t ncclDevCommCreate(ncclComm_t comm, const void* reqs, void* outDevComm) {
  (void)reqs; (void)outDevComm;
  return unsupported(comm, "ncclDevCommCreate (NCCL's device API) is not implemented by FlexLink");
}

ncclResult_t ncclDevCommDestroy(ncclComm_t comm, const void* devComm) {
  (void)devComm;
  return unsupported(comm, "ncclDevCommDestroy (NCCL's device API) is not implemented by FlexLink");
}

ncclResult_t ncclSend(const void* sendbuff, size_t count, ncclDataType_t datatype, int peer,
                      ncclComm_t comm, cudaStream_t stream) {
  (void)sendbuff; (void)count; (void)datatype; (void)peer; (void)stream;
  return unsupported(comm, "ncclSend is not implemented by FlexLink");
}

ncclResult_t ncclRecv(void* recvbuff, size_t count, ncclDataType_t datatype, int peer,
                      ncclComm_t comm, cudaStream_t stream) {
  (void)recvbuff; (void)count; (void)datatype; (void)peer; (void)stream;
  return unsupported(comm, "ncclRecv is not implemented by FlexLink");
}

/* ncclCommSplit: FlexLink's own split (collective over the parent); the config
 * maps as at init (maxCTAs).  NCCL_SPLIT_NOCOLOR == FLX_SPLIT_NOCOLOR. */
ncclResult_t ncclCommSplit(ncclComm_t comm, int color, int key, ncclComm_t* newcomm,
                           ncclConfig_t* config) {
  if (config && config->magic != 0xcafebeef) {
    flxSetLastError("ncclConfig_t was not initialised with NCCL_CONFIG_INITIALIZER");
    return ncclInvalidArgument;
  }
  ncclResult_t r = (ncclResult_t)flxCommSplit((flxComm_t)comm, color, key, (flxComm_t*)newcomm);
  if (r != ncclSuccess || !newcomm || !*newcomm || !config) return r;
  if (config->maxCTAs != NCCL_CONFIG_UNDEF_INT && config->maxCTAs > 0) {
    const int ctas = config->maxCTAs < 64 ? config->maxCTAs : 64;
    r = (ncclResult_t)flxSetNvlinkCtas((flxComm_t)*newcomm, ctas);
    if (r != ncclSuccess) {
      flxCommDestroy((flxComm_t)*newcomm);
      *newcomm = NULL;
    }
  }
  return r;
}

ncclResult_t ncclCommShrink(ncclComm_t comm, int* excludeRanksList, int excludeRanksCount,
                            ncclComm_t* newcomm, ncclConfig_t* config, int shrinkFlags) {
  (void)excludeRanksList; (void)excludeRanksCount; (void)config; (void)shrinkFlags;
  if (newcomm) *newcomm = NULL;
  return unsupported(comm, "ncclCommShrink is not implemented by FlexLink");
}

ncclResult_t ncclCommRegister(const ncclComm_t comm, void* buff, size_t size, void** handle) {
  (void)buff; (void)size;
  if (handle) *handle = NULL;
  return unsupported(comm, "ncclCommRegister is not implemented by FlexLink");
}

ncclResult_t ncclCommDeregister(const ncclComm_t comm, void* handle) {
  (void)handle;
  return unsupported(comm, "ncclCommDeregister is not implemented by FlexLink");
}

ncclResult_t ncclCommWindowRegister(ncclComm_t comm, void* buff, size_t size, ncclWindow_t* win,
                                    int winFlags) {
  (void)buff; (void)size; (void)winFlags;
  if (win) *win = NULL;
  return unsupported(comm, "ncclCommWindowRegister is not implemented by FlexLink");
}

ncclResult_t ncclCommWindowDeregister(ncclComm_t comm, ncclWindow_t win) {
  (void)win;
  return unsupported(comm, "ncclCommWindowDeregister is not implemented by FlexLink");
}

ncclResult_t ncclRedOpCreatePreMulSum(ncclRedOp_t* op, void* scalar, ncclDataType_t datatype,
                                      ncclScalarResidence_t residence, ncclComm_t comm) {
  (void)op; (void)scalar; (void)datatype; (void)residence;
  return unsupported(comm, "PreMulSum reduction ops are not implemented by FlexLink");
}

ncclResult_t ncclRedOpDestroy(ncclRedOp_t op, ncclComm_t comm) {
  (void)op;
  return unsupported(comm, "PreMulSum reduction ops are not implemented by FlexLink");
}
