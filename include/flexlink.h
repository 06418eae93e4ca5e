/*
 * flexlink.h — C-ABI of the B200-native FlexLink data plane (libflexlink.so).
 *
 * NCCL-shaped striped collectives: every AllReduce / AllGather message is
 * split by integer granule shares (1000 total) into contiguous per-path byte
 * slices — host-staged PCIe at offset 0, then RDMA, then NVLink last (it
 * takes partition()'s remainder at its end, so the secondary slices stay on
 * the alignment grid for any message length) — and
 * each slice runs a complete collective on its own path concurrently.
 *
 * The reference ("linkstripe", /root/reference/pkg/src/linkstripe) is a CPU
 * simulator whose data plane is the closed-form `simulate_collective`
 * (collectives.py:136-186); this library is the real executor that replaces
 * it.  Each entry point below names the reference interface it stands in for.
 *
 * Conventions (identical to /usr/include/nccl.h so the types are
 * interchangeable):
 *   - flxResult_t values equal ncclResult_t (nccl.h:40-48);
 *   - flxDataType_t values equal ncclDataType_t; flxRedOp_t equals ncclRedOp_t
 *     for sum/prod/max/min;
 *   - flxUniqueId is 128 opaque bytes like ncclUniqueId (nccl.h:36-37);
 *   - calls are stream-ordered and asynchronous; in-place is
 *     sendbuff == recvbuff (AllReduce) or sendbuff == recvbuff + rank*sendcount
 *     (AllGather);
 *   - no CPU fallback: without a usable sm_100 device every call fails.
 *
 * Virtual ranks: flxCommInitAll() accepts the SAME device more than once.
 * Ranks that share a device form a clique whose collectives run as one fused
 * kernel launch (plus one host-staged pipeline), driven from a single thread
 * inside flxGroupStart()/flxGroupEnd() exactly like ncclCommInitAll +
 * ncclGroupStart/End.  This is how an N-rank collective is exercised on one
 * GPU ("1-GPU tests where the N peers are N local buffers").
 */
#ifndef FLEXLINK_H_
#define FLEXLINK_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FLX_VERSION_CODE 10000   /* 1.0.0 */
#define FLX_UNIQUE_ID_BYTES 128
#define FLX_NUM_PATHS 3
#define FLX_GRANULE_TOTAL 1000   /* collectives.py:23 */
#define FLX_MAX_VIRTUAL_RANKS 16
#define FLX_BUCKET_ALL (-2)      /* flxSetShares: apply to every size bucket */

typedef struct { char internal[FLX_UNIQUE_ID_BYTES]; } flxUniqueId;
typedef struct flxComm* flxComm_t;

/* == ncclResult_t (nccl.h:40-48) */
typedef enum {
  flxSuccess = 0,
  flxUnhandledCudaError = 1,
  flxSystemError = 2,
  flxInternalError = 3,   /* also: semaphore wait timed out */
  flxInvalidArgument = 4,
  flxInvalidUsage = 5,
  flxRemoteError = 6,
  flxInProgress = 7
} flxResult_t;

/* == ncclDataType_t */
typedef enum {
  flxInt8 = 0, flxUint8 = 1, flxInt32 = 2, flxUint32 = 3, flxInt64 = 4,
  flxUint64 = 5, flxFloat16 = 6, flxFloat32 = 7, flxFloat64 = 8, flxBfloat16 = 9,
  flxNumTypes = 10
} flxDataType_t;

/* == ncclRedOp_t for the four supported operators */
typedef enum { flxSum = 0, flxProd = 1, flxMax = 2, flxMin = 3, flxNumOps = 4 } flxRedOp_t;
/* == ncclAvg: AllReduce / ReduceScatter only — the striped sum, then the
 * result divided by nranks on the caller's stream (floating types: one
 * rounding of fl(sum) / n in the accumulation type; integers: C division,
 * as NCCL's sum-then-divide for integers) */
#define FLX_OP_AVG 4

/* == linkstripe PathKind (topo.py:18-31); also the tie-break order */
typedef enum { flxPathNvlink = 0, flxPathPcie = 1, flxPathRdma = 2 } flxPath_t;

/* == linkstripe CollectiveOp (collectives.py:26-28), plus ReduceScatter
 * (ring_steps N-1) */
typedef enum {
  flxCollAllReduce = 0,
  flxCollAllGather = 1,
  flxCollReduceScatter = 2,
  flxCollAllToAll = 3
} flxCollOp_t;

/* ---- library / errors --------------------------------------------------- */
flxResult_t flxGetVersion(int* version);
const char* flxGetErrorString(flxResult_t result);
/* Last detailed error message of this thread (never NULL). */
const char* flxGetLastError(void);
/* Replace this thread's detailed error message (the NCCL shim uses it to
 * explain the NCCL calls FlexLink refuses). */
void flxSetLastError(const char* message);

/* ---- communicators (ncclGetUniqueId / ncclCommInitRank / ncclCommInitAll /
 *      ncclCommDestroy shapes, nccl.h) ----------------------------------- */
flxResult_t flxGetUniqueId(flxUniqueId* uniqueId);
/* One process (or thread) per GPU; collective over the nranks callers. */
flxResult_t flxCommInitRank(flxComm_t* comm, int nranks, flxUniqueId commId, int rank);
/* Single process, ndev ranks; repeated devices become virtual ranks. */
flxResult_t flxCommInitAll(flxComm_t* comms, int ndev, const int* devlist);
/* All nranks ranks of a flxCommInitRank-style world emulated on ONE device:
 * the multi-rank engine (peer-mapped scratch + flags kernels, host-hub PCIe
 * staging with cross-rank token handshakes) with every peer pointer local
 * and the NVLink-path kernel launched cooperatively over all ranks.  Driven
 * like flxCommInitAll (one group per collective).  For testing the N-GPU code
 * path on a single GPU; set CUDA_DEVICE_MAX_CONNECTIONS>=3*nranks+1. */
flxResult_t flxCommInitLoopback(flxComm_t* comms, int nranks, int device);
/* Loopback over another process's memory (bootstrap self-test of the rank
 * kernels on CUDA-IPC-mapped peer memory): a helper process calls
 * flxDebugHostRemoteRanks, which allocates ranks 1..nranks-1's scratch and
 * flag blocks on `device`, exports their IPC handles under `id` and blocks
 * until the loopback world built over them is destroyed (or `seconds`);
 * flxCommInitLoopbackIpc builds that world in this process — rank 0's memory
 * local, the others IPC mappings — driven like flxCommInitLoopback.  Only
 * this process launches kernels. */
flxResult_t flxDebugHostRemoteRanks(int nranks, int device, flxUniqueId id, double seconds);
flxResult_t flxCommInitLoopbackIpc(flxComm_t* comms, int nranks, int device, flxUniqueId id);
flxResult_t flxCommDestroy(flxComm_t comm);
/* ncclCommSplit (nccl.h ncclCommSplit): collective over every rank of `comm`
 * (a flxCommInitRank communicator).  Ranks passing the same `color` form a new
 * communicator, ranked by `key` (ties: the parent rank); FLX_SPLIT_NOCOLOR
 * joins none and gets *newcomm = NULL.  The new communicator bootstraps like
 * flxCommInitRank on the parent's device, under an id derived from the
 * parent's id, the split's sequence number and the color. */
#define FLX_SPLIT_NOCOLOR (-1)
flxResult_t flxCommSplit(flxComm_t comm, int color, int key, flxComm_t* newcomm);
/* ncclCommAbort (nccl.h:186): stop waiting for peers — kernels still spinning
 * on a peer flag give up at once, the destroy barrier is skipped — then free
 * everything like flxCommDestroy.  For a rank that saw flxInternalError. */
flxResult_t flxCommAbort(flxComm_t comm);
/* ncclCommFinalize (nccl.h:177): block until the comm's internal side streams
 * (PCIe copies, reduce-on-receive) are idle; flxInternalError if a peer wait
 * timed out.  Collectives stay stream-ordered on the caller's streams. */
flxResult_t flxCommFinalize(flxComm_t comm);
flxResult_t flxCommCount(const flxComm_t comm, int* count);
flxResult_t flxCommUserRank(const flxComm_t comm, int* rank);
flxResult_t flxCommCuDevice(const flxComm_t comm, int* device);
/* ncclCommGetAsyncError (nccl.h:227): flxInternalError once a multi-rank
 * kernel of this comm gave up waiting for a peer (FLX_TIMEOUT_S), else
 * flxSuccess.  Virtual-rank comms never time out. */
flxResult_t flxCommGetAsyncError(flxComm_t comm, flxResult_t* async_error);

/* ---- collectives --------------------------------------------------------
 * Replace linkstripe `simulate_collective(topo, spec, shares)`
 * (collectives.py:136-186): the shares come from the comm's share table
 * (keyed by op and size_bucket, collectives.py:189-204), bytes are split by
 * `partition` (collectives.py:93-114), and each path's completion is recorded
 * with CUDA events for flxGetPathTimes (PathTimingReport, collectives.py:117-133).
 * Shapes: ncclAllReduce (nccl.h:392-393), ncclAllGather (nccl.h:425-426). */
flxResult_t flxAllReduce(const void* sendbuff, void* recvbuff, size_t count,
                         flxDataType_t datatype, flxRedOp_t op, flxComm_t comm,
                         cudaStream_t stream);
flxResult_t flxAllGather(const void* sendbuff, void* recvbuff, size_t sendcount,
                         flxDataType_t datatype, flxComm_t comm, cudaStream_t stream);
/* ncclReduceScatter shape (nccl.h:408-410): sendbuff holds nranks*recvcount
 * elements, rank r receives the fold of block r; in place when
 * recvbuff == sendbuff + rank*recvcount.  Partitioned per recv block. */
flxResult_t flxReduceScatter(const void* sendbuff, void* recvbuff, size_t recvcount,
                             flxDataType_t datatype, flxRedOp_t op, flxComm_t comm,
                             cudaStream_t stream);
/* AllToAll: sendbuff holds nranks blocks of `count` elements, block j goes to
 * rank j; recvbuff block i comes from rank i.  Not in place.  Partitioned per
 * block. */
flxResult_t flxAllToAll(const void* sendbuff, void* recvbuff, size_t count,
                        flxDataType_t datatype, flxComm_t comm, cudaStream_t stream);
/* ncclReduce (nccl.h ncclReduce): the fold of every rank's sendbuff lands in
 * rank `root`'s recvbuff (unused elsewhere; in place when sendbuff == recvbuff
 * on the root).  A striped AllReduce whose non-root result goes to
 * stream-ordered scratch (cudaMallocAsync, freed after the collective). */
flxResult_t flxReduce(const void* sendbuff, void* recvbuff, size_t count,
                      flxDataType_t datatype, flxRedOp_t op, int root, flxComm_t comm,
                      cudaStream_t stream);
/* ncclGather / ncclScatter (NCCL 2.28): Gather = an AllGather whose non-root
 * output goes to stream-ordered scratch (the root's recvbuff holds rank i's
 * count elements at i*count); Scatter = an AllToAll in which only the root's
 * blocks are kept, block `root` of the result copied to recvbuff.  For
 * completeness of the NCCL surface, not a hot path (N times a tree's traffic). */
flxResult_t flxGather(const void* sendbuff, void* recvbuff, size_t count,
                      flxDataType_t datatype, int root, flxComm_t comm, cudaStream_t stream);
flxResult_t flxScatter(const void* sendbuff, void* recvbuff, size_t count,
                       flxDataType_t datatype, int root, flxComm_t comm, cudaStream_t stream);
/* ncclBroadcast (nccl.h ncclBroadcast): rank `root`'s sendbuff (count
 * elements) lands in every rank's recvbuff; in place when sendbuff == recvbuff.
 * Runs as one striped AllReduce of the bytes with MAX over uint8, the non-roots
 * contributing zeros — bit-exact for any dtype (-0.0 and NaN payloads kept).
 * Twice a ring broadcast's traffic: for state sync (DDP's construction), not a
 * hot path. */
flxResult_t flxBroadcast(const void* sendbuff, void* recvbuff, size_t count,
                         flxDataType_t datatype, int root, flxComm_t comm, cudaStream_t stream);
/* Convenience for single-process communicator sets (flxCommInitAll /
 * flxCommInitLoopback): the same collective on every comms[i] with
 * sendbuffs[i]/recvbuffs[i] in ONE call — exactly flxGroupStart + n calls +
 * flxGroupEnd, minus n+1 host crossings.  `op` is ignored for gather/alltoall. */
flxResult_t flxGroupCollective(flxCollOp_t coll, flxComm_t* comms, int n,
                               const void* const* sendbuffs, void* const* recvbuffs,
                               size_t count, flxDataType_t datatype, flxRedOp_t op,
                               cudaStream_t stream);
flxResult_t flxGroupStart(void);
flxResult_t flxGroupEnd(void);

/* ---- balancer plumbing ---------------------------------------------------
 * Shares are ShareDistribution.granules (collectives.py:55-90) as
 * {nvlink, pcie, rdma}, summing to 1000.  bucket = size_bucket(bytes)
 * (floor(log2)), or FLX_BUCKET_ALL.  Every rank must install identical
 * shares (the Python layer agrees them across ranks first).  Setting shares
 * PINS the bucket (or every bucket): the in-library balancer
 * (flexlink_tuner.h) leaves pinned buckets alone; granules == NULL unpins. */
flxResult_t flxSetShares(flxComm_t comm, flxCollOp_t op, int bucket, const int granules[3]);
flxResult_t flxGetShares(flxComm_t comm, flxCollOp_t op, int bucket, int granules[3]);
/* Per-path duration (ms, collective start -> path done) of the most recent
 * call on this comm; blocks until that call finished.  A path that carried
 * no bytes reports 0.  (PathTimingReport.durations, collectives.py:117-133) */
flxResult_t flxGetPathTimes(flxComm_t comm, float ms[3]);
/* The same for the last min(max_calls, calls issued, 64) calls, oldest first:
 * ms[3*i + path].  Blocks until those calls finished.  Lets a caller time a
 * run of calls without synchronising between them. */
flxResult_t flxGetPathTimesHistory(flxComm_t comm, int max_calls, float* ms, int* n);
/* Per-rank bytes each path carried in the most recent call (partition()). */
flxResult_t flxGetPathBytes(flxComm_t comm, size_t bytes[3]);
/* Byte alignment of every secondary-path slice (partition's `alignment`
 * argument) that this comm applies for `op`. */
flxResult_t flxGetAlignment(flxComm_t comm, flxCollOp_t op, size_t* alignment);

/* ---- path configuration --------------------------------------------------
 * nctas: CTAs of the NVLink-path kernel (0 = automatic).  Config 4 caps it to
 * emulate a slower NVLink.  Must match on all ranks. */
flxResult_t flxSetNvlinkCtas(flxComm_t comm, int nctas);
/* enabled = 1 (default): every collective records per-path CUDA events, read
 * back by flxGetPathTimes / flxGetPathTimesHistory (Stage 1 / Stage 2's
 * MeasurePathTimings).  0: no timing events — a timed event record costs as
 * much host time as a kernel launch, so small-message callers that do not
 * rebalance at run time save ~5 us per call; path times then read as 0.
 * Must match on all ranks of a group. */
flxResult_t flxSetTiming(flxComm_t comm, int enabled);
/* PCIe staging: bytes per chunk per rank and ring depth (1 or 2 buffers;
 * PipelineSpec, staging.py:24-42).  Must match on all ranks. */
flxResult_t flxSetStaging(flxComm_t comm, size_t chunk_bytes, int buffers);
/* Which optional paths this build/box can use: bit p set => path p usable. */
flxResult_t flxGetPathMask(flxComm_t comm, int* mask);
/* NVLink-SHARP (in-switch reduction, multimem.ld_reduce / multimem.st).
 * flxNvlsProbe: can `device` make a multicast object and run the NVLS kernel
 * on it (checked end to end on a one-device object)?  *available 0/1 and the
 * reason (e.g. the driver's error for cuMulticastCreate).  flxCommGetNvls:
 * whether this multi-GPU communicator runs its AllReduce sums on NVLS
 * (opt-in FLX_NVLS=1 on every rank; off, with the reason, where the box
 * cannot).  Results of NVLS sums are within 1 ulp of the fixed-order fold
 * (the switch picks the order); exact for integer-valued data. */
flxResult_t flxNvlsProbe(int device, int* available, char* reason, size_t reason_len);
flxResult_t flxCommGetNvls(flxComm_t comm, int* on, char* reason, size_t reason_len);
/* Number of device kernels this library has launched (process-wide). */
flxResult_t flxGetLaunchCount(unsigned long long* count);
/* Bootstrap self-test (multi-rank comms only): write=1 copies `bytes` from
 * buf into this rank's scratch head (host_region=0) or shared host staging
 * region (host_region=1); write=0 reads peer `peer`'s through the CUDA-IPC
 * mapping / the shared segment.  Plain copies; no collective runs. */
flxResult_t flxCommDebugPeer(flxComm_t comm, int peer, int host_region, int write, void* buf,
                             size_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* FLEXLINK_H_ */
