// Host-side internals shared by the translation units of libflexlink.so.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <cstdarg>
#include <map>
#include <string>
#include <vector>

#include "../../include/flexlink.h"
#include "../../include/flexlink_tuner.h"

namespace flx {

struct FoldArgs;
struct FanoutArgs;
struct RowsArgs;
struct XposeArgs;
cudaError_t launch_xpose(const XposeArgs& a, int grid, cudaStream_t s);
cudaError_t launch_fold(int dtype, int op, const FoldArgs& a, int grid, cudaStream_t s);
cudaError_t launch_rows(int dtype, int op, const RowsArgs& a, int grid, cudaStream_t s);
cudaError_t launch_fanout(const FanoutArgs& a, int grid, cudaStream_t s);
cudaError_t launch_div(int dtype, void* buf, size_t count, int n, cudaStream_t s);
extern std::atomic<unsigned long long> g_launches;

// ---- errors
flxResult_t fail(flxResult_t code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));

#define FLX_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return ::flx::fail(flxUnhandledCudaError, "%s: %s (%s:%d)", #call,                  \
                         cudaGetErrorString(e_), __FILE__, __LINE__);                     \
  } while (0)

#define FLX_TRY(call)                  \
  do {                                 \
    flxResult_t r_ = (call);           \
    if (r_ != flxSuccess) return r_;   \
  } while (0)

// ---- the caller's CUDA context is restored on return (NCCL's rule): entry
// points switch devices internally (cudaSetDevice) — a multi-device process, or
// a thread that never touched CUDA (a framework's watchdog), must find its
// current context unchanged afterwards, and no context is left bound on a device
// the caller never used.  Entry points that never touch CUDA (flxGetUniqueId,
// flxCommGetAsyncError) take no guard: its driver lookup initialises CUDA, and
// ncclGetUniqueId must stay fork-safe (a parent makes the id, then forks ranks)
struct CtxGuard {
  CUcontext saved = nullptr;
  bool ok = false;
  CtxGuard();
  ~CtxGuard();
  CtxGuard(const CtxGuard&) = delete;
  CtxGuard& operator=(const CtxGuard&) = delete;
};

// ---- driver stream memory ops (resolved at run time; no -lcuda)
struct MemOps {
  CUresult (*wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  bool ok = false;
};
const MemOps& memops();
// Load every kernel of the module that contains `kernel` (one module per
// translation unit) into the current device's context.  CUDA's lazy loading
// otherwise loads a kernel at its first launch, and that load waits behind
// work already queued on the device — a PCIe leg parked on a peer's token, a
// rank kernel spinning on a peer — so a first launch could block the host
// thread (and a cudaFuncSetAttribute at launch time likewise).  NCCL does the
// same at init (cudaFuncGetAttributes on its kernels).
cudaError_t preload_module(const void* kernel);
// Every module of libflexlink on the current device, once per device.
cudaError_t preload_all_kernels();
// per-translation-unit anchors (each loads its own module)
cudaError_t preload_launch_cu();
cudaError_t preload_world_cu();
cudaError_t preload_nvls_cu();
flxResult_t sem_wait_geq(cudaStream_t s, uint32_t* word, uint32_t value);
flxResult_t sem_wait_eq(cudaStream_t s, uint32_t* word, uint32_t value);
flxResult_t sem_write(cudaStream_t s, uint32_t* word, uint32_t value);

size_t dtype_size(int dtype);
// largest automatic PCIe chunk per member (pick_chunk)
constexpr size_t kMaxAutoChunk = 12 << 20;

// ---- share table (ShareTable, collectives.py:189-204)
using Granules = std::array<int, FLX_NUM_PATHS>;
int size_bucket(size_t bytes);
struct ShareTable {
  Granules fallback{{FLX_GRANULE_TOTAL, 0, 0}};
  bool fallback_pinned = false;  // flxSetShares(FLX_BUCKET_ALL): every bucket pinned
  std::map<std::pair<int, int>, Granules> entries;  // (op, bucket) -> granules (pinned)
  Granules lookup(int op, size_t bytes) const;
  // the user fixed this bucket's split (flxSetShares): the autotuner leaves it alone
  bool pinned(int op, size_t bytes) const {
    return fallback_pinned || entries.count({op, size_bucket(bytes)});
  }
};
// partition (collectives.py:93-114): per-path bytes, floored to alignment,
// remainder to NVLink.
std::array<size_t, FLX_NUM_PATHS> partition(size_t bytes, const Granules& g, size_t alignment);
// Byte offset of every path's slice inside a rank's message.  The secondary
// slices come first (PCIe at 0, then RDMA): partition() makes each a multiple
// of the alignment, so both start 16 B aligned whenever the user buffer is.
// NVLink comes last and absorbs partition()'s remainder at its END — a ragged
// message length never shifts the copy-engine/reduce-on-receive slices off
// the 16 B grid (their kernels would otherwise fall back to scalar forms).
// The reference fixes per-path byte COUNTS only (collectives.py:93-114); the
// placement is this executor's choice.
inline std::array<size_t, FLX_NUM_PATHS> path_offsets(const std::array<size_t, FLX_NUM_PATHS>& split) {
  return {{split[1] + split[2], 0, split[1]}};
}

// FLX_SHARES="nvlink,pcie[,rdma]" (granules summing to FLX_GRANULE_TOTAL): every
// collective's every bucket pinned to this split at comm creation, as
// flxSetShares(FLX_BUCKET_ALL) would — for programs that only use the NCCL names
// (e.g. PyTorch's ProcessGroupNCCL under LD_PRELOAD).  *set = false when unset;
// malformed values fail comm creation.  Multi-rank worlds check it across ranks.
flxResult_t env_shares(Granules* g, bool* set);
inline uint64_t pack_env_shares(const Granules& g, bool set) {
  return set ? (1ull << 48) | (uint64_t)g[0] | (uint64_t)g[1] << 16 | (uint64_t)g[2] << 32 : 0;
}

struct Comm;
class AutoTuner;

// Ranks living in this process on one device.  With virtual ranks (repeated
// device in flxCommInitAll) there are several members and every collective is
// a single fused launch over all of them.
struct Clique {
  int device = 0;
  int sm_count = 0;
  std::vector<Comm*> members;  // index = position in clique == rank
  cudaStream_t d2h = nullptr;  // PCIe path: producer copies
  cudaStream_t h2d = nullptr;  // PCIe path: consumer copies
  cudaStream_t red = nullptr;  // PCIe path: reduce-on-receive / fan-out kernels
  // [mode][slot]: mode 1 = recorded inside a CUDA-graph capture (such an event
  // may not be awaited by eager work afterwards, so the two modes never share)
  cudaEvent_t ev_landed[2][2] = {};  // H2D of slot b done
  cudaEvent_t ev_folded[2][2] = {};  // fold of slot b done (slot reusable)
  cudaEvent_t ev_filled[2] = {nullptr, nullptr};   // capture-mode semFull
  cudaEvent_t ev_drained[2] = {nullptr, nullptr};  // capture-mode semEmpty
  // per-call timing ring: call k uses slot k % kTimingSlots
  static constexpr int kTimingSlots = 64;
  struct Timing {
    cudaEvent_t start = nullptr, nv = nullptr, pcie = nullptr;
    bool used[FLX_NUM_PATHS] = {false, false, false};
  };
  Timing timing[kTimingSlots];
  uint64_t calls = 0;  // collectives issued on this clique
  cudaEvent_t ev_join = nullptr;
  std::vector<cudaEvent_t> ev_fork;
  // fork/join points when a call is not timed (flxSetTiming 0 or capture):
  // a timing event record costs as much host time as a kernel launch
  cudaEvent_t ev_start_nt = nullptr, ev_pcie_nt = nullptr;
  // host-staged ring: buffers x members x chunk_cap bytes, pinned + device
  char* host_stage = nullptr;
  char* dev_stage = nullptr;
  uint32_t* sems = nullptr;  // [0..B) semFull, [B..2B) semEmpty
  bool sems_on_host = false;  // pinned+mapped host words instead of device words
  size_t stage_cap = 0;      // chunk capacity per member
  int stage_bufs = 0;        // buffers allocated
  int ring_depth = 0;        // buffers the pipeline cycles through (flxSetStaging)
  // rings replaced by a larger one: a CUDA graph captured earlier may still
  // copy through them, so they live until clique_destroy (grow-only staging)
  std::vector<char*> retired_host, retired_dev;
  uint64_t piece_seq = 0;    // monotone chunk counter -> counter semaphores
  std::array<size_t, FLX_NUM_PATHS> last_bytes{{0, 0, 0}};
  int destroyed = 0;
  AutoTuner* tuner = nullptr;  // in-library Stage 1 / Stage 2 (autotune.cpp)
  std::string gpu_name;
};

// Multi-rank worlds (world.cu): one process per GPU, or loopback emulation.
struct World;
flxResult_t world_create_loopback(int nranks, int device, World** out);
flxResult_t world_create_rank(int nranks, int rank, int device, const char* id_hex, World** out);
flxResult_t world_create_loopback_ipc(int nranks, int device, const char* id_hex, World** out);
flxResult_t world_host_remote_ranks(int nranks, int device, const char* id_hex, double seconds);
void world_attach(World* w, int local, Comm* c);
int world_release(World* w);
flxResult_t run_world(World* w, const std::vector<const void*>& send,
                      const std::vector<void*>& recv, const std::vector<cudaStream_t>& streams,
                      int coll, size_t count, int dtype, int op, const Granules& g,
                      size_t alignment, bool timing);
flxResult_t world_read_timing(World* w, int local, uint64_t seq, float ms[3]);
uint64_t world_calls(World* w, int local);
std::array<size_t, FLX_NUM_PATHS> world_last_bytes(World* w, int local);
void world_set_nctas(World* w, int n);
int world_nlocal(World* w);
bool world_aborted(World* w);
void world_abort(World* w);
flxResult_t world_finalize(World* w, int local);
AutoTuner* world_tuner(World* w);
const char* world_nvls_status(World* w, int* on);
// run one collective over the world with the autotuner deciding the split
flxResult_t run_world_tuned(World* w, const std::vector<const void*>& send,
                            const std::vector<void*>& recv,
                            const std::vector<cudaStream_t>& streams, int coll, size_t count,
                            int dtype, int op, const Comm& lead, bool pinned,
                            const Granules& fallback, int path_mask, size_t alignment);
flxResult_t world_debug_peer(World* w, int local, int peer, int host_region, int write,
                             void* buf, size_t bytes);
// elementwise max of n doubles over every rank (the balancer's agreement board)
flxResult_t world_agree(World* w, double* vals, int n);

constexpr uint64_t kCommMagic = 0x4b4e494c58454c46ull;  // "FLEXLINK"
struct Comm {
  // first member: validate_comm rejects anything that is not a live FlexLink
  // communicator (e.g. a real ncclComm_t handed to the NCCL-named entry points)
  uint64_t magic = kCommMagic;
  int rank = 0;
  int nranks = 1;
  int device = 0;
  Clique* clique = nullptr;  // virtual-rank (fused) mode
  World* world = nullptr;    // multi-rank mode
  int local = 0;             // index among the world's ranks in this process
  ShareTable shares[4];  // per flxCollOp_t
  int nvlink_ctas = 0;   // 0 = auto
  size_t chunk_bytes = 0;  // 0 = auto
  int buffers = 2;
  bool timing = true;    // record per-path CUDA events (flxSetTiming)
  // in-library balancer (flxSetAutoTune / flxSetTunerConfig / flxSetLinkProfile)
  bool autotune = true;
  size_t tune_min_bytes = 16 << 20;
  flxTunerConfig tune_s1{32, 0.05, 3, 100};
  flxBalancerConfig tune_s2{10, 0.10, 10, 10};
  bool have_profile = false;
  flxLinkProfile profile{};
  // flxCommInitRank communicators: the id they were made from and the number of
  // flxCommSplit calls so far (same on every rank: splits are collective)
  flxUniqueId uid{};
  uint64_t splits = 0;
};

}  // namespace flx
