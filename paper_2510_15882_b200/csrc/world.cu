// Multi-rank communicators: one process per GPU (flxCommInitRank), or every
// rank of such a world emulated on one GPU (flxCommInitLoopback).
//
// Data plane per call (per rank r, message split by partition()):
//   NVLink slice : rank_allreduce/rank_allgather kernel over peer-mapped
//                  scratch (rank_kernels.cuh)
//   PCIe slice   : host-hub staging through one shared host segment; copy
//                  engines on two side streams; per-edge tokens on the shared
//                  words, set with cuStreamWriteValue32 and awaited with
//                  cuStreamWaitValue32 (EQ) — constant values, so the same
//                  memops replay correctly from a CUDA graph:
//     AllReduce  1 take H_r; D2H send[sub c] -> H_r[c]; post prod[r][c]  (c != r)
//                2 accept prod[p][r]; H2D H_p[r] -> stage[p]; give hfree[p][r]
//                  fold stage[*] + own sub r -> recv sub r
//                3 take R_r; D2H recv sub r -> R_r; post rprod[r][c]
//                4 accept rprod[c][r]; H2D R_c -> recv sub c; give rfree[c][r]
//     AllGather  1 take H_r; D2H send -> H_r; post prod[r][c]
//                2 accept prod[c][r]; H2D H_c -> recv block c; give hfree[c][r]
//     ReduceScatter / AllToAll = steps 1-2 on the PCIe part of each block
//                (AllToAll lands straight in recv, no fold).
//   The slice moves in chunks (FLX_PCIE_CHUNK_KB per reader) through two
//   buffers b = k % 2 of H_r, R_r and the landing zone, every token indexed by
//   [buffer]; "take H_r[b]" waits for every reader's free token of the
//   previous use of that buffer, whichever protocol that was; R_r likewise.
//   Issue order is global and software-pipelined (steps 1-2 of chunk k for all
//   ranks, then steps 3-4 of chunk k-1) so every wait refers to a write issued
//   earlier: no deadlock even when streams share a hardware queue (loopback).
// Bootstrap (multi-process): a POSIX shm segment named by the unique id
// carries each rank's CUDA IPC handles (scratch + flags) and a second one is
// the PCIe staging area, cudaHostRegister'ed by every rank.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

#include "autotune.h"
#include "board.h"
#include "internal.h"
#include "nvls.h"
#include "nvls_kernels.cuh"
#include "rank_kernels.cuh"
#include "rank_launch.h"

namespace flx {

namespace {

// uint32 words at the head of the staging segment: [0, 4096) token words,
// [4096, 12288) the balancer's agreement board (world_agree_max)
constexpr int kSemWords = 12288;
constexpr int kBoardWord = 4096;
static_assert((size_t)(kSemWords - kBoardWord) * 4 >= 16 * kBoardSlots * kBoardSlotWords * 8,
              "the agreement board must fit its words of the staging segment head");
// token word layout: [kind][buffer][producer][reader] over kMaxRanks, see token_post
inline size_t tok(int kind, int r, int c, int b) {
  return ((size_t)(kind * 2 + b) * kMaxRanks + r) * kMaxRanks + c;
}
inline size_t sem_prod(int r, int c, int b) { return tok(0, r, c, b); }   // H_r[b] piece ready
inline size_t sem_hfree(int r, int c, int b) { return tok(1, r, c, b); }  // H_r[b] taken/free
inline size_t sem_rprod(int r, int c, int b) { return tok(2, r, c, b); }  // R_r[b] ready
inline size_t sem_rfree(int r, int c, int b) { return tok(3, r, c, b); }  // R_r[b] taken/free

size_t env_mib(const char* name, size_t dflt) {
  const char* v = getenv(name);
  return v ? (size_t)atoll(v) << 20 : dflt << 20;
}

// World layout and protocol settings every rank must share: each rank reads
// them from its own environment (FLX_SLOT_MB, FLX_PCIE_STAGE_MB,
// FLX_PCIE_CHUNK_KB, FLX_ONESHOT_KB, FLX_LL, FLX_NVLINK_CTAS, FLX_NVLS, FLX_SHARES) and a mismatch
// would shift scratch / staging offsets between ranks, so bootstrap compares them.
struct BootConfig {
  uint64_t nranks, slot, small_slot, hcap, pcie_chunk, oneshot_max, ll, nctas, sem_words, nvls,
      shares;
};

struct BootSlot {
  int ready;
  int device;
  int pid;
  char pad[4];
  cudaIpcMemHandle_t scratch;
  cudaIpcMemHandle_t flags;
  char bus_id[32];
  BootConfig config;
};

struct BootHeader {
  int arrived;
  int mapped;
  int leaving;  // destroy barrier: no rank frees what peers may still touch
  int nranks;
  int pad;
  BootSlot slot[kMaxRanks];
  NvlsBoot nvls;  // NVLS multicast rendezvous (nvls.cu)
};

}  // namespace

struct World {
  int nranks = 0;
  bool loopback = false;
  int nctas = 0;
  int max_nctas = kMaxCtas;  // loopback: every CTA of every rank co-resident
  size_t slot = 0;       // inbox slot bytes per source rank
  size_t small_slot = 0;  // one-shot inbox bytes per source rank and parity
  long long spin_limit = 0;  // peer-wait limit in SM clock cycles (FLX_TIMEOUT_S)
  // FLX_TIMEOUT_S: peer waits (kernel spins, the balancer's agreement board) and the
  // PCIe-leg watchdog.  The default follows PyTorch's NCCL process-group timeout
  // (10 min): ranks legitimately drift by seconds to minutes (a checkpoint save, an
  // eval on rank 0), and NCCL waits that out rather than failing the collective
  double timeout_s = 600.0;
  size_t oneshot_max = 0;  // AllReduce NVLink slices up to this size run one-shot (if they fit)
  bool ll = true;          // one-shot slices that fit kLLRegion / 2 per CTA use the LL format (FLX_LL)
  bool bulk = true;        // two-shot push / pull as TMA bulk copies (FLX_BULK=0: register copies)
  size_t hcap = 0;       // PCIe staging bytes per rank region
  size_t pcie_chunk = 0;  // PCIe pipeline chunk, bytes per reader (FLX_PCIE_CHUNK_KB)
  // (NVLink-path flag epochs live on the device: kStateWords in each flag block)
  // host staging segment: [sem words][H_0 .. H_{n-1}][R_0 .. R_{n-1}]
  char* host = nullptr;
  size_t host_bytes = 0;
  bool host_shm = false;
  uint32_t* abort_word = nullptr;  // pinned, mapped
  // per local rank i: [2i] = PCIe legs started, [2i+1] = PCIe legs finished,
  // written by the rank's h2d stream (same pinned block as abort_word)
  uint32_t* progress = nullptr;
  struct Local {
    Comm* comm = nullptr;
    int rank = 0;
    int device = 0;
    char* scratch = nullptr;
    uint32_t* flags = nullptr;
    char* dstage = nullptr;  // device landing zone for PCIe sub-chunks
    cudaStream_t d2h = nullptr, h2d = nullptr;
    cudaEvent_t fold_done[2] = {nullptr, nullptr}, ev_join = nullptr;
    cudaEvent_t ev_start_nt = nullptr, ev_pcie_nt = nullptr;  // untimed fork/join points
    cudaEvent_t ev_d2h_done = nullptr;  // joins the D2H stream's last token writes
    std::vector<cudaEvent_t> ev_fork;
    Clique::Timing timing[Clique::kTimingSlots];
    uint64_t calls = 0;
    std::array<size_t, FLX_NUM_PATHS> last_bytes{{0, 0, 0}};
    // PCIe-leg watchdog (flxCommGetAsyncError): PCIe legs issued (host count,
    // release-published); the h2d stream itself writes the leg's number into
    // World::progress when the leg starts and when it ends, so the watchdog
    // tells a leg that is running from one still queued behind user work
    uint32_t pcie_gen = 0;
    // the watchdog's own view (guarded by World::watch_mu): the running leg it
    // last saw and when it first saw it running
    uint32_t seen_leg = 0;
    std::chrono::steady_clock::time_point seen_started{};
    // scratch/flags are CUDA-IPC mappings of another process's allocation
    // (flxCommInitLoopbackIpc): closed, not freed
    bool remote_mem = false;
  };
  std::vector<Local> local;
  // peer views (as mapped in this process): scratch/flags of every rank
  char* peer_scratch[kMaxRanks] = {};
  uint32_t* peer_flags[kMaxRanks] = {};
  std::vector<void*> ipc_opened;
  struct BootHeader* boot = nullptr;  // kept mapped (name unlinked) for the destroy barrier
  int destroyed = 0;
  bool aborting = false;  // flxCommAbort: skip the destroy barrier
  bool shared_gpu = false;  // ranks share a GPU (bootstrap self-tests): no NVLink-path tuning
  uint64_t agree_seq = 0;   // decision points agreed so far (same on every rank)
  AutoTuner tuner;
  std::mutex watch_mu;  // world_aborted's watchdog state (callers may be threads)
  NvlsBuffer nvls;          // NVLink-SHARP multicast buffer (FLX_NVLS=1, multi-GPU only)
  void* ipc_debug = nullptr;  // flxCommInitLoopbackIpc: the exporter's segment

  // semaphore words as the GPU addresses them (registered host memory may map
  // to a different device address than its host pointer)
  char* host_dev = nullptr;
  uint32_t* sem(size_t word) { return reinterpret_cast<uint32_t*>(host_dev) + word; }
  char* hregion(int r) { return host + kSemWords * 4 + (size_t)r * hcap; }
  char* rregion(int r) { return host + kSemWords * 4 + (size_t)nranks * hcap + (size_t)r * hcap; }
};

namespace {

// One rank's peer-visible memory: scratch [n inbox slots][outbox][one-shot
// inboxes: 2 parities x n sources][LL packets: 2 parities x n sources x
// kLLSlot] (LL zeroed: epochs start at 1) and the flag block (zeroed).
flxResult_t alloc_rank_mem(const World* w, char** scratch, uint32_t** flags) {
  const size_t ll_off = w->slot * (w->nranks + 1) + 2 * w->nranks * w->small_slot;
  const size_t scratch_bytes = ll_off + 2 * w->nranks * kLLSlot;
  FLX_CUDA(cudaMalloc(reinterpret_cast<void**>(scratch), scratch_bytes));
  FLX_CUDA(cudaMemset(*scratch + ll_off, 0, 2 * w->nranks * kLLSlot));
  FLX_CUDA(cudaMalloc(reinterpret_cast<void**>(flags), (kFlagWords + kStateWords) * 4));
  FLX_CUDA(cudaMemset(*flags, 0, (kFlagWords + kStateWords) * 4));
  return flxSuccess;
}

flxResult_t local_init(World* w, World::Local& L) {
  FLX_CUDA(cudaSetDevice(L.device));
  FLX_CUDA(preload_all_kernels());  // no lazy load behind a parked PCIe leg / spinning kernel
  int khz = 0;
  FLX_CUDA(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, L.device));
  const char* to = getenv("FLX_TIMEOUT_S");
  const double secs = to ? atof(to) : 600.0;
  w->spin_limit = (long long)(std::max(0.01, secs) * khz * 1e3);
  w->timeout_s = std::max(0.01, secs);
  if (!L.remote_mem) FLX_TRY(alloc_rank_mem(w, &L.scratch, &L.flags));
  FLX_CUDA(cudaMalloc(reinterpret_cast<void**>(&L.dstage), w->hcap));
  FLX_CUDA(cudaStreamCreateWithFlags(&L.d2h, cudaStreamNonBlocking));
  FLX_CUDA(cudaStreamCreateWithFlags(&L.h2d, cudaStreamNonBlocking));
  for (auto& e : L.fold_done) FLX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  FLX_CUDA(cudaEventCreateWithFlags(&L.ev_join, cudaEventDisableTiming));
  FLX_CUDA(cudaEventCreateWithFlags(&L.ev_start_nt, cudaEventDisableTiming));
  FLX_CUDA(cudaEventCreateWithFlags(&L.ev_pcie_nt, cudaEventDisableTiming));
  FLX_CUDA(cudaEventCreateWithFlags(&L.ev_d2h_done, cudaEventDisableTiming));
  for (auto& t : L.timing) {
    FLX_CUDA(cudaEventCreate(&t.start));
    FLX_CUDA(cudaEventCreate(&t.nv));
    FLX_CUDA(cudaEventCreate(&t.pcie));
  }
  L.ev_fork.resize(w->loopback ? w->nranks : 1);
  for (auto& e : L.ev_fork) FLX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  FLX_CUDA(cudaDeviceSynchronize());
  return flxSuccess;
}

// Wait (at most `seconds`) until every stream of this world's ranks is idle.
// On abort, a peer that died mid PCIe slice leaves this rank's copy streams
// parked in cuStreamWaitValue32 on the shared token words, which have no
// timeout: keep forcing every token to the value its waiters expect — ready
// tokens (prod, rprod) are awaited == 1, free tokens (hfree, rfree) == 0 — so
// each pending wait, and the ones queued behind it, fall through.  The NVLink
// kernels already gave up on the abort word.
bool drain_streams(World* w, double seconds, bool release_tokens) {
  const auto t0 = std::chrono::steady_clock::now();
  while (true) {
    bool idle = true;
    for (auto& L : w->local) {
      cudaSetDevice(L.device);
      if (L.d2h && cudaStreamQuery(L.d2h) == cudaErrorNotReady) idle = false;
      if (L.h2d && cudaStreamQuery(L.h2d) == cudaErrorNotReady) idle = false;
    }
    if (idle) return true;
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > seconds)
      return false;
    if (release_tokens && w->host) {
      auto* words = reinterpret_cast<volatile uint32_t*>(w->host);
      for (int b = 0; b < 2; ++b)
        for (int r = 0; r < w->nranks; ++r)
          for (int c = 0; c < w->nranks; ++c) {
            words[sem_prod(r, c, b)] = 1;
            words[sem_rprod(r, c, b)] = 1;
            words[sem_hfree(r, c, b)] = 0;
            words[sem_rfree(r, c, b)] = 0;
          }
    }
    std::this_thread::sleep_for(std::chrono::microseconds(100));
  }
}

void world_free(World* w) {
  // Every kernel / copy that may touch peer memory must be done before the
  // destroy barrier.  An aborted world releases its parked PCIe waits; if its
  // streams still do not drain, its memory is leaked rather than freed under
  // a hung stream (cudaFree would block on it forever).
  bool drained = true;
  const bool aborted = w->aborting || (w->abort_word && *(volatile uint32_t*)w->abort_word);
  if (aborted) drained = drain_streams(w, std::min(30.0, std::max(5.0, w->timeout_s)), true);
  if (drained)
    for (auto& L : w->local) {
      cudaSetDevice(L.device);
      cudaDeviceSynchronize();
    }
  if (w->boot) {
    // destroy barrier: a peer may still be pushing into my scratch or reading
    // my outbox / host region until it, too, has drained its device
    __atomic_fetch_add(&w->boot->leaving, 1, __ATOMIC_ACQ_REL);
    const auto t0 = std::chrono::steady_clock::now();
    const double limit = w->aborting ? 0.0 : 60.0;  // abort: do not wait for peers
    while (__atomic_load_n(&w->boot->leaving, __ATOMIC_ACQUIRE) < w->nranks &&
           std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < limit)
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    munmap(w->boot, sizeof(BootHeader));
    w->boot = nullptr;
  }
  if (!drained) {
    fprintf(stderr, "[flexlink] aborted communicator: side streams did not drain; leaking its "
                    "device and staging memory\n");
    delete w;
    return;
  }
  for (void* p : w->ipc_opened) cudaIpcCloseMemHandle(p);
  nvls_free(&w->nvls);
  for (auto& L : w->local) {
    if (L.remote_mem) {
      if (L.scratch) cudaIpcCloseMemHandle(L.scratch);
      if (L.flags) cudaIpcCloseMemHandle(L.flags);
    } else {
      if (L.scratch) cudaFree(L.scratch);
      if (L.flags) cudaFree(L.flags);
    }
    if (L.dstage) cudaFree(L.dstage);
    if (L.d2h) cudaStreamDestroy(L.d2h);
    if (L.h2d) cudaStreamDestroy(L.h2d);
    for (auto e : L.fold_done)
      if (e) cudaEventDestroy(e);
    if (L.ev_join) cudaEventDestroy(L.ev_join);
    if (L.ev_start_nt) cudaEventDestroy(L.ev_start_nt);
    if (L.ev_pcie_nt) cudaEventDestroy(L.ev_pcie_nt);
    if (L.ev_d2h_done) cudaEventDestroy(L.ev_d2h_done);
    for (auto e : L.ev_fork) cudaEventDestroy(e);
    for (auto& t : L.timing) {
      cudaEventDestroy(t.start);
      cudaEventDestroy(t.nv);
      cudaEventDestroy(t.pcie);
    }
  }
  if (w->host) {
    cudaHostUnregister(w->host);
    if (w->host_shm)
      munmap(w->host, w->host_bytes);
    else
      free(w->host);
  }
  if (w->abort_word) cudaFreeHost(w->abort_word);
  if (w->ipc_debug) {  // tell the exporting process its memory is no longer used
    int* done = &static_cast<int*>(w->ipc_debug)[1];
    __atomic_store_n(done, 1, __ATOMIC_RELEASE);
    munmap(w->ipc_debug, sizeof(int) * 4 + sizeof(cudaIpcMemHandle_t) * 2 * kMaxRanks);
  }
  delete w;
}

flxResult_t alloc_host_staging(World* w, const char* shm_name) {
  w->host_bytes = (size_t)kSemWords * 4 + 2 * (size_t)w->nranks * w->hcap;
  if (shm_name) {
    int fd = shm_open(shm_name, O_CREAT | O_RDWR, 0600);
    if (fd < 0) return fail(flxSystemError, "shm_open(%s) failed", shm_name);
    if (ftruncate(fd, (off_t)w->host_bytes) != 0) {
      close(fd);
      return fail(flxSystemError, "ftruncate of %zu-byte staging segment failed", w->host_bytes);
    }
    void* p = mmap(nullptr, w->host_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) return fail(flxSystemError, "mmap of staging segment failed");
    w->host = static_cast<char*>(p);
    w->host_shm = true;
  } else {
    void* p = nullptr;
    if (posix_memalign(&p, 4096, w->host_bytes) != 0)
      return fail(flxSystemError, "host staging allocation failed");
    memset(p, 0, w->host_bytes);
    w->host = static_cast<char*>(p);
  }
  FLX_CUDA(cudaHostRegister(w->host, w->host_bytes,
                            cudaHostRegisterMapped | cudaHostRegisterPortable));
  void* dev = nullptr;
  FLX_CUDA(cudaHostGetDevicePointer(&dev, w->host, 0));
  w->host_dev = static_cast<char*>(dev);
  FLX_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&w->abort_word), 64 + 8 * kMaxRanks,
                         cudaHostAllocMapped | cudaHostAllocPortable));
  *w->abort_word = 0;
  w->progress = w->abort_word + 16;
  memset(w->progress, 0, 8 * kMaxRanks);
  return flxSuccess;
}

void world_config(World* w, int nranks) {
  w->nranks = nranks;
  // 64 MiB: kMaxCtas regions of 1 MiB, so 32 CTAs move 256 MiB per AllReduce round
  w->slot = std::max<size_t>(env_mib("FLX_SLOT_MB", 64), 1 << 20);
  w->hcap = env_mib("FLX_PCIE_STAGE_MB", 64);
  // per-reader bytes of one PCIe pipeline chunk (the paper's 4 MiB staging buffer)
  const char* ck = getenv("FLX_PCIE_CHUNK_KB");
  w->pcie_chunk = std::max<size_t>(4096, (size_t)(ck ? atoll(ck) : 4096) << 10);
  // 64 CTAs of 512 threads per GPU: the rank kernels fit 64 registers (2 CTAs
  // per SM), 4 x 16 B loads in flight per thread in the copy phases — the same
  // bytes in flight as 32 CTAs x 8 loads, on 32 SMs, leaving the rest of the
  // GPU to compute (loopback, all ranks on one GPU: 8-rank 256 MiB AllReduce
  // 1.78 -> 1.65 ms; 2 ranks 0.63 -> 0.40 ms; profiles/r2/loopback_occupancy.jsonl)
  w->nctas = kMaxCtas;
  if (const char* v = getenv("FLX_NVLINK_CTAS")) w->nctas = std::max(1, std::min(kMaxCtas, atoi(v)));
  // one-shot AllReduce up to this many bytes per rank (FLX_ONESHOT_KB=0: off);
  // its inbox holds kMaxCtas regions, so 2x the threshold covers nctas >= 32
  const char* os = getenv("FLX_ONESHOT_KB");
  w->oneshot_max = (size_t)(os ? atoll(os) : 256) << 10;
  w->small_slot = std::max<size_t>(2 * w->oneshot_max, 16 * kMaxCtas);
  const char* ll = getenv("FLX_LL");
  w->ll = !(ll && atoi(ll) == 0);
  // a per-rank choice of copy mechanism: the protocol and layout are the same
  const char* bulk = getenv("FLX_BULK");
  w->bulk = !(bulk && atoi(bulk) == 0);
}

template <typename F>
bool spin_until(F pred, double seconds) {
  const auto t0 = std::chrono::steady_clock::now();
  while (!pred()) {
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > seconds)
      return false;
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  return true;
}

// ------------------------------------------------------------- launches
// SCATTER selects ReduceScatter (push + fold) instead of AllReduce (push +
// fold + pull); the per-dtype launchers live in rank_launch_*.cu.
template <bool SCATTER>
cudaError_t launch_rank_reduce(int dtype, int op, bool loop, const void* a, int nctas, int n,
                               cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  switch (dtype) {
    case flxInt8: case flxUint8: return rank_reduce_i8(dtype, op, SCATTER, loop, a, nctas, n, s);
    case flxInt32: case flxUint32: return rank_reduce_i32(dtype, op, SCATTER, loop, a, nctas, n, s);
    case flxInt64: case flxUint64: return rank_reduce_i64(dtype, op, SCATTER, loop, a, nctas, n, s);
    case flxFloat16: case flxBfloat16:
      return rank_reduce_f16(dtype, op, SCATTER, loop, a, nctas, n, s);
    case flxFloat32: return rank_reduce_f32(dtype, op, SCATTER, loop, a, nctas, n, s);
    case flxFloat64: return rank_reduce_f64(dtype, op, SCATTER, loop, a, nctas, n, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_rank_allgather(bool loop, const void* args, int nctas, int nranks,
                                  cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  static std::atomic<uint64_t> opted{0};  // the bulk-copy ring (RankArgs::bulk)
  opt_in_dyn_smem(opted, {(const void*)loopback_allgather_kernel, (const void*)rank_allgather_kernel},
                  (int)kRankDynSmem);
  const size_t dyn = (loop ? static_cast<const LoopbackArgs*>(args)->r[0].bulk
                           : static_cast<const RankArgs*>(args)->bulk) ? kRankDynSmem : 0;
  if (loop) {
    void* params[] = {const_cast<void*>(args)};
    return cudaLaunchCooperativeKernel((const void*)loopback_allgather_kernel, dim3(nctas, nranks),
                                       dim3(512), params, dyn, s);
  }
  rank_allgather_kernel<<<nctas, 512, dyn, s>>>(*static_cast<const RankArgs*>(args));
  return cudaGetLastError();
}

cudaError_t launch_rank_alltoall(bool loop, const void* args, int nctas, int nranks,
                                 cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  static std::atomic<uint64_t> opted{0};  // the bulk-copy ring (RankArgs::bulk)
  opt_in_dyn_smem(opted, {(const void*)loopback_alltoall_kernel, (const void*)rank_alltoall_kernel},
                  (int)kRankDynSmem);
  const size_t dyn = (loop ? static_cast<const LoopbackArgs*>(args)->r[0].bulk
                           : static_cast<const RankArgs*>(args)->bulk) ? kRankDynSmem : 0;
  if (loop) {
    void* params[] = {const_cast<void*>(args)};
    return cudaLaunchCooperativeKernel((const void*)loopback_alltoall_kernel, dim3(nctas, nranks),
                                       dim3(512), params, dyn, s);
  }
  rank_alltoall_kernel<<<nctas, 512, dyn, s>>>(*static_cast<const RankArgs*>(args));
  return cudaGetLastError();
}

}  // namespace

// Token handshake on the shared host words (all values are constants, so the
// same stream memory operations are correct eagerly and replayed from a CUDA
// graph):  ready tokens prod/rprod[r][c] = 1 posted by producer r, consumed
// (reset to 0) by reader c; free tokens hfree/rfree[r][c] = 0 while reader c
// is done with region H_r / R_r, set to 1 by producer r when it takes the
// region, returned (0) by the reader after its H2D.  Every edge strictly
// alternates take -> post -> accept -> give, each write ordered after the
// wait that licenses it on the same stream.
static flxResult_t token_post(cudaStream_t s, uint32_t* w) { return sem_write(s, w, 1); }
static flxResult_t token_give(cudaStream_t s, uint32_t* w) { return sem_write(s, w, 0); }
static flxResult_t token_accept(cudaStream_t s, uint32_t* w) {
  FLX_TRY(sem_wait_eq(s, w, 1));
  return sem_write(s, w, 0);
}
// Rank r takes H_r (or R_r): every reader returned its free token.
static flxResult_t take_region(World* w, cudaStream_t s, int r, bool result, int b) {
  for (int p = 0; p < w->nranks; ++p) {
    if (p == r) continue;
    uint32_t* word = w->sem(result ? sem_rfree(r, p, b) : sem_hfree(r, p, b));
    FLX_TRY(sem_wait_eq(s, word, 0));
    FLX_TRY(sem_write(s, word, 1));
  }
  return flxSuccess;
}

// One collective over every local rank of a world; calls[i] is local rank i.
flxResult_t run_world(World* w, const std::vector<const void*>& send,
                      const std::vector<void*>& recv, const std::vector<cudaStream_t>& streams,
                      int coll, size_t count, int dtype, int op, const Granules& g,
                      size_t alignment, bool timing) {
  const int n = w->nranks;
  const int nl = (int)w->local.size();
  const size_t esz = dtype_size(dtype);
  const size_t bytes = count * esz;
  auto split = partition(bytes, g, alignment);
  if (split[flxPathRdma] > 0) return fail(flxInvalidUsage, "rdma path is not available");
  const size_t nv = split[flxPathNvlink], pc = split[flxPathPcie];
  const auto offs = path_offsets(split);  // PCIe slice first, NVLink last (internal.h)
  const size_t opc = offs[flxPathPcie], onv = offs[flxPathNvlink];
  const bool gather = coll == flxCollAllGather;
  const bool scatter = coll == flxCollReduceScatter;
  const bool a2a = coll == flxCollAllToAll;
  if (*w->abort_word) return fail(flxInternalError, "communicator aborted by an earlier timeout");
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  FLX_CUDA(cudaStreamIsCapturing(streams[0], &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  // The NVLink kernels keep their epochs on the device and the PCIe path's
  // token handshake uses constant values: both replay correctly from a graph.
  if (pc > 0 && !memops().ok) return fail(flxInvalidUsage, "pcie path needs stream memory ops");
  // Ranks of this world share a GPU (FLX_ALLOW_SHARED_GPU self-tests): an
  // NVLink-path kernel would spin on another process's kernel on the same
  // GPU, which is not guaranteed to be co-scheduled (context-switch timeouts).
  // Only host-staged PCIe bytes may move; FLX_SHARED_GPU_KERNELS=1 lets the
  // peer-timeout test launch one kernel whose peer never comes.
  if (w->shared_gpu && !w->loopback && nv > 0 && n > 1 && !getenv("FLX_SHARED_GPU_KERNELS"))
    return fail(flxInvalidUsage,
                "ranks of this world share one GPU: NVLink-path kernels would wait on another "
                "process's kernel; pin every byte to PCIe (FLX_SHARES=0,1000 or flxSetShares) "
                "with a message size that is a multiple of the alignment (%zu B)", alignment);

  // fork: in loopback every rank's stream joins local rank 0's stream
  cudaStream_t s0 = streams[0];
  FLX_CUDA(cudaSetDevice(w->local[0].device));
  for (int i = 1; i < nl; ++i) {
    if (streams[i] == s0) continue;
    FLX_CUDA(cudaEventRecord(w->local[0].ev_fork[i], streams[i]));
    FLX_CUDA(cudaStreamWaitEvent(s0, w->local[0].ev_fork[i], 0));
  }
  std::vector<Clique::Timing*> tm(nl);
  for (int i = 0; i < nl; ++i) {
    World::Local& L = w->local[i];
    tm[i] = &L.timing[L.calls % Clique::kTimingSlots];
  }
  // every local rank shares s0: one start/nv event pair (local rank 0's) times
  // the NVLink slice for all of them; the PCIe legs keep per-rank events
  const bool timed = timing && !capturing;
  const cudaEvent_t ev_start = timed ? tm[0]->start : w->local[0].ev_start_nt;
  auto ev_pcie = [&](int i) { return timed ? tm[i]->pcie : w->local[i].ev_pcie_nt; };
  if (timed || pc > 0) FLX_CUDA(cudaEventRecord(ev_start, s0));

  // ---------------- PCIe slice (issued first so the copies overlap the kernel)
  // Chunked and double-buffered (buffer b = chunk k % 2 of H_r, R_r and each
  // rank's device landing zone), so chunk k+1's D2H runs while chunk k's H2D
  // and fold do: both PCIe directions stay busy (staging.py's two-hop
  // pipeline, PipelineSpec with buffers=2).  Issue order is software-pipelined
  // and global — step 1 and 2 of chunk k for every rank, then AllReduce steps 3
  // and 4 of chunk k-1 — so every wait refers to a write issued earlier.
  if (pc > 0) {
    for (int i = 0; i < nl; ++i) {
      World::Local& L = w->local[i];
      FLX_CUDA(cudaStreamWaitEvent(L.d2h, ev_start, 0));
      FLX_CUDA(cudaStreamWaitEvent(L.h2d, ev_start, 0));
      if (!capturing)  // the leg has started (user work before the call is done)
        FLX_TRY(sem_write(L.h2d, &w->progress[2 * i], L.pcie_gen + 1));
    }
    const bool ar = !gather && !scatter && !a2a;
    const size_t q = ar ? pc / n : pc;  // bytes per reader (AR sub-chunk / RS, A2A block part)
    // bytes per reader of one chunk, a multiple of 4096 such that 2 buffers fit
    // a rank's host region and landing zone.  AllGather's buffer holds one piece
    // for all readers (not one per reader) and its H2D side carries N-1 times
    // the D2H side, so it takes N-times larger chunks: fewer hand-offs, and
    // overlap would buy it at most 1/N (profiles/r1/pcie_world_256.jsonl).
    const size_t fit = ((w->hcap / (gather ? 2 : 2 * (size_t)n)) / 4096) * 4096;
    const size_t want = gather ? w->pcie_chunk * n : w->pcie_chunk;
    const size_t cq = std::max<size_t>(4096, std::min(want, fit));
    const size_t chunks = (q + cq - 1) / cq;
    const size_t slot_h = gather ? cq : cq * n;  // one buffer of H_r
    auto piece = [&](size_t k) { return std::min(cq, q - k * cq); };

    auto step12 = [&](size_t k) -> flxResult_t {
      const int b = (int)(k & 1);
      const size_t len = piece(k), at = k * cq;
      for (int i = 0; i < nl; ++i) {  // step 1: take H_r[b], D2H, post per reader
        World::Local& L = w->local[i];
        const int r = L.rank;
        FLX_TRY(take_region(w, L.d2h, r, false, b));
        const char* src = static_cast<const char*>(send[i]);
        char* h = w->hregion(r) + b * slot_h;
        if (gather) {
          FLX_CUDA(cudaMemcpyAsync(h, src + opc + at, len, cudaMemcpyDeviceToHost, L.d2h));
        } else {
          for (int s = 1; s < n; ++s) {
            const int c = (r + s) % n;
            const char* from = ar ? src + opc + c * q + at : src + (size_t)c * bytes + opc + at;
            FLX_CUDA(cudaMemcpyAsync(h + c * cq, from, len, cudaMemcpyDeviceToHost, L.d2h));
          }
        }
        for (int s = 1; s < n; ++s)
          FLX_TRY(token_post(L.d2h, w->sem(sem_prod(r, (r + s) % n, b))));
      }
      for (int i = 0; i < nl; ++i) {  // step 2: accept, H2D, give; fold (AR / RS)
        World::Local& L = w->local[i];
        const int r = L.rank;
        char* dst = static_cast<char*>(recv[i]);
        const char* src = static_cast<const char*>(send[i]);
        char* land = L.dstage + b * cq * n;
        for (int s = 1; s < n; ++s) {
          const int p = (r - s + n) % n;
          FLX_TRY(token_accept(L.h2d, w->sem(sem_prod(p, r, b))));
          const char* from = w->hregion(p) + b * slot_h + (gather ? 0 : r * cq);
          char* to = (gather || a2a) ? dst + (size_t)p * bytes + opc + at : land + p * cq;
          FLX_CUDA(cudaMemcpyAsync(to, from, len, cudaMemcpyHostToDevice, L.h2d));
          FLX_TRY(token_give(L.h2d, w->sem(sem_hfree(p, r, b))));
        }
        if (ar || scatter) {  // fold every source's piece in rank order
          FoldArgs a{};
          for (int p = 0; p < n; ++p)
            a.src[p] = p != r    ? land + p * cq
                       : scatter ? src + (size_t)r * bytes + opc + at
                                 : src + opc + r * q + at;
          a.dst[0] = scatter ? dst + opc + at : dst + opc + r * q + at;
          a.n = n;
          a.ndst = 1;
          a.bytes = len;
          FLX_CUDA(launch_fold(dtype, op, a, 16, L.h2d));
          if (ar) FLX_CUDA(cudaEventRecord(L.fold_done[b], L.h2d));
        }
      }
      return flxSuccess;
    };
    auto step34 = [&](size_t k) -> flxResult_t {  // AllReduce: share the reduced piece
      const int b = (int)(k & 1);
      const size_t len = piece(k), at = k * cq;
      for (int i = 0; i < nl; ++i) {  // step 3: take R_r[b], D2H my reduced piece, post
        World::Local& L = w->local[i];
        const int r = L.rank;
        FLX_CUDA(cudaStreamWaitEvent(L.d2h, L.fold_done[b], 0));
        FLX_TRY(take_region(w, L.d2h, r, true, b));
        FLX_CUDA(cudaMemcpyAsync(w->rregion(r) + b * cq,
                                 static_cast<char*>(recv[i]) + opc + r * q + at, len,
                                 cudaMemcpyDeviceToHost, L.d2h));
        for (int s = 1; s < n; ++s)
          FLX_TRY(token_post(L.d2h, w->sem(sem_rprod(r, (r + s) % n, b))));
      }
      for (int i = 0; i < nl; ++i) {  // step 4: accept, H2D every other piece, give
        World::Local& L = w->local[i];
        const int r = L.rank;
        for (int s = 1; s < n; ++s) {
          const int c = (r + s) % n;
          FLX_TRY(token_accept(L.h2d, w->sem(sem_rprod(c, r, b))));
          FLX_CUDA(cudaMemcpyAsync(static_cast<char*>(recv[i]) + opc + c * q + at,
                                   w->rregion(c) + b * cq, len, cudaMemcpyHostToDevice, L.h2d));
          FLX_TRY(token_give(L.h2d, w->sem(sem_rfree(c, r, b))));
        }
      }
      return flxSuccess;
    };

    for (int i = 0; i < nl; ++i) {  // own pieces that never leave the GPU
      World::Local& L = w->local[i];
      const int r = L.rank;
      char* dst = static_cast<char*>(recv[i]);
      const char* src = static_cast<const char*>(send[i]);
      if (gather) {
        char* own = dst + (size_t)r * bytes + opc;
        if (own != src + opc)
          FLX_CUDA(cudaMemcpyAsync(own, src + opc, pc, cudaMemcpyDeviceToDevice, L.h2d));
      } else if (a2a) {
        const size_t own = (size_t)r * bytes + opc;
        FLX_CUDA(cudaMemcpyAsync(dst + own, src + own, pc, cudaMemcpyDeviceToDevice, L.h2d));
      }
    }
    for (size_t k = 0; k <= chunks; ++k) {
      if (k < chunks) FLX_TRY(step12(k));
      if (ar && k >= 1) FLX_TRY(step34(k - 1));
    }
    for (int i = 0; i < nl; ++i) {
      FLX_CUDA(cudaEventRecord(ev_pcie(i), w->local[i].h2d));
      if (!capturing) {  // the leg has finished; publish it as issued
        World::Local& L = w->local[i];
        FLX_TRY(sem_write(L.h2d, &w->progress[2 * i + 1], L.pcie_gen + 1));
        __atomic_store_n(&L.pcie_gen, L.pcie_gen + 1, __ATOMIC_RELEASE);
      }
    }
  }

  // ---------------- NVLink slice
  if (nv > 0) {
    LoopbackArgs la;
    memset(&la, 0, sizeof(la));
    for (int i = 0; i < nl; ++i) {
      RankArgs& a = la.r[w->loopback ? w->local[i].rank : 0];
      a.send = static_cast<const char*>(send[i]) + onv;
      a.recv = static_cast<char*>(recv[i]) + onv;
      for (int p = 0; p < n; ++p) {
        a.scratch[p] = w->loopback ? w->local[p].scratch : w->peer_scratch[p];
        a.flags[p] = w->loopback ? w->local[p].flags : w->peer_flags[p];
      }
      a.rank = w->local[i].rank;
      a.nranks = n;
      a.bytes = nv;
      a.rank_stride = bytes;
      a.slot = w->slot;
      a.small_slot = w->small_slot;
      // one-shot when the slice fits this grid's share of the one-shot inbox
      // (every CTA part <= its region); AllReduce also below FLX_ONESHOT_KB
      // (above it the two-shot's 2(N-1)/N traffic wins), the other protocols
      // move the same bytes either way and save a signal hop
      // (or, in the LL format, when every CTA part fits half an LL region).
      // Depends only on rank-agreed values (bytes, grid), never on addresses.
      const size_t part = (((nv + w->nctas - 1) / w->nctas) + 15) & ~(size_t)15;
      const bool fits_ll = w->ll && 2 * part <= kLLRegion;
      const bool fits_flagged =
          nv <= ((w->small_slot / kMaxCtas) & ~(size_t)15) * (size_t)w->nctas;
      a.oneshot = w->oneshot_max > 0 && n > 1 && (fits_ll || fits_flagged) &&
                  (gather || scatter || a2a || nv <= w->oneshot_max);
      a.ll = a.oneshot && fits_ll;
      a.bulk = w->bulk;
      a.abort_word = w->abort_word;
      a.spin_limit = w->spin_limit;
    }
    const void* args = w->loopback ? static_cast<const void*>(&la) : &la.r[0];
    // NVLS AllReduce (nvls_kernels.cuh): the switch reduces; for sums of
    // fp32/bf16/fp16 above the one-shot range whose slice splits into 16 B
    // vectors per rank chunk, in rounds of the multicast buffer's capacity
    const bool nvls = w->nvls.on && !gather && !scatter && !a2a && op == kSum &&
                      nvls_dtype_ok(dtype) && !la.r[0].oneshot && nv % (16 * (size_t)n) == 0;
    // NVLS AllGather: one multicast store per slice, in rounds of capacity / N
    const bool nvls_ag = w->nvls.on && gather && !la.r[0].oneshot && nv % 16 == 0 &&
                         bytes % 16 == 0 && w->nvls.capacity / n >= 16;
    if (nvls_ag) {
      const size_t step = (w->nvls.capacity / n) & ~(size_t)15;
      for (size_t at = 0; at < nv; at += step) {
        NvlsArgs na{la.r[0].send + at, la.r[0].recv + at, reinterpret_cast<char*>(w->nvls.uc),
                    reinterpret_cast<char*>(w->nvls.mcva), w->nvls.state, w->local[0].rank, n,
                    std::min(step, nv - at), w->abort_word, w->spin_limit};
        cudaError_t e = launch_nvls_allgather(&na, bytes, std::min(w->nctas, kNvlsCtas), s0);
        if (e != cudaSuccess)
          return fail(flxUnhandledCudaError, "nvls kernel launch: %s", cudaGetErrorString(e));
      }
    }
    if (nvls) {
      const size_t step = w->nvls.capacity / (16 * (size_t)n) * (16 * (size_t)n);
      for (size_t at = 0; at < nv; at += step) {
        NvlsArgs na{la.r[0].send + at, la.r[0].recv + at, reinterpret_cast<char*>(w->nvls.uc),
                    reinterpret_cast<char*>(w->nvls.mcva), w->nvls.state, w->local[0].rank, n,
                    std::min(step, nv - at), w->abort_word, w->spin_limit};
        cudaError_t e = launch_nvls_allreduce(dtype, &na, std::min(w->nctas, kNvlsCtas), s0);
        if (e != cudaSuccess)
          return fail(flxUnhandledCudaError, "nvls kernel launch: %s", cudaGetErrorString(e));
      }
    }
    cudaError_t err =
        nvls || nvls_ag ? cudaSuccess
        : a2a     ? launch_rank_alltoall(w->loopback, args, w->nctas, n, s0)
        : gather  ? launch_rank_allgather(w->loopback, args, w->nctas, n, s0)
        : scatter ? launch_rank_reduce<true>(dtype, op, w->loopback, args, w->nctas, n, s0)
                  : launch_rank_reduce<false>(dtype, op, w->loopback, args, w->nctas, n, s0);
    if (err != cudaSuccess)
      return fail(flxUnhandledCudaError, "rank kernel launch: %s", cudaGetErrorString(err));
  }
  if (timed) FLX_CUDA(cudaEventRecord(tm[0]->nv, s0));
  if (pc > 0)
    for (int i = 0; i < nl; ++i) {
      FLX_CUDA(cudaStreamWaitEvent(s0, ev_pcie(i), 0));
      // the D2H stream ends with token posts: join it too (a CUDA-graph
      // capture must end with every forked stream joined)
      FLX_CUDA(cudaEventRecord(w->local[i].ev_d2h_done, w->local[i].d2h));
      FLX_CUDA(cudaStreamWaitEvent(s0, w->local[i].ev_d2h_done, 0));
    }
  bool joined = false;
  for (int i = 1; i < nl; ++i) {
    if (streams[i] == s0) continue;
    if (!joined) {
      FLX_CUDA(cudaEventRecord(w->local[0].ev_join, s0));
      joined = true;
    }
    FLX_CUDA(cudaStreamWaitEvent(streams[i], w->local[0].ev_join, 0));
  }
  for (int i = 0; i < nl; ++i) {
    World::Local& L = w->local[i];
    // events recorded inside a capture are graph edges, not timestamps
    tm[i]->used[flxPathNvlink] = nv > 0 && timed;
    tm[i]->used[flxPathPcie] = pc > 0 && timed;
    tm[i]->used[flxPathRdma] = false;
    L.last_bytes = split;
    L.calls++;
  }
  return flxSuccess;
}

flxResult_t world_read_timing(World* w, int local, uint64_t seq, float ms[3]) {
  World::Local& L = w->local[local];
  const Clique::Timing& t = L.timing[seq % Clique::kTimingSlots];
  // start/nv events are local rank 0's (shared by every local rank of a call)
  const Clique::Timing& t0 = w->local[0].timing[seq % Clique::kTimingSlots];
  FLX_CUDA(cudaSetDevice(L.device));
  ms[0] = ms[1] = ms[2] = 0.f;
  FLX_CUDA(cudaEventSynchronize(t0.nv));
  if (*w->abort_word) return fail(flxInternalError, "a peer wait timed out (rank died or hung?)");
  if (t.used[flxPathNvlink]) FLX_CUDA(cudaEventElapsedTime(&ms[0], t0.start, t0.nv));
  if (t.used[flxPathPcie]) {
    FLX_CUDA(cudaEventSynchronize(t.pcie));
    FLX_CUDA(cudaEventElapsedTime(&ms[1], t0.start, t.pcie));
  }
  return flxSuccess;
}

uint64_t world_calls(World* w, int local) { return w->local[local].calls; }
std::array<size_t, FLX_NUM_PATHS> world_last_bytes(World* w, int local) {
  return w->local[local].last_bytes;
}
int world_nranks(World* w) { return w->nranks; }
int world_nlocal(World* w) { return (int)w->local.size(); }
const char* world_nvls_status(World* w, int* on) {
  *on = w->nvls.on ? 1 : 0;
  return w->nvls.why;
}

bool world_aborted(World* w) {
  if (*(volatile uint32_t*)w->abort_word != 0) return true;
  // PCIe-leg watchdog: copy-engine waits on a dead peer's tokens never time
  // out by themselves.  A PCIe leg that has STARTED on the GPU (its h2d stream
  // got past the caller's earlier work) and is still unfinished FLX_TIMEOUT_S
  // after this watchdog first saw it running is reported, and aborts the
  // world like a timed-out NVLink wait.  Time queued behind the caller's own
  // kernels never counts; legs run in issue order on the h2d stream, so
  // started - finished is 0 (idle or queued) or 1 (leg `started` running).
  std::lock_guard<std::mutex> lock(w->watch_mu);
  const auto now = std::chrono::steady_clock::now();
  for (size_t i = 0; i < w->local.size(); ++i) {
    World::Local& L = w->local[i];
    const uint32_t issued = __atomic_load_n(&L.pcie_gen, __ATOMIC_ACQUIRE);
    const uint32_t finished = __atomic_load_n(&w->progress[2 * i + 1], __ATOMIC_ACQUIRE);
    const uint32_t started = __atomic_load_n(&w->progress[2 * i], __ATOMIC_ACQUIRE);
    if (finished == issued || started == finished) continue;  // idle, or next leg queued
    if (L.seen_leg != started) {  // first sight of this leg running
      L.seen_leg = started;
      L.seen_started = now;
      continue;
    }
    if (std::chrono::duration<double>(now - L.seen_started).count() > w->timeout_s) {
      *(volatile uint32_t*)w->abort_word = 1;
      return true;
    }
  }
  return false;
}
void world_set_nctas(World* w, int n) {
  if (n <= 0) {  // automatic: as at creation
    n = kMaxCtas;
    if (const char* v = getenv("FLX_NVLINK_CTAS")) n = std::max(1, std::min(kMaxCtas, atoi(v)));
    n = std::min(n, w->max_nctas);
    while (n & (n - 1)) n &= n - 1;
  }
  w->nctas = std::max(1, std::min(w->max_nctas, n));
}

AutoTuner* world_tuner(World* w) { return &w->tuner; }

// Elementwise max over every rank of n doubles, through the shared host
// segment's board: rank r publishes into its slot (agree_seq % kBoardSlots)
// with a release-ordered stamp, then waits for every rank's stamp of the same
// decision point.  Ranks reach decision points in the same order and none can
// pass point k+1 before every rank published point k+1, i.e. after it finished
// reading point k — so a slot is never overwritten while a peer still reads it.
static flxResult_t world_agree_max(World* w, double* vals, int n) {
  if (w->loopback || w->nranks == 1 || w->local.size() != 1) return flxSuccess;
  Board b;
  b.base = w->host + (size_t)kBoardWord * 4;
  b.nranks = w->nranks;
  b.me = w->local[0].rank;
  b.seq = &w->agree_seq;
  b.abort_word = w->abort_word;
  b.timeout_s = w->timeout_s;
  int bad = -1;
  switch (board_agree_max(b, vals, n, &bad)) {
    case 1:
      return fail(flxInternalError, "balancer agreement: rank %d never reached decision %llu",
                  bad, (unsigned long long)w->agree_seq - 1);
    case 2:
      return fail(flxInternalError, "balancer agreement: rank %d is at a different decision",
                  bad);
  }
  return flxSuccess;
}

namespace {
struct WorldPort : TimingPort {
  World* w;
  explicit WorldPort(World* w_) : w(w_) {}
  flxResult_t read(uint64_t seq, float ms[FLX_NUM_PATHS]) override {
    ms[0] = ms[1] = ms[2] = 0.f;
    for (int i = 0; i < (int)w->local.size(); ++i) {
      float t[FLX_NUM_PATHS];
      FLX_TRY(world_read_timing(w, i, seq, t));
      for (int p = 0; p < FLX_NUM_PATHS; ++p) ms[p] = std::max(ms[p], t[p]);
    }
    return flxSuccess;
  }
  flxResult_t agree_max(double* vals, int n) override { return world_agree_max(w, vals, n); }
  uint64_t calls() const override { return w->local[0].calls; }
  std::string scope() const override {
    char name[256] = "gpu";
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, w->local[0].device) == cudaSuccess)
      snprintf(name, sizeof(name), "%s", prop.name);
    for (char* c = name; *c; ++c)
      if (*c == ' ') *c = '_';
    return std::string(name) + (w->loopback ? "/loopback/n" : "/world/n") +
           std::to_string(w->nranks);
  }
  bool cache_writer() const override { return w->local[0].rank == 0; }
};
}  // namespace

flxResult_t run_world_tuned(World* w, const std::vector<const void*>& send,
                            const std::vector<void*>& recv,
                            const std::vector<cudaStream_t>& streams, int coll, size_t count,
                            int dtype, int op, const Comm& lead, bool pinned,
                            const Granules& fallback, int path_mask, size_t alignment) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  FLX_CUDA(cudaStreamIsCapturing(streams[0], &cap));
  const size_t bytes = count * dtype_size(dtype);
  const bool tunable = !pinned && lead.autotune && !w->shared_gpu &&
                       bytes >= lead.tune_min_bytes && !*(volatile uint32_t*)w->abort_word;
  WorldPort port(w);
  TunePolicy pol{lead.tune_s1, lead.tune_s2, lead.have_profile, lead.profile, w->nctas};
  Granules g = fallback;
  bool measured = false;
  FLX_TRY(w->tuner.before_call(port, pol, coll, bytes, tunable,
                               cap == cudaStreamCaptureStatusNone && lead.timing, path_mask,
                               fallback, &g, &measured));
  const uint64_t seq = w->local[0].calls;
  FLX_TRY(run_world(w, send, recv, streams, coll, count, dtype, op, g, alignment, lead.timing));
  w->tuner.after_call(coll, bytes, seq, w->local[0].last_bytes, measured);
  return flxSuccess;
}

// ------------------------------------------------------------ creation
namespace {
// Frees a partially built world when creation fails (the destroy barrier is
// skipped: `boot` is only set once bootstrap has fully succeeded).
struct WorldGuard {
  World* w;
  ~WorldGuard() {
    if (w) world_free(w);
  }
};
}  // namespace

flxResult_t world_create_loopback(int nranks, int device, World** out) {
  if (nranks < 1 || nranks > kMaxRanks)
    return fail(flxInvalidArgument, "loopback supports 1..%d ranks", kMaxRanks);
  auto* w = new World();
  WorldGuard guard{w};
  world_config(w, nranks);
  w->loopback = true;
  w->local.resize(nranks);
  FLX_CUDA(cudaSetDevice(device));
  int coop = 0;
  FLX_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
  if (!coop) return fail(flxInvalidUsage, "device %d lacks cooperative launch", device);
  int sms = 0;
  FLX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  // every CTA of every rank co-resident (cooperative launch): the rank kernels
  // fit 64 registers x 512 threads, i.e. 2 CTAs per SM
  int per_sm = 1;
  per_sm = loopback_blocks_per_sm();
  w->max_nctas = std::max(1, std::min(kMaxCtas, std::max(1, per_sm) * sms / nranks));
  // largest power of two that keeps every rank's CTAs co-resident: 8 ranks
  // get 32 (37 would fit, 32 measured faster), 2-4 ranks 64
  w->nctas = std::min(w->nctas, w->max_nctas);
  while (w->nctas & (w->nctas - 1)) w->nctas &= w->nctas - 1;
  for (int r = 0; r < nranks; ++r) {
    w->local[r].rank = r;
    w->local[r].device = device;
    FLX_TRY(local_init(w, w->local[r]));
  }
  FLX_TRY(alloc_host_staging(w, nullptr));
  guard.w = nullptr;
  *out = w;
  return flxSuccess;
}

// ---- loopback over another process's memory (bootstrap self-test) -----------
// Process B (flxDebugHostRemoteRanks) allocates ranks 1..n-1's scratch and
// flag blocks and exports their CUDA-IPC handles through a shm segment;
// process A (flxCommInitLoopbackIpc) builds a loopback world whose ranks
// 1..n-1 live in those IPC mappings.  The rank kernels then run against
// IPC-mapped peer memory — release/acquire flags, LL packets, pushes and
// pulls — while only process A launches kernels (process B launches none: two
// processes' kernels waiting on each other on one GPU are not guaranteed to be
// co-scheduled, B200_PROFILING.md).
namespace {
struct IpcDebugSeg {
  int ready;  // B published the handles
  int done;   // A is finished with them
  int nranks;
  int pad;
  cudaIpcMemHandle_t scratch[kMaxRanks];
  cudaIpcMemHandle_t flags[kMaxRanks];
};

IpcDebugSeg* map_ipc_debug(const char* id_hex, bool create) {
  char name[96];
  snprintf(name, sizeof(name), "/flx-%s-ipcdbg", id_hex);
  int fd = shm_open(name, create ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
  if (fd < 0) return nullptr;
  if (create && ftruncate(fd, sizeof(IpcDebugSeg)) != 0) {
    close(fd);
    return nullptr;
  }
  void* p = mmap(nullptr, sizeof(IpcDebugSeg), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  return p == MAP_FAILED ? nullptr : static_cast<IpcDebugSeg*>(p);
}
}  // namespace

flxResult_t world_host_remote_ranks(int nranks, int device, const char* id_hex, double seconds) {
  if (nranks < 2 || nranks > kMaxRanks) return fail(flxInvalidArgument, "bad nranks %d", nranks);
  World cfg;
  world_config(&cfg, nranks);
  FLX_CUDA(cudaSetDevice(device));
  IpcDebugSeg* seg = map_ipc_debug(id_hex, true);
  if (!seg) return fail(flxSystemError, "shm for the IPC self-test failed");
  std::vector<char*> scratch(nranks, nullptr);
  std::vector<uint32_t*> flags(nranks, nullptr);
  flxResult_t rc = flxSuccess;
  for (int r = 1; r < nranks && rc == flxSuccess; ++r) {
    rc = alloc_rank_mem(&cfg, &scratch[r], &flags[r]);
    if (rc == flxSuccess && (cudaIpcGetMemHandle(&seg->scratch[r], scratch[r]) != cudaSuccess ||
                             cudaIpcGetMemHandle(&seg->flags[r], flags[r]) != cudaSuccess))
      rc = fail(flxUnhandledCudaError, "cudaIpcGetMemHandle failed");
  }
  if (rc == flxSuccess && cudaDeviceSynchronize() != cudaSuccess)
    rc = fail(flxUnhandledCudaError, "zeroing the exported scratch failed");
  seg->nranks = nranks;
  __atomic_store_n(&seg->ready, rc == flxSuccess ? 1 : -1, __ATOMIC_RELEASE);
  if (rc == flxSuccess &&
      !spin_until([&] { return __atomic_load_n(&seg->done, __ATOMIC_ACQUIRE) != 0; }, seconds))
    rc = fail(flxSystemError, "the loopback process never finished with the exported ranks");
  cudaDeviceSynchronize();
  for (int r = 1; r < nranks; ++r) {
    if (scratch[r]) cudaFree(scratch[r]);
    if (flags[r]) cudaFree(flags[r]);
  }
  munmap(seg, sizeof(IpcDebugSeg));
  return rc;
}

flxResult_t world_create_loopback_ipc(int nranks, int device, const char* id_hex, World** out) {
  IpcDebugSeg* seg = nullptr;
  if (!spin_until([&] { return (seg = map_ipc_debug(id_hex, false)) != nullptr; }, 60.0))
    return fail(flxSystemError, "no exporting process for the IPC self-test");
  if (!spin_until([&] { return __atomic_load_n(&seg->ready, __ATOMIC_ACQUIRE) != 0; }, 60.0) ||
      seg->ready < 0 || seg->nranks != nranks) {
    munmap(seg, sizeof(IpcDebugSeg));
    return fail(flxSystemError, "the exporting process did not publish %d ranks", nranks);
  }
  auto* w = new World();
  WorldGuard guard{w};
  world_config(w, nranks);
  w->loopback = true;
  w->ipc_debug = seg;
  w->local.resize(nranks);
  FLX_CUDA(cudaSetDevice(device));
  int sms = 0, per_sm = 1;
  FLX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  per_sm = loopback_blocks_per_sm();
  w->max_nctas = std::max(1, std::min(kMaxCtas, std::max(1, per_sm) * sms / nranks));
  world_set_nctas(w, 0);
  for (int r = 0; r < nranks; ++r) {
    World::Local& L = w->local[r];
    L.rank = r;
    L.device = device;
    if (r > 0) {
      void* p = nullptr;
      FLX_CUDA(cudaIpcOpenMemHandle(&p, seg->scratch[r], cudaIpcMemLazyEnablePeerAccess));
      L.scratch = static_cast<char*>(p);
      L.remote_mem = true;
      FLX_CUDA(cudaIpcOpenMemHandle(&p, seg->flags[r], cudaIpcMemLazyEnablePeerAccess));
      L.flags = static_cast<uint32_t*>(p);
    }
    FLX_TRY(local_init(w, L));
  }
  FLX_TRY(alloc_host_staging(w, nullptr));
  guard.w = nullptr;
  *out = w;
  return flxSuccess;
}

flxResult_t world_create_rank(int nranks, int rank, int device, const char* id_hex, World** out) {
  auto* w = new World();
  WorldGuard guard{w};
  world_config(w, nranks);
  w->local.resize(1);
  w->local[0].rank = rank;
  w->local[0].device = device;
  FLX_TRY(local_init(w, w->local[0]));

  char boot_name[96], stage_name[96];
  snprintf(boot_name, sizeof(boot_name), "/flx-%s-boot", id_hex);
  snprintf(stage_name, sizeof(stage_name), "/flx-%s-stage", id_hex);
  int fd = shm_open(boot_name, O_CREAT | O_RDWR, 0600);
  if (fd < 0) return fail(flxSystemError, "shm_open(%s) failed", boot_name);
  if (ftruncate(fd, sizeof(BootHeader)) != 0) {
    close(fd);
    return fail(flxSystemError, "ftruncate(%s) failed", boot_name);
  }
  auto* hdr = static_cast<BootHeader*>(
      mmap(nullptr, sizeof(BootHeader), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
  close(fd);
  if (hdr == MAP_FAILED) return fail(flxSystemError, "mmap(%s) failed", boot_name);

  BootSlot& mine = hdr->slot[rank];
  FLX_CUDA(cudaIpcGetMemHandle(&mine.scratch, w->local[0].scratch));
  FLX_CUDA(cudaIpcGetMemHandle(&mine.flags, w->local[0].flags));
  FLX_CUDA(cudaDeviceGetPCIBusId(mine.bus_id, sizeof(mine.bus_id), device));
  mine.device = device;
  mine.pid = getpid();
  const bool want_nvls = getenv("FLX_NVLS") && atoi(getenv("FLX_NVLS")) != 0;
  Granules env_g{{0, 0, 0}};
  bool env_set = false;
  FLX_TRY(env_shares(&env_g, &env_set));
  mine.config = BootConfig{(uint64_t)nranks, w->slot, w->small_slot, w->hcap, w->pcie_chunk,
                           w->oneshot_max, (uint64_t)w->ll, (uint64_t)w->nctas,
                           (uint64_t)kSemWords, (uint64_t)want_nvls,
                           pack_env_shares(env_g, env_set)};
  __atomic_store_n(&mine.ready, 1, __ATOMIC_RELEASE);
  __atomic_fetch_add(&hdr->arrived, 1, __ATOMIC_ACQ_REL);
  // ranks of one job can start minutes apart (PyTorch's store waits 30 min)
  const double timeout = getenv("FLX_BOOT_TIMEOUT") ? atof(getenv("FLX_BOOT_TIMEOUT")) : 600.0;
  if (!spin_until([&] { return __atomic_load_n(&hdr->arrived, __ATOMIC_ACQUIRE) >= nranks; },
                  timeout))
    return fail(flxSystemError, "bootstrap timed out: %d of %d ranks arrived",
                __atomic_load_n(&hdr->arrived, __ATOMIC_ACQUIRE), nranks);
  static const char* kFields[] = {"nranks", "FLX_SLOT_MB", "one-shot inbox (FLX_ONESHOT_KB)",
                                  "FLX_PCIE_STAGE_MB", "FLX_PCIE_CHUNK_KB", "FLX_ONESHOT_KB",
                                  "FLX_LL", "FLX_NVLINK_CTAS", "library build (staging words)",
                                  "FLX_NVLS", "FLX_SHARES"};
  for (int p = 0; p < nranks; ++p) {
    const uint64_t* a = reinterpret_cast<const uint64_t*>(&mine.config);
    const uint64_t* b = reinterpret_cast<const uint64_t*>(&hdr->slot[p].config);
    for (size_t f = 0; f < sizeof(BootConfig) / sizeof(uint64_t); ++f)
      if (a[f] != b[f])
        return fail(flxInvalidUsage,
                    "rank %d and rank %d disagree on %s (%llu vs %llu): every rank must use the "
                    "same world settings",
                    rank, p, kFields[f], (unsigned long long)a[f], (unsigned long long)b[f]);
  }
  // any two ranks on one GPU (bootstrap self-tests) keep the whole world off
  // the NVLink-path kernels' autotuning — decided identically on every rank
  for (int p = 0; p < nranks; ++p)
    for (int q = p + 1; q < nranks; ++q)
      if (strcmp(hdr->slot[p].bus_id, hdr->slot[q].bus_id) == 0) w->shared_gpu = true;
  for (int p = 0; p < nranks; ++p) {
    if (p == rank) {
      w->peer_scratch[p] = w->local[0].scratch;
      w->peer_flags[p] = w->local[0].flags;
      continue;
    }
    // FLX_ALLOW_SHARED_GPU: bootstrap self-tests only (no collective may run:
    // the rank kernels of two processes on one GPU would wait on each other)
    if (strcmp(hdr->slot[p].bus_id, mine.bus_id) == 0) {
      if (!getenv("FLX_ALLOW_SHARED_GPU"))
        return fail(flxInvalidUsage, "ranks %d and %d share GPU %s; one GPU per rank", rank, p,
                    mine.bus_id);
    }
    void* ptr = nullptr;
    FLX_CUDA(cudaIpcOpenMemHandle(&ptr, hdr->slot[p].scratch, cudaIpcMemLazyEnablePeerAccess));
    w->ipc_opened.push_back(ptr);
    w->peer_scratch[p] = static_cast<char*>(ptr);
    FLX_CUDA(cudaIpcOpenMemHandle(&ptr, hdr->slot[p].flags, cudaIpcMemLazyEnablePeerAccess));
    w->ipc_opened.push_back(ptr);
    w->peer_flags[p] = static_cast<uint32_t*>(ptr);
  }
  FLX_TRY(alloc_host_staging(w, stage_name));
  __atomic_fetch_add(&hdr->mapped, 1, __ATOMIC_ACQ_REL);
  if (!spin_until([&] { return __atomic_load_n(&hdr->mapped, __ATOMIC_ACQUIRE) >= nranks; },
                  timeout))
    return fail(flxSystemError, "bootstrap timed out mapping the staging segment");
  // NVLink-SHARP: opt-in (FLX_NVLS=1, agreed above), distinct GPUs only; every
  // rank ends with the same verdict (nvls.cu), a failure only leaves it off
  if (want_nvls && !w->shared_gpu) {
    const char* mb = getenv("FLX_NVLS_MB");
    nvls_setup_rank(&w->nvls, &hdr->nvls, rank, nranks, device,
                    (size_t)(mb ? std::max(1, atoi(mb)) : 256) << 20, timeout);
  }
  w->boot = hdr;  // unmapped in world_free, after the destroy barrier
  if (rank == 0) {
    shm_unlink(boot_name);
    shm_unlink(stage_name);
  }
  guard.w = nullptr;
  *out = w;
  return flxSuccess;
}

void world_attach(World* w, int local, Comm* c) { w->local[local].comm = c; }

// Bootstrap self-test: write my scratch head / host region, or read a peer's
// through the IPC mapping / shared segment.  Plain copies, no waiting kernels.
flxResult_t world_debug_peer(World* w, int local, int peer, int host_region, int write,
                             void* buf, size_t bytes) {
  World::Local& L = w->local[local];
  if (peer < 0 || peer >= w->nranks) return fail(flxInvalidArgument, "bad peer %d", peer);
  if (host_region) {
    if (bytes > w->hcap) return fail(flxInvalidArgument, "too many bytes");
    char* region = w->host + kSemWords * 4 + (size_t)(write ? L.rank : peer) * w->hcap;
    if (write)
      memcpy(region, buf, bytes);
    else
      memcpy(buf, region, bytes);
    return flxSuccess;
  }
  if (bytes > w->slot) return fail(flxInvalidArgument, "too many bytes");
  FLX_CUDA(cudaSetDevice(L.device));
  char* dev = write ? L.scratch : (w->loopback ? w->local[peer].scratch : w->peer_scratch[peer]);
  FLX_CUDA(cudaMemcpy(write ? dev : buf, write ? buf : dev, bytes,
                      write ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost));
  return flxSuccess;
}

flxResult_t world_finalize(World* w, int local) {
  World::Local& L = w->local[local];
  FLX_CUDA(cudaSetDevice(L.device));
  FLX_CUDA(cudaStreamSynchronize(L.d2h));
  FLX_CUDA(cudaStreamSynchronize(L.h2d));
  if (*(volatile uint32_t*)w->abort_word)
    return fail(flxInternalError, "a peer wait timed out (rank died or hung?)");
  return flxSuccess;
}

void world_abort(World* w) {
  *(volatile uint32_t*)w->abort_word = 1;  // any kernel still spinning on a peer gives up
  w->aborting = true;
}

int world_release(World* w) {
  if (++w->destroyed < (int)w->local.size()) return 0;
  world_free(w);
  return 1;
}

flxResult_t world_agree(World* w, double* vals, int n) { return world_agree_max(w, vals, n); }

cudaError_t preload_world_cu() {
  return preload_module((const void*)rank_allgather_kernel);
}

}  // namespace flx
