// libflexlink.so — C-ABI, communicators, groups, and the striped executor.
//
// One collective call = partition the message by the comm's granule shares
// (collectives.py:93-114), then run every path's slice concurrently:
//   NVLink slice : one fused kernel on the caller's stream (kernels.cuh)
//   PCIe slice   : chunked D2H -> pinned host -> H2D ring on two side streams
//                  gated by monotone counter semaphores (staging.py:176-188),
//                  reduce-on-receive kernel on the consumer stream
// and record per-path CUDA events so flxGetPathTimes can hand the balancer a
// PathTimingReport (collectives.py:117-133).
#include <dlfcn.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <random>
#include <vector>

#include "internal.h"
#include "rank_launch.h"
#include "args.h"
#include "autotune.h"

namespace flx {

// ------------------------------------------------------------------ errors
namespace {
thread_local std::string t_last_error = "no error";
}

flxResult_t fail(flxResult_t code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_last_error = buf;
  if (getenv("FLX_DEBUG")) fprintf(stderr, "[flexlink] error %d: %s\n", (int)code, buf);
  return code;
}

// --------------------------------------------------------- driver memops
const MemOps& memops() {
  static MemOps ops;
  static std::once_flag once;
  std::call_once(once, [] {
    void* w = nullptr;
    void* x = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) ==
            cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWriteValue32", &x, cudaEnableDefault, &q2) ==
            cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess) {
      ops.wait32 = reinterpret_cast<decltype(ops.wait32)>(w);
      ops.write32 = reinterpret_cast<decltype(ops.write32)>(x);
      ops.ok = true;
    }
  });
  return ops;
}

// ------------------------------------------------------- context guard
namespace {
struct CtxOps {
  CUresult (*get)(CUcontext*) = nullptr;
  CUresult (*set)(CUcontext) = nullptr;
};
const CtxOps& ctx_ops() {
  static CtxOps ops;
  static std::once_flag once;
  std::call_once(once, [] {
    void* g = nullptr;
    void* s = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuCtxGetCurrent", &g, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuCtxSetCurrent", &s, cudaEnableDefault, &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess) {
      ops.get = reinterpret_cast<CUresult (*)(CUcontext*)>(g);
      ops.set = reinterpret_cast<CUresult (*)(CUcontext)>(s);
    }
  });
  return ops;
}
}  // namespace

CtxGuard::CtxGuard() {
  const CtxOps& o = ctx_ops();
  ok = o.get && o.get(&saved) == CUDA_SUCCESS;
}
CtxGuard::~CtxGuard() {
  if (ok) ctx_ops().set(saved);
}

// ---------------------------------------------------- kernel preloading
namespace {
struct ModuleOps {
  CUresult (*get_module)(CUmodule*, CUfunction) = nullptr;
  CUresult (*count)(unsigned int*, CUmodule) = nullptr;
  CUresult (*enumerate)(CUfunction*, unsigned int, CUmodule) = nullptr;
  CUresult (*load)(CUfunction) = nullptr;
  bool ok = false;
};
template <typename F>
bool driver_entry(const char* name, F* out) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return false;
  *out = reinterpret_cast<F>(p);
  return true;
}
const ModuleOps& module_ops() {
  static ModuleOps ops;
  static std::once_flag once;
  std::call_once(once, [] {
    ops.ok = driver_entry("cuFuncGetModule", &ops.get_module) &&
             driver_entry("cuModuleGetFunctionCount", &ops.count) &&
             driver_entry("cuModuleEnumerateFunctions", &ops.enumerate) &&
             driver_entry("cuFuncLoad", &ops.load);
  });
  return ops;
}
}  // namespace

cudaError_t preload_module(const void* kernel) {
  cudaFunction_t fn = nullptr;
  cudaError_t e = cudaGetFuncBySymbol(&fn, kernel);  // loads this kernel
  if (e != cudaSuccess) return e;
  const ModuleOps& m = module_ops();
  if (!m.ok) return cudaSuccess;  // older driver: first launches load lazily
  CUmodule mod = nullptr;
  unsigned int n = 0;
  if (m.get_module(&mod, reinterpret_cast<CUfunction>(fn)) != CUDA_SUCCESS ||
      m.count(&n, mod) != CUDA_SUCCESS)
    return cudaErrorUnknown;
  std::vector<CUfunction> fns(n);
  if (n && m.enumerate(fns.data(), n, mod) != CUDA_SUCCESS) return cudaErrorUnknown;
  for (CUfunction f : fns)
    if (m.load(f) != CUDA_SUCCESS) return cudaErrorUnknown;
  return cudaSuccess;
}

cudaError_t preload_all_kernels() {
  static std::mutex mu;
  static uint64_t done = 0;  // bit per device ordinal
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  const uint64_t bit = 1ull << (dev & 63);
  if (done & bit) return cudaSuccess;
  for (cudaError_t (*f)() : {preload_launch_cu, preload_world_cu, preload_nvls_cu, preload_rank_i8,
                             preload_rank_i32, preload_rank_i64, preload_rank_f16,
                             preload_rank_f32, preload_rank_f64})
    if ((e = f()) != cudaSuccess) return e;
  done |= bit;
  return cudaSuccess;
}

// Counter semaphores on pinned host words.  GEQ is the cyclic 32-bit
// comparison ((int32)(*addr - value) >= 0), so monotone counters may wrap.
flxResult_t sem_wait_geq(cudaStream_t s, uint32_t* word, uint32_t value) {
  const MemOps& m = memops();
  if (!m.ok) return fail(flxInternalError, "stream memory operations unavailable");
  CUresult r = m.wait32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(word),
                        value, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(flxUnhandledCudaError, "cuStreamWaitValue32: %d", (int)r);
  return flxSuccess;
}

flxResult_t sem_wait_eq(cudaStream_t s, uint32_t* word, uint32_t value) {
  const MemOps& m = memops();
  if (!m.ok) return fail(flxInternalError, "stream memory operations unavailable");
  CUresult r = m.wait32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(word),
                        value, CU_STREAM_WAIT_VALUE_EQ);
  if (r != CUDA_SUCCESS) return fail(flxUnhandledCudaError, "cuStreamWaitValue32: %d", (int)r);
  return flxSuccess;
}

flxResult_t sem_write(cudaStream_t s, uint32_t* word, uint32_t value) {
  const MemOps& m = memops();
  if (!m.ok) return fail(flxInternalError, "stream memory operations unavailable");
  CUresult r = m.write32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(word),
                         value, CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return fail(flxUnhandledCudaError, "cuStreamWriteValue32: %d", (int)r);
  return flxSuccess;
}

size_t dtype_size(int dtype) {
  switch (dtype) {
    case flxInt8: case flxUint8: return 1;
    case flxFloat16: case flxBfloat16: return 2;
    case flxInt32: case flxUint32: case flxFloat32: return 4;
    case flxInt64: case flxUint64: case flxFloat64: return 8;
  }
  return 0;
}

// ---------------------------------------------------------------- shares
int size_bucket(size_t bytes) {
  if (bytes == 0) return -1;
  return 63 - __builtin_clzll((unsigned long long)bytes);
}

Granules ShareTable::lookup(int op, size_t bytes) const {
  auto it = entries.find({op, size_bucket(bytes)});
  return it == entries.end() ? fallback : it->second;
}

std::array<size_t, FLX_NUM_PATHS> partition(size_t bytes, const Granules& g, size_t alignment) {
  std::array<size_t, FLX_NUM_PATHS> out{{0, 0, 0}};
  long long denom = 0;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) denom += g[p];
  size_t used = 0;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) {
    const unsigned __int128 raw =
        denom ? (unsigned __int128)bytes * (unsigned)g[p] / (unsigned long long)denom : 0;
    out[p] = (size_t)raw / alignment * alignment;
    used += out[p];
  }
  out[flxPathNvlink] += bytes - used;
  return out;
}

// ------------------------------------------------------------- registry
namespace {

std::mutex g_mutex;

size_t allreduce_alignment(int nranks) { return (size_t)nranks * 4096; }
constexpr size_t kAllGatherAlignment = 4096;

size_t alignment_for(const Comm* c, int coll) {
  return coll == flxCollAllReduce ? allreduce_alignment(c->nranks) : kAllGatherAlignment;
}

int path_mask() {
  int mask = 1 << flxPathNvlink;
  if (memops().ok) mask |= 1 << flxPathPcie;
  // RDMA NIC loopback needs ibverbs (rdma-core); not built in this image.
  return mask;
}

// The device the caller made current.  This library carries its own (static)
// CUDA runtime, whose per-thread "current device" is not the one torch's
// runtime set; the driver's current context is shared by both, so ask it.
flxResult_t current_device(int* dev) {
  static CUresult (*ctx_get_device)(CUdevice*) = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuCtxGetDevice", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      ctx_get_device = reinterpret_cast<CUresult (*)(CUdevice*)>(fn);
  });
  CUdevice d;
  if (ctx_get_device && ctx_get_device(&d) == CUDA_SUCCESS) {
    *dev = (int)d;
    return flxSuccess;
  }
  FLX_CUDA(cudaGetDevice(dev));
  return flxSuccess;
}

flxResult_t validate_comm(const flxComm* comm);

flxResult_t clique_create(int device, int members, Clique** out) {
  FLX_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  FLX_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(flxInvalidUsage, "device %d is sm_%d%d; this build targets sm_100a", device,
                prop.major, prop.minor);
  FLX_CUDA(preload_all_kernels());  // first launches never wait on a lazy module load
  auto* c = new Clique();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  c->gpu_name = prop.name;
  c->tuner = new AutoTuner();
  FLX_CUDA(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
  FLX_CUDA(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
  FLX_CUDA(cudaStreamCreateWithFlags(&c->red, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b) {
    for (int m = 0; m < 2; ++m) {
      FLX_CUDA(cudaEventCreateWithFlags(&c->ev_landed[m][b], cudaEventDisableTiming));
      FLX_CUDA(cudaEventCreateWithFlags(&c->ev_folded[m][b], cudaEventDisableTiming));
    }
    FLX_CUDA(cudaEventCreateWithFlags(&c->ev_filled[b], cudaEventDisableTiming));
    FLX_CUDA(cudaEventCreateWithFlags(&c->ev_drained[b], cudaEventDisableTiming));
  }
  for (auto& t : c->timing) {
    FLX_CUDA(cudaEventCreate(&t.start));
    FLX_CUDA(cudaEventCreate(&t.nv));
    FLX_CUDA(cudaEventCreate(&t.pcie));
  }
  FLX_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  FLX_CUDA(cudaEventCreateWithFlags(&c->ev_start_nt, cudaEventDisableTiming));
  FLX_CUDA(cudaEventCreateWithFlags(&c->ev_pcie_nt, cudaEventDisableTiming));
  c->ev_fork.resize(members);
  for (auto& e : c->ev_fork) FLX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // semaphore words: [0,B) semFull, [B,2B) semEmpty; start at zero (staging.py:224-225)
  // Producer and consumer streams live on the same GPU here, so the words sit
  // in device memory (the front end polls them without a PCIe round trip);
  // FLX_SEM_HOST=1 puts them in pinned host memory as cross-process worlds must.
  c->sems_on_host = getenv("FLX_SEM_HOST") != nullptr;
  if (c->sems_on_host) {
    FLX_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->sems), 4096,
                           cudaHostAllocMapped | cudaHostAllocPortable));
    memset(c->sems, 0, 4096);
  } else {
    FLX_CUDA(cudaMalloc(reinterpret_cast<void**>(&c->sems), 4096));
    FLX_CUDA(cudaMemset(c->sems, 0, 4096));
    FLX_CUDA(cudaDeviceSynchronize());
  }
  *out = c;
  return flxSuccess;
}

flxResult_t clique_destroy(Clique* c) {
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->d2h);
  cudaStreamSynchronize(c->h2d);
  cudaStreamSynchronize(c->red);
  cudaStreamDestroy(c->d2h);
  cudaStreamDestroy(c->h2d);
  cudaStreamDestroy(c->red);
  for (int b = 0; b < 2; ++b) {
    for (int m = 0; m < 2; ++m) {
      cudaEventDestroy(c->ev_landed[m][b]);
      cudaEventDestroy(c->ev_folded[m][b]);
    }
    cudaEventDestroy(c->ev_filled[b]);
    cudaEventDestroy(c->ev_drained[b]);
  }
  for (auto& t : c->timing) {
    cudaEventDestroy(t.start);
    cudaEventDestroy(t.nv);
    cudaEventDestroy(t.pcie);
  }
  cudaEventDestroy(c->ev_join);
  cudaEventDestroy(c->ev_start_nt);
  cudaEventDestroy(c->ev_pcie_nt);
  for (auto e : c->ev_fork) cudaEventDestroy(e);
  if (c->host_stage) cudaFreeHost(c->host_stage);
  if (c->dev_stage) cudaFree(c->dev_stage);
  for (char* p : c->retired_host) cudaFreeHost(p);
  for (char* p : c->retired_dev) cudaFree(p);
  if (c->sems) c->sems_on_host ? cudaFreeHost(c->sems) : cudaFree(c->sems);
  delete c->tuner;
  delete c;
  return flxSuccess;
}

// Grow the staging ring to hold `chunk` bytes per member in `bufs` buffers.
// Grow-only: a CUDA graph captured earlier bakes the current ring's pointers
// into its copy nodes, so a ring is never freed while the clique lives — a
// larger ring replaces it and the old one is retired (freed in
// clique_destroy).  Capacities are powers of two from 4 MiB per member, so a
// handful of sizes covers every message.
flxResult_t ensure_staging(Clique* c, size_t chunk, int bufs) {
  if (c->stage_cap >= chunk && c->stage_bufs >= bufs) {
    if (c->ring_depth == bufs) return flxSuccess;
    // a new pipeline depth re-indexes the counter words: restart the protocol
    FLX_CUDA(cudaStreamSynchronize(c->d2h));
    FLX_CUDA(cudaStreamSynchronize(c->h2d));
    FLX_CUDA(cudaStreamSynchronize(c->red));
    if (c->sems_on_host)
      memset(c->sems, 0, 4096);
    else
      FLX_CUDA(cudaMemset(c->sems, 0, 4096));
    FLX_CUDA(cudaDeviceSynchronize());
    c->piece_seq = 0;
    c->ring_depth = bufs;
    return flxSuccess;
  }
  FLX_CUDA(cudaStreamSynchronize(c->d2h));
  FLX_CUDA(cudaStreamSynchronize(c->h2d));
  FLX_CUDA(cudaStreamSynchronize(c->red));
  if (c->host_stage) c->retired_host.push_back(c->host_stage);
  if (c->dev_stage) c->retired_dev.push_back(c->dev_stage);
  c->host_stage = nullptr;
  c->dev_stage = nullptr;
  size_t cap = std::max<size_t>(4 << 20, c->stage_cap);
  while (cap < chunk) cap <<= 1;
  const int nb = std::max(std::max(bufs, c->stage_bufs), 2);
  const size_t total = cap * c->members.size() * nb;
  FLX_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->host_stage), total, cudaHostAllocPortable));
  FLX_CUDA(cudaMalloc(reinterpret_cast<void**>(&c->dev_stage), total));
  // a fresh ring starts a fresh protocol epoch: counters restart from zero
  if (c->sems_on_host)
    memset(c->sems, 0, 4096);
  else
    FLX_CUDA(cudaMemset(c->sems, 0, 4096));
  FLX_CUDA(cudaDeviceSynchronize());
  c->piece_seq = 0;
  c->stage_cap = cap;
  c->stage_bufs = nb;
  c->ring_depth = bufs;
  return flxSuccess;
}

// Chunk size per member for a PCIe slice of `bytes` per rank: the configured
// value, or 5 pipeline stages of up to 12 MiB (4 KiB multiples).  Each chunk
// costs N D2H copies + one 2-D H2D + a fold launch + four stream memory ops,
// so small chunks are overhead-bound and few large ones pay the pipeline fill:
// measured on B200, 8 ranks (profiles/r2/pcie_chunks_*.jsonl), a 56 MiB slice
// runs 11.84 ms at 4 MiB chunks and 11.58 at 8-12 MiB, a 14 MiB slice is
// fastest at 3-4 MiB, a PCIe-only 256 MiB message moves 41.6 GB/s each way at
// 4 MiB and 45.7 at 16 MiB.
//
// The stage COUNT is what is held fixed — 5, fewer for slices under 5 x 64 KiB,
// more once a stage would exceed 12 MiB — so it changes only at those
// thresholds and the PCIe path's time grows smoothly with its share.  (A chunk
// size derived per call made the count jump 5 -> 6 with a few KiB of share: one
// granule moved the PCIe time by a whole stage and Stage 1 cycled between
// "move 1 nvlink->pcie" and "move 1 pcie->nvlink" at 2-4 MiB messages.)
size_t pick_chunk(const Comm* lead, size_t bytes) {
  size_t chunk = lead->chunk_bytes;
  if (chunk == 0) {
    const size_t few = std::min<size_t>(5, std::max<size_t>(1, bytes / (64 << 10)));
    const size_t stages = std::max<size_t>((bytes + kMaxAutoChunk - 1) / kMaxAutoChunk, few);
    chunk = std::max<size_t>(4096, ((bytes + stages - 1) / stages + 4095) / 4096 * 4096);
  }
  return chunk;
}

// ---------------------------------------------------------------- groups
struct Call {
  Comm* comm;
  int coll;  // flxCollOp_t
  const void* send;
  void* recv;
  size_t count;
  int dtype;
  int op;
  cudaStream_t stream;
  bool avg = false;  // FLX_OP_AVG: ran as a sum; recv is divided by nranks afterwards
  void* tmp = nullptr;  // flxReduce / flxGather / flxScatter scratch, freed after
  void* tmp2 = nullptr;
  // flxScatter: after the collective, copy bytes from post_src to post_dst
  void* post_dst = nullptr;
  const void* post_src = nullptr;
  size_t post_bytes = 0;
};

thread_local int t_group_depth = 0;
thread_local std::vector<void*> t_freed;  // scratch finish_calls released in this flush
thread_local std::vector<Call> t_pending;

// The autotuner's view of a clique: one timing ring, one process (no
// agreement needed — every virtual rank shares the same events).
struct CliquePort : TimingPort {
  Clique* c;
  explicit CliquePort(Clique* c_) : c(c_) {}
  flxResult_t read(uint64_t seq, float ms[FLX_NUM_PATHS]) override;
  flxResult_t agree_max(double*, int) override { return flxSuccess; }
  uint64_t calls() const override { return c->calls; }
  std::string scope() const override {
    std::string name = c->gpu_name;
    for (char& ch : name)
      if (ch == ' ') ch = '_';
    return name + "/virtual/n" + std::to_string(c->members.size());
  }
  bool cache_writer() const override { return true; }
};

// One collective over all members of a clique.  calls[i] belongs to member i.
flxResult_t run_clique(Clique* c, const std::vector<Call>& calls) {
  const int n = (int)c->members.size();
  const Call& head = calls[0];
  const Comm* lead = head.comm;
  for (int i = 1; i < n; ++i) {
    const Call& k = calls[i];
    if (k.coll != head.coll || k.count != head.count || k.dtype != head.dtype ||
        k.op != head.op)
      return fail(flxInvalidUsage, "rank %d called a different collective than rank 0", i);
    const Comm* m = k.comm;
    if (m->nvlink_ctas != lead->nvlink_ctas || m->chunk_bytes != lead->chunk_bytes ||
        m->buffers != lead->buffers || m->timing != lead->timing)
      return fail(flxInvalidUsage, "rank %d path configuration differs from rank 0", i);
  }
  FLX_CUDA(cudaSetDevice(c->device));
  const size_t esz = dtype_size(head.dtype);
  const size_t bytes = head.count * esz;  // per-rank send bytes
  const Granules fallback = lead->shares[head.coll].lookup(head.coll, bytes);
  const bool pinned = lead->shares[head.coll].pinned(head.coll, bytes);
  for (int i = 1; i < n; ++i) {
    const Comm* m = calls[i].comm;
    if (m->shares[head.coll].lookup(head.coll, bytes) != fallback ||
        m->shares[head.coll].pinned(head.coll, bytes) != pinned)
      return fail(flxInvalidUsage, "rank %d has different shares than rank 0", i);
    if (m->autotune != lead->autotune || m->tune_min_bytes != lead->tune_min_bytes)
      return fail(flxInvalidUsage, "rank %d has a different autotune setting than rank 0", i);
  }
  cudaStream_t s0 = head.stream;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  FLX_CUDA(cudaStreamIsCapturing(s0, &cap));
  const bool capturing = cap == cudaStreamCaptureStatusActive;
  // the split: the pinned / default share table, or the in-library balancer's
  Granules g = fallback;
  bool measured = false;
  {
    // untimed calls (flxSetTiming 0) and captures keep the bucket's tuned split
    // but take no tuning step: there is nothing to measure
    const bool tunable = !pinned && lead->autotune && bytes >= lead->tune_min_bytes;
    CliquePort port(c);
    const TunePolicy pol{lead->tune_s1, lead->tune_s2, lead->have_profile, lead->profile,
                         lead->nvlink_ctas};
    FLX_TRY(c->tuner->before_call(port, pol, head.coll, bytes, tunable,
                                  !capturing && lead->timing, path_mask(), fallback, &g,
                                  &measured));
  }
  auto split = partition(bytes, g, alignment_for(lead, head.coll));
  if (split[flxPathRdma] > 0)
    return fail(flxInvalidUsage, "rdma path is not available on this box");
  if (split[flxPathPcie] > 0 && !(path_mask() & (1 << flxPathPcie)))
    return fail(flxInvalidUsage, "pcie path is not available (no stream memory ops)");

  // fork: every member's stream joins the lead stream
  for (int i = 1; i < n; ++i) {
    if (calls[i].stream == s0) continue;
    FLX_CUDA(cudaEventRecord(c->ev_fork[i], calls[i].stream));
    FLX_CUDA(cudaStreamWaitEvent(s0, c->ev_fork[i], 0));
  }
  Clique::Timing& tm = c->timing[c->calls % Clique::kTimingSlots];
  const size_t nv = split[flxPathNvlink];
  const size_t pc = split[flxPathPcie];
  const auto offs = path_offsets(split);
  const size_t off_nv = offs[flxPathNvlink], off_pc = offs[flxPathPcie];
  // events recorded inside a capture are graph edges, not timestamps
  const bool timed = lead->timing && !capturing;
  const cudaEvent_t ev_start = timed ? tm.start : c->ev_start_nt;
  const cudaEvent_t ev_pcie = timed ? tm.pcie : c->ev_pcie_nt;
  if (timed || pc > 0) FLX_CUDA(cudaEventRecord(ev_start, s0));

  // Uncapped, the fold runs one 16 B vector per thread (grid = slice/8 KiB):
  // measured 6.73 TB/s vs 6.24 TB/s for one persistent CTA per SM
  // (profiles/r1/fold_variants_standalone.jsonl) — CTA turnover hides the
  // tail and DRAM turnaround better than a grid-stride loop.  A cap
  // (flxSetNvlinkCtas, config 4) makes it a persistent grid-stride kernel.
  static const int ctas_per_sm = getenv("FLX_FOLD_CTAS_PER_SM") ? atoi(getenv("FLX_FOLD_CTAS_PER_SM")) : 0;
  const size_t nvec_nv = split[flxPathNvlink] / 16;
  const int grid_nv =
      lead->nvlink_ctas > 0 ? lead->nvlink_ctas
      : ctas_per_sm > 0     ? c->sm_count * ctas_per_sm
                            : (int)std::max<size_t>(c->sm_count,
                                                    std::min<size_t>((nvec_nv + 511) / 512, 1u << 30));
  const bool gather = head.coll == flxCollAllGather;
  const bool scatter = head.coll == flxCollReduceScatter;
  const bool a2a = head.coll == flxCollAllToAll;
  const bool rows = scatter || a2a;  // n x n (source, block) rows per piece

  // ---- PCIe slice: issue the side-stream pipeline first so its copies start
  // while the NVLink kernel runs.
  if (pc > 0) {
    // ReduceScatter / AllToAll stage every (source, row) pair: n*n rows of one
    // chunk, so their automatic chunk keeps a slot at <= 32 MiB per member
    size_t chunk = pick_chunk(lead, pc);
    if (rows && lead->chunk_bytes == 0)
      chunk = std::max<size_t>(4096, std::min(chunk, ((32u << 20) / n) & ~(size_t)4095));
    const size_t need = rows ? chunk * n : chunk;
    if (capturing && (c->stage_cap < need || c->ring_depth != lead->buffers))
      return fail(flxInvalidUsage,
                  "PCIe staging must be sized before CUDA-graph capture: run the collective "
                  "once eagerly with the same size/shares first");
    FLX_TRY(ensure_staging(c, need, lead->buffers));
    const int bufs = c->ring_depth;
    const size_t pitch = rows ? chunk : c->stage_cap;  // row pitch in the slot
    const size_t slot_bytes = c->stage_cap * n;
    FLX_CUDA(cudaStreamWaitEvent(c->d2h, ev_start, 0));
    FLX_CUDA(cudaStreamWaitEvent(c->h2d, ev_start, 0));
    uint64_t local_piece = 0;
    // inside a capture only events recorded earlier in the SAME capture may be
    // awaited; the first use of a slot needs no wait (the graph starts after
    // all earlier work on the caller's stream, including the side streams)
    bool drained_rec[2] = {false, false}, folded_rec[2] = {false, false};
    for (size_t done = 0; done < pc; done += chunk) {
      const size_t len = std::min(chunk, pc - done);
      const size_t at = off_pc + done;  // byte offset inside each rank's message
      // Under capture the monotone counters cannot be baked into a graph that
      // is replayed, so the same handshake is expressed with captured events
      // (graph edges); the eager counters are left untouched.
      const uint64_t piece = capturing ? local_piece++ : c->piece_seq++;
      const int buf = (int)(piece % bufs);
      const uint32_t lap = (uint32_t)(piece / bufs);
      uint32_t* sem_full = c->sems + buf;
      uint32_t* sem_empty = c->sems + bufs + buf;
      char* host = c->host_stage + buf * slot_bytes;
      char* dev = c->dev_stage + buf * slot_bytes;
      // producer: wait slot drained, D2H each rank's piece, mark full
      if (!capturing)
        FLX_TRY(sem_wait_geq(c->d2h, sem_empty, lap));
      else if (drained_rec[buf])
        FLX_CUDA(cudaStreamWaitEvent(c->d2h, c->ev_drained[buf], 0));
      for (int i = 0; i < n; ++i) {
        const char* src = static_cast<const char*>(calls[i].send) + at;
        if (rows)  // this piece of every block r of rank i: rows at stride `bytes`
          FLX_CUDA(cudaMemcpy2DAsync(host + (size_t)i * n * pitch, pitch, src, bytes, len, n,
                                     cudaMemcpyDeviceToHost, c->d2h));
        else
          FLX_CUDA(cudaMemcpyAsync(host + i * pitch, src, len, cudaMemcpyDeviceToHost, c->d2h));
      }
      if (capturing)
        FLX_CUDA(cudaEventRecord(c->ev_filled[buf], c->d2h));
      else
        FLX_TRY(sem_write(c->d2h, sem_full, lap + 1));
      // consumer: wait full (and the device slot drained by its last fold),
      // H2D the whole slot, mark empty; reduce-on-receive runs on its own
      // stream so the next H2D starts immediately
      if (capturing)
        FLX_CUDA(cudaStreamWaitEvent(c->h2d, c->ev_filled[buf], 0));
      else
        FLX_TRY(sem_wait_geq(c->h2d, sem_full, lap + 1));
      if (!capturing || folded_rec[buf])
        FLX_CUDA(cudaStreamWaitEvent(c->h2d, c->ev_folded[capturing][buf], 0));
      FLX_CUDA(cudaMemcpy2DAsync(dev, pitch, host, pitch, len, rows ? n * n : n,
                                 cudaMemcpyHostToDevice, c->h2d));
      if (capturing) {
        FLX_CUDA(cudaEventRecord(c->ev_drained[buf], c->h2d));
        drained_rec[buf] = true;
      } else {
        FLX_TRY(sem_write(c->h2d, sem_empty, lap + 1));
      }
      FLX_CUDA(cudaEventRecord(c->ev_landed[capturing][buf], c->h2d));
      FLX_CUDA(cudaStreamWaitEvent(c->red, c->ev_landed[capturing][buf], 0));
      if (gather) {
        FanoutArgs a{};
        for (int i = 0; i < n; ++i) {
          a.src[i] = dev + i * pitch;
          a.dst[i] = static_cast<char*>(calls[i].recv) + at;
        }
        a.nsrc = a.ndst = n;
        a.bytes = len;
        a.dst_stride = bytes;
        FLX_CUDA(launch_fanout(a, 16, c->red));
      } else if (a2a) {
        XposeArgs a{};
        for (int i = 0; i < n; ++i) {
          a.src[i] = dev + (size_t)i * n * pitch;
          a.dst[i] = static_cast<char*>(calls[i].recv) + at;
        }
        a.n = n;
        a.bytes = len;
        a.src_stride = pitch;
        a.dst_stride = bytes;
        FLX_CUDA(launch_xpose(a, 8, c->red));
      } else if (scatter) {
        RowsArgs a{};
        for (int i = 0; i < n; ++i) {
          a.src[i] = dev + (size_t)i * n * pitch;
          a.dst[i] = static_cast<char*>(calls[i].recv) + at;
        }
        a.n = a.nrows = n;
        a.bytes = len;
        a.src_stride = pitch;
        FLX_CUDA(launch_rows(head.dtype, head.op, a, 8, c->red));
      } else {
        FoldArgs a{};
        for (int i = 0; i < n; ++i) {
          a.src[i] = dev + i * pitch;
          a.dst[i] = static_cast<char*>(calls[i].recv) + at;
        }
        a.n = a.ndst = n;
        a.bytes = len;
        FLX_CUDA(launch_fold(head.dtype, head.op, a, 32, c->red));
      }
      FLX_CUDA(cudaEventRecord(c->ev_folded[capturing][buf], c->red));
      folded_rec[buf] = true;
    }
    FLX_CUDA(cudaEventRecord(ev_pcie, c->red));
  }

  // ---- NVLink slice: one fused kernel over all members on the lead stream
  if (nv > 0) {
    if (gather) {
      FanoutArgs a{};
      for (int i = 0; i < n; ++i) {
        a.src[i] = static_cast<const char*>(calls[i].send) + off_nv;
        a.dst[i] = static_cast<char*>(calls[i].recv) + off_nv;
      }
      a.nsrc = a.ndst = n;
      a.bytes = nv;
      a.dst_stride = bytes;
      // one vector per thread per source row when uncapped (6.25 TB/s vs 5.27
      // persistent, 0.84 of peak for the TMA variant:
      // profiles/r1/fanout_variants_standalone.jsonl); a cap divides over sources
      const int gx = lead->nvlink_ctas > 0
                         ? std::max(1, lead->nvlink_ctas / n)
                         : (int)std::max<size_t>(1, std::min<size_t>((nv / 16 + 511) / 512,
                                                                     1u << 30));
      FLX_CUDA(launch_fanout(a, gx, s0));
    } else if (a2a) {
      XposeArgs a{};
      for (int i = 0; i < n; ++i) {
        a.src[i] = static_cast<const char*>(calls[i].send) + off_nv;
        a.dst[i] = static_cast<char*>(calls[i].recv) + off_nv;
      }
      a.n = n;
      a.bytes = nv;
      a.src_stride = a.dst_stride = bytes;
      FLX_CUDA(launch_xpose(a, lead->nvlink_ctas > 0 ? std::max(1, lead->nvlink_ctas / (n * n))
                                                       : 1 << 30, s0));
    } else if (scatter) {
      RowsArgs a{};
      for (int i = 0; i < n; ++i) {
        a.src[i] = static_cast<const char*>(calls[i].send) + off_nv;
        a.dst[i] = static_cast<char*>(calls[i].recv) + off_nv;
      }
      a.n = a.nrows = n;
      a.bytes = nv;
      a.src_stride = bytes;
      FLX_CUDA(launch_rows(head.dtype, head.op, a, std::max(1, grid_nv / n), s0));
    } else {
      FoldArgs a{};
      for (int i = 0; i < n; ++i) {
        a.src[i] = static_cast<const char*>(calls[i].send) + off_nv;
        a.dst[i] = static_cast<char*>(calls[i].recv) + off_nv;
      }
      a.n = a.ndst = n;
      a.bytes = nv;
      FLX_CUDA(launch_fold(head.dtype, head.op, a, grid_nv, s0));
    }
  }
  if (timed) FLX_CUDA(cudaEventRecord(tm.nv, s0));
  if (pc > 0) FLX_CUDA(cudaStreamWaitEvent(s0, ev_pcie, 0));

  // join: every member's stream waits for the collective
  bool joined = false;
  for (int i = 1; i < n; ++i) {
    if (calls[i].stream == s0) continue;
    if (!joined) {
      FLX_CUDA(cudaEventRecord(c->ev_join, s0));
      joined = true;
    }
    FLX_CUDA(cudaStreamWaitEvent(calls[i].stream, c->ev_join, 0));
  }
  c->last_bytes = split;
  tm.used[flxPathNvlink] = nv > 0 && timed;
  tm.used[flxPathPcie] = pc > 0 && timed;
  tm.used[flxPathRdma] = false;
  c->tuner->after_call(head.coll, bytes, c->calls, split, measured);
  c->calls++;
  return flxSuccess;
}

// One collective over all local ranks of a world (calls[i] = local rank i).
flxResult_t run_world_calls(World* w, const std::vector<Call>& calls) {
  const Call& head = calls[0];
  const Comm* lead = head.comm;
  std::vector<const void*> send;
  std::vector<void*> recv;
  std::vector<cudaStream_t> streams;
  const size_t bytes = head.count * dtype_size(head.dtype);
  const Granules g = lead->shares[head.coll].lookup(head.coll, bytes);
  const bool pinned = lead->shares[head.coll].pinned(head.coll, bytes);
  for (size_t i = 0; i < calls.size(); ++i) {
    const Call& k = calls[i];
    if (k.coll != head.coll || k.count != head.count || k.dtype != head.dtype || k.op != head.op)
      return fail(flxInvalidUsage, "local rank %zu called a different collective", i);
    if (k.comm->shares[head.coll].lookup(head.coll, bytes) != g ||
        k.comm->shares[head.coll].pinned(head.coll, bytes) != pinned)
      return fail(flxInvalidUsage, "local rank %zu has different shares", i);
    if (k.comm->autotune != lead->autotune || k.comm->tune_min_bytes != lead->tune_min_bytes)
      return fail(flxInvalidUsage, "local rank %zu has a different autotune setting", i);
    if (k.comm->timing != lead->timing)
      return fail(flxInvalidUsage, "local rank %zu has a different timing setting", i);
    send.push_back(k.send);
    recv.push_back(k.recv);
    streams.push_back(k.stream);
  }
  return run_world_tuned(w, send, recv, streams, head.coll, head.count, head.dtype, head.op, *lead,
                         pinned, g, path_mask(), alignment_for(lead, head.coll));
}

// After a collective, on each member's own stream (which the collective's join
// already ordered after the data landed): FLX_OP_AVG divides the recv
// (AllReduce: count elements, ReduceScatter: its recvcount block) by nranks;
// flxReduce's non-root scratch is released (stream-ordered)
flxResult_t finish_calls(const std::vector<Call>& calls) {
  for (const Call& k : calls) {
    if (!k.avg && !k.tmp && !k.post_bytes) continue;
    FLX_CUDA(cudaSetDevice(k.comm->device));
    if (k.avg) FLX_CUDA(launch_div(k.dtype, k.recv, k.count, k.comm->nranks, k.stream));
    if (k.post_bytes)
      FLX_CUDA(cudaMemcpyAsync(k.post_dst, k.post_src, k.post_bytes, cudaMemcpyDeviceToDevice,
                               k.stream));
    for (void* t : {k.tmp, k.tmp2})
      if (t) {
        t_freed.push_back(t);
        FLX_CUDA(cudaFreeAsync(t, k.stream));
      }
  }
  return flxSuccess;
}

flxResult_t flush_group_calls(const std::vector<Call>& calls);

// A group that fails before a call ran still releases that call's scratch
// (stream-ordered: after whatever did run).
flxResult_t flush_group() {
  std::vector<Call> calls;
  calls.swap(t_pending);
  t_freed.clear();
  const flxResult_t r = flush_group_calls(calls);
  if (r != flxSuccess)
    for (const Call& k : calls)
      for (void* t : {k.tmp, k.tmp2})
        if (t && std::find(t_freed.begin(), t_freed.end(), t) == t_freed.end()) {
          cudaSetDevice(k.comm->device);
          cudaFreeAsync(t, k.stream);
        }
  return r;
}

flxResult_t flush_group_calls(const std::vector<Call>& calls) {
  // multi-rank worlds: bucket by world, by local rank
  std::map<World*, std::vector<std::vector<Call>>> by_world;
  std::vector<World*> world_order;
  for (const Call& k : calls) {
    if (!k.comm->world) continue;
    auto& per = by_world[k.comm->world];
    if (per.empty()) world_order.push_back(k.comm->world);
    if ((int)per.size() <= k.comm->local) per.resize(k.comm->local + 1);
    per[k.comm->local].push_back(k);
  }
  for (World* w : world_order) {
    auto& per = by_world[w];
    if ((int)per.size() != world_nlocal(w))
      return fail(flxInvalidUsage, "every local rank of a world must take part in the group");
    const size_t rounds = per[0].size();
    for (size_t i = 0; i < per.size(); ++i)
      if (per[i].size() != rounds)
        return fail(flxInvalidUsage, "every local rank of a world must take part in the group");
    for (size_t k = 0; k < rounds; ++k) {
      std::vector<Call> one;
      for (auto& v : per) one.push_back(v[k]);
      FLX_TRY(run_world_calls(w, one));
      FLX_TRY(finish_calls(one));
    }
  }
  // bucket calls by clique, preserving per-member order
  std::map<Clique*, std::vector<std::vector<Call>>> by_clique;
  for (const Call& k : calls) {
    if (k.comm->world) continue;
    Clique* c = k.comm->clique;
    auto& per = by_clique[c];
    if (per.empty()) per.resize(c->members.size());
    per[k.comm->rank - 0].push_back(k);
  }
  for (auto& [clique, per] : by_clique) {
    const size_t rounds = per[0].size();
    for (size_t i = 0; i < per.size(); ++i)
      if (per[i].size() != rounds)
        return fail(flxInvalidUsage,
                    "group issued %zu collectives on rank 0 but %zu on rank %zu of the same "
                    "device; every virtual rank must take part",
                    rounds, per[i].size(), i);
    for (size_t k = 0; k < rounds; ++k) {
      std::vector<Call> one;
      for (auto& v : per) one.push_back(v[k]);
      FLX_TRY(run_clique(clique, one));
      FLX_TRY(finish_calls(one));
    }
  }
  return flxSuccess;
}

flxResult_t enqueue(const Call& in) {
  Call k = in;
  if (k.op == FLX_OP_AVG) {  // the striped sum, then finish_avg
    k.op = flxSum;
    k.avg = true;
  }
  t_pending.push_back(k);
  if (t_group_depth > 0) return flxSuccess;
  return flush_group();
}

// Per-path ms of call number `seq` (must still be in the ring); blocks on it.
flxResult_t read_timing(Clique* c, uint64_t seq, float ms[3]) {
  const Clique::Timing& t = c->timing[seq % Clique::kTimingSlots];
  FLX_CUDA(cudaSetDevice(c->device));
  ms[0] = ms[1] = ms[2] = 0.f;
  FLX_CUDA(cudaEventSynchronize(t.nv));
  if (t.used[flxPathNvlink]) FLX_CUDA(cudaEventElapsedTime(&ms[0], t.start, t.nv));
  if (t.used[flxPathPcie]) {
    FLX_CUDA(cudaEventSynchronize(t.pcie));
    FLX_CUDA(cudaEventElapsedTime(&ms[1], t.start, t.pcie));
  }
  return flxSuccess;
}

flxResult_t CliquePort::read(uint64_t seq, float ms[FLX_NUM_PATHS]) {
  return read_timing(c, seq, ms);
}

void init_tuning(Comm* c) {
  c->autotune = autotune_default();
  c->tune_min_bytes = autotune_min_bytes_default();
  Granules g;
  bool set = false;
  if (env_shares(&g, &set) == flxSuccess && set)  // validated by the init entry points
    for (ShareTable& t : c->shares) {
      t.fallback = g;
      t.fallback_pinned = true;
    }
}

AutoTuner* tuner_of(const Comm* c) { return c->clique ? c->clique->tuner : world_tuner(c->world); }

flxResult_t check_call(const flxComm* comm, int dtype, int op, bool reduce) {
  FLX_TRY(validate_comm(comm));
  if (dtype < 0 || dtype >= flxNumTypes) return fail(flxInvalidArgument, "bad datatype %d", dtype);
  if (reduce && (op < 0 || (op >= flxNumOps && op != FLX_OP_AVG)))
    return fail(flxInvalidArgument, "unsupported reduction op %d", op);
  return flxSuccess;
}

}  // namespace

flxResult_t env_shares(Granules* g, bool* set) {
  *set = false;
  const char* v = getenv("FLX_SHARES");
  if (!v || !*v) return flxSuccess;
  Granules out{{0, 0, 0}};
  int n = 0, sum = 0;
  const char* p = v;
  while (*p && n < FLX_NUM_PATHS) {
    char* end = nullptr;
    const long x = strtol(p, &end, 10);
    if (end == p || x < 0 || x > FLX_GRANULE_TOTAL)
      return fail(flxInvalidArgument, "FLX_SHARES=\"%s\": expected granules \"nvlink,pcie[,rdma]\"", v);
    out[n++] = (int)x;
    sum += (int)x;
    p = *end == ',' ? end + 1 : end;
    if (*end && *end != ',') return fail(flxInvalidArgument, "FLX_SHARES=\"%s\": bad separator", v);
  }
  if (*p || n < 2 || sum != FLX_GRANULE_TOTAL)
    return fail(flxInvalidArgument, "FLX_SHARES=\"%s\": 2 or 3 granules summing to %d", v,
                FLX_GRANULE_TOTAL);
  const int mask = path_mask();
  for (int q = 1; q < FLX_NUM_PATHS; ++q)
    if (out[q] > 0 && !(mask & (1 << q)))
      return fail(flxInvalidArgument, "FLX_SHARES: path %d is not available on this box", q);
  *g = out;
  *set = true;
  return flxSuccess;
}

}  // namespace flx

using namespace flx;

struct flxComm : public flx::Comm {};

namespace flx {
namespace {
flxResult_t validate_comm(const flxComm* comm) {
  if (comm == nullptr) return fail(flxInvalidArgument, "null communicator");
  if (static_cast<const Comm*>(comm)->magic != kCommMagic)
    return fail(flxInvalidArgument,
                "not a live FlexLink communicator (destroyed, or a handle from another library)");
  return flxSuccess;
}
}  // namespace
}  // namespace flx

// ====================================================================== ABI
extern "C" {

flxResult_t flxGetVersion(int* version) {
  if (!version) return fail(flxInvalidArgument, "null version pointer");
  *version = FLX_VERSION_CODE;
  return flxSuccess;
}

const char* flxGetErrorString(flxResult_t r) {
  switch (r) {
    case flxSuccess: return "no error";
    case flxUnhandledCudaError: return "unhandled cuda error";
    case flxSystemError: return "unhandled system error";
    case flxInternalError: return "internal error";
    case flxInvalidArgument: return "invalid argument";
    case flxInvalidUsage: return "invalid usage";
    case flxRemoteError: return "remote process exited or there was a network error";
    case flxInProgress: return "operation in progress";
  }
  return "unknown result code";
}

const char* flxGetLastError(void) { return t_last_error.c_str(); }

void flxSetLastError(const char* message) { t_last_error = message ? message : ""; }

flxResult_t flxGetUniqueId(flxUniqueId* id) {
  if (!id) return fail(flxInvalidArgument, "null id");
  memset(id, 0, sizeof(*id));
  std::random_device rd;
  uint64_t words[4] = {0x31584c46ull /* "FLX1" */, ((uint64_t)rd() << 32) | rd(),
                       ((uint64_t)rd() << 32) | rd(), (uint64_t)getpid()};
  memcpy(id->internal, words, sizeof(words));
  return flxSuccess;
}

flxResult_t flxCommInitAll(flxComm_t* comms, int ndev, const int* devlist) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  {
    Granules g;
    bool set;
    FLX_TRY(env_shares(&g, &set));  // a malformed FLX_SHARES fails here, loudly
  }
  if (!comms || ndev < 1) return fail(flxInvalidArgument, "bad comms/ndev");
  int visible = 0;
  FLX_CUDA(cudaGetDeviceCount(&visible));
  std::vector<int> devs(ndev);
  for (int i = 0; i < ndev; ++i) {
    devs[i] = devlist ? devlist[i] : i;
    if (devs[i] < 0 || devs[i] >= visible)
      return fail(flxInvalidArgument, "device %d not visible (%d devices)", devs[i], visible);
  }
  std::map<int, int> per_device;
  for (int d : devs) per_device[d]++;
  if (per_device.size() > 1)
    return fail(flxInvalidUsage,
                "flxCommInitAll over distinct devices needs the peer-mapped multi-GPU "
                "path; use one process per GPU with flxCommInitRank");
  if (ndev > FLX_MAX_VIRTUAL_RANKS)
    return fail(flxInvalidArgument, "at most %d virtual ranks per device", FLX_MAX_VIRTUAL_RANKS);
  std::lock_guard<std::mutex> lock(g_mutex);
  Clique* c = nullptr;
  FLX_TRY(clique_create(devs[0], ndev, &c));
  for (int i = 0; i < ndev; ++i) {
    auto* comm = new flxComm();
    comm->rank = i;
    comm->nranks = ndev;
    comm->device = devs[i];
    comm->clique = c;
    init_tuning(comm);
    // FLX_NVLINK_CTAS caps the fused NVLink-path kernel (config 4) for
    // programs that only use the NCCL names
    if (const char* v = getenv("FLX_NVLINK_CTAS")) comm->nvlink_ctas = std::max(0, atoi(v));
    c->members.push_back(comm);
    comms[i] = comm;
  }
  return flxSuccess;
}

flxResult_t flxCommInitRank(flxComm_t* comm, int nranks, flxUniqueId id, int rank) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  {
    Granules g;
    bool set;
    FLX_TRY(env_shares(&g, &set));  // a malformed FLX_SHARES fails here, loudly
  }
  if (!comm || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(flxInvalidArgument, "bad comm/nranks/rank");
  uint64_t magic;
  memcpy(&magic, id.internal, sizeof(magic));
  if (magic != 0x31584c46ull) return fail(flxInvalidArgument, "not a flxUniqueId");
  if (nranks > FLX_MAX_VIRTUAL_RANKS)
    return fail(flxInvalidArgument, "at most %d ranks per communicator", FLX_MAX_VIRTUAL_RANKS);
  int dev = 0;
  FLX_TRY(current_device(&dev));
  if (nranks == 1) {
    FLX_TRY(flxCommInitAll(comm, 1, &dev));
    (*comm)->uid = id;
    return flxSuccess;
  }
  cudaDeviceProp prop;
  FLX_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (prop.major < 10)
    return fail(flxInvalidUsage, "device %d is sm_%d%d; this build targets sm_100a", dev,
                prop.major, prop.minor);
  char hex[40];
  uint64_t nonce[2];
  memcpy(nonce, id.internal + 8, sizeof(nonce));
  snprintf(hex, sizeof(hex), "%016llx%016llx", (unsigned long long)nonce[0],
           (unsigned long long)nonce[1]);
  World* w = nullptr;
  FLX_TRY(world_create_rank(nranks, rank, dev, hex, &w));
  auto* c = new flxComm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = dev;
  c->world = w;
  c->uid = id;
  init_tuning(c);
  c->local = 0;
  world_attach(w, 0, c);
  *comm = c;
  return flxSuccess;
}

flxResult_t flxCommSplit(flxComm_t comm, int color, int key, flxComm_t* newcomm) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  if (!newcomm) return fail(flxInvalidArgument, "null newcomm");
  *newcomm = nullptr;
  if (color < 0 && color != FLX_SPLIT_NOCOLOR)
    return fail(flxInvalidArgument, "color %d: a color is >= 0 or FLX_SPLIT_NOCOLOR", color);
  uint64_t magic;
  memcpy(&magic, comm->uid.internal, sizeof(magic));
  const bool single = comm->nranks == 1 && comm->clique && magic == 0x31584c46ull;
  if (!single && (!comm->world || world_nlocal(comm->world) != 1))
    return fail(flxInvalidUsage, "flxCommSplit needs a communicator from flxCommInitRank");
  // every rank's (color, key), agreed through the parent's board: slot 2r is
  // rank r's color, 2r+1 its key; the others contribute -inf
  const int n = comm->nranks;
  std::vector<double> v(2 * (size_t)n, -1e300);
  v[2 * (size_t)comm->rank] = color;
  v[2 * (size_t)comm->rank + 1] = key;
  if (!single) FLX_TRY(world_agree(comm->world, v.data(), 2 * n));
  const uint64_t seq = ++comm->splits;
  if (color == FLX_SPLIT_NOCOLOR) return flxSuccess;
  std::vector<std::pair<double, int>> members;  // (key, parent rank)
  for (int p = 0; p < n; ++p)
    if (v[2 * (size_t)p] == (double)color) members.push_back({v[2 * (size_t)p + 1], p});
  std::sort(members.begin(), members.end());
  int me = -1;
  for (size_t i = 0; i < members.size(); ++i)
    if (members[i].second == comm->rank) me = (int)i;
  // the child's id: the parent's nonce mixed with (split number, color) —
  // identical on every member, distinct for every split and color
  flxUniqueId child = comm->uid;
  uint64_t words[2];
  memcpy(words, child.internal + 8, sizeof(words));
  uint64_t h = 1469598103934665603ull;  // FNV-1a over (seq, color)
  for (uint64_t x : {seq, (uint64_t)(uint32_t)color})
    for (int b = 0; b < 8; ++b) h = (h ^ ((x >> (8 * b)) & 0xff)) * 1099511628211ull;
  words[0] ^= h;
  words[1] ^= h * 0x9e3779b97f4a7c15ull;
  memcpy(child.internal + 8, words, sizeof(words));
  FLX_CUDA(cudaSetDevice(comm->device));
  return flxCommInitRank(newcomm, (int)members.size(), child, me);
}

namespace {
void id_hex(const flxUniqueId& id, char hex[40]) {
  uint64_t nonce[2];
  memcpy(nonce, id.internal + 8, sizeof(nonce));
  snprintf(hex, 40, "%016llx%016llx", (unsigned long long)nonce[0],
           (unsigned long long)nonce[1]);
}
}  // namespace

flxResult_t flxDebugHostRemoteRanks(int nranks, int device, flxUniqueId id, double seconds) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  uint64_t magic;
  memcpy(&magic, id.internal, sizeof(magic));
  if (magic != 0x31584c46ull) return fail(flxInvalidArgument, "not a flxUniqueId");
  char hex[40];
  id_hex(id, hex);
  return world_host_remote_ranks(nranks, device, hex, seconds > 0 ? seconds : 120.0);
}

flxResult_t flxCommInitLoopbackIpc(flxComm_t* comms, int nranks, int device, flxUniqueId id) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  {
    Granules g;
    bool set;
    FLX_TRY(env_shares(&g, &set));  // a malformed FLX_SHARES fails here, loudly
  }
  if (!comms || nranks < 2) return fail(flxInvalidArgument, "bad comms/nranks");
  uint64_t magic;
  memcpy(&magic, id.internal, sizeof(magic));
  if (magic != 0x31584c46ull) return fail(flxInvalidArgument, "not a flxUniqueId");
  char hex[40];
  id_hex(id, hex);
  std::lock_guard<std::mutex> lock(g_mutex);
  World* w = nullptr;
  FLX_TRY(world_create_loopback_ipc(nranks, device, hex, &w));
  for (int r = 0; r < nranks; ++r) {
    auto* c = new flxComm();
    c->rank = r;
    c->nranks = nranks;
    c->device = device;
    c->world = w;
    c->local = r;
    init_tuning(c);
    world_attach(w, r, c);
    comms[r] = c;
  }
  return flxSuccess;
}

flxResult_t flxCommInitLoopback(flxComm_t* comms, int nranks, int device) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  {
    Granules g;
    bool set;
    FLX_TRY(env_shares(&g, &set));  // a malformed FLX_SHARES fails here, loudly
  }
  if (!comms || nranks < 1) return fail(flxInvalidArgument, "bad comms/nranks");
  int visible = 0;
  FLX_CUDA(cudaGetDeviceCount(&visible));
  if (device < 0 || device >= visible) return fail(flxInvalidArgument, "bad device %d", device);
  cudaDeviceProp prop;
  FLX_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(flxInvalidUsage, "device %d is sm_%d%d; this build targets sm_100a", device,
                prop.major, prop.minor);
  std::lock_guard<std::mutex> lock(g_mutex);
  World* w = nullptr;
  FLX_TRY(world_create_loopback(nranks, device, &w));
  for (int r = 0; r < nranks; ++r) {
    auto* c = new flxComm();
    c->rank = r;
    c->nranks = nranks;
    c->device = device;
    c->world = w;
    c->local = r;
    init_tuning(c);
    world_attach(w, r, c);
    comms[r] = c;
  }
  return flxSuccess;
}

flxResult_t flxCommDestroy(flxComm_t comm) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  std::lock_guard<std::mutex> lock(g_mutex);
  if (comm->world) {
    world_release(comm->world);
    comm->magic = 0;
    delete comm;
    return flxSuccess;
  }
  Clique* c = comm->clique;
  c->destroyed++;
  if (c->destroyed == (int)c->members.size()) {
    for (Comm* m : c->members) {
      m->magic = 0;
      delete static_cast<flxComm*>(m);
    }
    clique_destroy(c);
  }
  return flxSuccess;
}

flxResult_t flxCommFinalize(flxComm_t comm) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  if (comm->world) return world_finalize(comm->world, comm->local);
  Clique* c = comm->clique;
  FLX_CUDA(cudaSetDevice(c->device));
  FLX_CUDA(cudaStreamSynchronize(c->d2h));
  FLX_CUDA(cudaStreamSynchronize(c->h2d));
  FLX_CUDA(cudaStreamSynchronize(c->red));
  return flxSuccess;
}

flxResult_t flxCommAbort(flxComm_t comm) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  {
    std::lock_guard<std::mutex> lock(g_mutex);
    if (comm->world) world_abort(comm->world);
  }
  return flxCommDestroy(comm);
}

flxResult_t flxCommCount(const flxComm_t comm, int* count) {
  FLX_TRY(validate_comm(comm));
  if (!count) return fail(flxInvalidArgument, "null count");
  *count = comm->nranks;
  return flxSuccess;
}

flxResult_t flxCommUserRank(const flxComm_t comm, int* rank) {
  FLX_TRY(validate_comm(comm));
  if (!rank) return fail(flxInvalidArgument, "null rank");
  *rank = comm->rank;
  return flxSuccess;
}

flxResult_t flxCommCuDevice(const flxComm_t comm, int* device) {
  FLX_TRY(validate_comm(comm));
  if (!device) return fail(flxInvalidArgument, "null device");
  *device = comm->device;
  return flxSuccess;
}

flxResult_t flxCommGetAsyncError(flxComm_t comm, flxResult_t* async_error) {
  FLX_TRY(validate_comm(comm));
  if (!async_error) return fail(flxInvalidArgument, "null async_error");
  *async_error = comm->world && world_aborted(comm->world) ? flxInternalError : flxSuccess;
  return flxSuccess;
}

flxResult_t flxAllReduce(const void* sendbuff, void* recvbuff, size_t count,
                         flxDataType_t datatype, flxRedOp_t op, flxComm_t comm,
                         cudaStream_t stream) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(check_call(comm, datatype, op, true));
  if (count > 0 && (!sendbuff || !recvbuff)) return fail(flxInvalidArgument, "null buffer");
  return enqueue(Call{comm, flxCollAllReduce, sendbuff, recvbuff, count, datatype, op, stream});
}

flxResult_t flxAllGather(const void* sendbuff, void* recvbuff, size_t sendcount,
                         flxDataType_t datatype, flxComm_t comm, cudaStream_t stream) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(check_call(comm, datatype, 0, false));
  if (sendcount > 0 && (!sendbuff || !recvbuff)) return fail(flxInvalidArgument, "null buffer");
  return enqueue(Call{comm, flxCollAllGather, sendbuff, recvbuff, sendcount, datatype, 0, stream});
}

flxResult_t flxReduceScatter(const void* sendbuff, void* recvbuff, size_t recvcount,
                             flxDataType_t datatype, flxRedOp_t op, flxComm_t comm,
                             cudaStream_t stream) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(check_call(comm, datatype, op, true));
  if (recvcount > 0 && (!sendbuff || !recvbuff)) return fail(flxInvalidArgument, "null buffer");
  return enqueue(
      Call{comm, flxCollReduceScatter, sendbuff, recvbuff, recvcount, datatype, op, stream});
}

flxResult_t flxAllToAll(const void* sendbuff, void* recvbuff, size_t count,
                        flxDataType_t datatype, flxComm_t comm, cudaStream_t stream) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(check_call(comm, datatype, 0, false));
  if (count > 0 && (!sendbuff || !recvbuff)) return fail(flxInvalidArgument, "null buffer");
  if (count > 0 && sendbuff == recvbuff)
    return fail(flxInvalidArgument, "in-place AllToAll is not supported");
  return enqueue(Call{comm, flxCollAllToAll, sendbuff, recvbuff, count, datatype, 0, stream});
}

flxResult_t flxReduce(const void* sendbuff, void* recvbuff, size_t count,
                      flxDataType_t datatype, flxRedOp_t op, int root, flxComm_t comm,
                      cudaStream_t stream) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(check_call(comm, datatype, op, true));
  if (root < 0 || root >= comm->nranks) return fail(flxInvalidArgument, "bad root %d", root);
  const bool is_root = comm->rank == root;
  if (count > 0 && (!sendbuff || (is_root && !recvbuff)))
    return fail(flxInvalidArgument, "null buffer");
  Call k{comm, flxCollAllReduce, sendbuff, recvbuff, count, datatype, op, stream};
  if (!is_root && count > 0) {  // the striped AllReduce lands in scratch here
    FLX_CUDA(cudaSetDevice(comm->device));
    FLX_CUDA(cudaMallocAsync(&k.tmp, count * dtype_size(datatype), stream));
    k.recv = k.tmp;
  }
  return enqueue(k);
}

flxResult_t flxGather(const void* sendbuff, void* recvbuff, size_t count,
                      flxDataType_t datatype, int root, flxComm_t comm, cudaStream_t stream) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(check_call(comm, datatype, 0, false));
  if (root < 0 || root >= comm->nranks) return fail(flxInvalidArgument, "bad root %d", root);
  const bool is_root = comm->rank == root;
  if (count > 0 && (!sendbuff || (is_root && !recvbuff)))
    return fail(flxInvalidArgument, "null buffer");
  // the root's recvbuff is exactly an AllGather's output (and NCCL's in-place
  // rule for Gather, sendbuff == recvbuff + root*count, is AllGather's);
  // elsewhere the gathered blocks land in scratch
  Call k{comm, flxCollAllGather, sendbuff, recvbuff, count, datatype, 0, stream};
  if (!is_root && count > 0) {
    FLX_CUDA(cudaSetDevice(comm->device));
    FLX_CUDA(cudaMallocAsync(&k.tmp, count * dtype_size(datatype) * comm->nranks, stream));
    k.recv = k.tmp;
  }
  return enqueue(k);
}

flxResult_t flxScatter(const void* sendbuff, void* recvbuff, size_t count,
                       flxDataType_t datatype, int root, flxComm_t comm, cudaStream_t stream) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(check_call(comm, datatype, 0, false));
  if (root < 0 || root >= comm->nranks) return fail(flxInvalidArgument, "bad root %d", root);
  const bool is_root = comm->rank == root;
  if (count > 0 && (!recvbuff || (is_root && !sendbuff)))
    return fail(flxInvalidArgument, "null buffer");
  if (count == 0) return flxSuccess;
  // an AllToAll in which only the root's blocks matter: block j of the root's
  // sendbuff reaches rank j's scratch block `root`, copied to recvbuff after
  const size_t block = count * dtype_size(datatype), all = block * comm->nranks;
  FLX_CUDA(cudaSetDevice(comm->device));
  Call k{comm, flxCollAllToAll, sendbuff, nullptr, count, datatype, 0, stream};
  FLX_CUDA(cudaMallocAsync(&k.tmp, all, stream));
  k.recv = k.tmp;
  if (!is_root) {  // this rank's outgoing blocks are never read by anyone
    const cudaError_t e = cudaMallocAsync(&k.tmp2, all, stream);
    if (e != cudaSuccess) {
      cudaFreeAsync(k.tmp, stream);
      return fail(flxUnhandledCudaError, "flxScatter scratch: %s", cudaGetErrorString(e));
    }
    k.send = k.tmp2;
  }
  k.post_dst = recvbuff;
  k.post_src = static_cast<const char*>(k.tmp) + (size_t)root * block;
  k.post_bytes = block;
  return enqueue(k);
}

flxResult_t flxBroadcast(const void* sendbuff, void* recvbuff, size_t count,
                         flxDataType_t datatype, int root, flxComm_t comm, cudaStream_t stream) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(check_call(comm, datatype, 0, false));
  if (root < 0 || root >= comm->nranks) return fail(flxInvalidArgument, "bad root %d", root);
  if (count == 0) return flxSuccess;
  if (!recvbuff || (comm->rank == root && !sendbuff))
    return fail(flxInvalidArgument, "null buffer");
  const size_t bytes = count * dtype_size(datatype);
  FLX_CUDA(cudaSetDevice(comm->device));
  // the root's bytes, zeros elsewhere; then MAX over uint8 leaves the root's
  if (comm->rank == root) {
    if (sendbuff != recvbuff)
      FLX_CUDA(cudaMemcpyAsync(recvbuff, sendbuff, bytes, cudaMemcpyDeviceToDevice, stream));
  } else {
    FLX_CUDA(cudaMemsetAsync(recvbuff, 0, bytes, stream));
  }
  return flxAllReduce(recvbuff, recvbuff, bytes, flxUint8, flxMax, comm, stream);
}

// One collective for ALL ranks of a single-process communicator set in one
// call: equivalent to flxGroupStart; per-rank flx<Coll>(...); flxGroupEnd, but
// one host crossing instead of n+2 (small messages are host-issue bound).
flxResult_t flxGroupCollective(flxCollOp_t coll, flxComm_t* comms, int n,
                               const void* const* sendbuffs, void* const* recvbuffs,
                               size_t count, flxDataType_t datatype, flxRedOp_t op,
                               cudaStream_t stream) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  if (!comms || n < 1 || !sendbuffs || !recvbuffs)
    return fail(flxInvalidArgument, "bad group arguments");
  if (coll < flxCollAllReduce || coll > flxCollAllToAll)
    return fail(flxInvalidArgument, "bad collective %d", (int)coll);
  const bool reduce = coll == flxCollAllReduce || coll == flxCollReduceScatter;
  for (int i = 0; i < n; ++i) {
    FLX_TRY(check_call(comms[i], datatype, reduce ? op : 0, reduce));
    if (count > 0 && (!sendbuffs[i] || !recvbuffs[i]))
      return fail(flxInvalidArgument, "null buffer for rank %d", i);
    if (coll == flxCollAllToAll && count > 0 && sendbuffs[i] == recvbuffs[i])
      return fail(flxInvalidArgument, "in-place AllToAll is not supported");
  }
  ++t_group_depth;
  for (int i = 0; i < n; ++i) {
    Call k{comms[i], (int)coll, sendbuffs[i], recvbuffs[i], count, datatype,
           reduce ? (int)op : 0, stream};
    if (k.op == FLX_OP_AVG) {  // the striped sum, then finish_avg
      k.op = flxSum;
      k.avg = true;
    }
    t_pending.push_back(k);
  }
  --t_group_depth;
  if (t_group_depth > 0) return flxSuccess;  // inside an outer group: flushed by its end
  return flush_group();
}

flxResult_t flxGroupStart(void) {
  ++t_group_depth;
  return flxSuccess;
}

flxResult_t flxGroupEnd(void) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  if (t_group_depth <= 0) return fail(flxInvalidUsage, "flxGroupEnd without flxGroupStart");
  if (--t_group_depth > 0) return flxSuccess;
  return flush_group();
}

flxResult_t flxSetShares(flxComm_t comm, flxCollOp_t op, int bucket, const int granules[3]) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  if (op < flxCollAllReduce || op > flxCollAllToAll)
    return fail(flxInvalidArgument, "bad collective op %d", (int)op);
  if (!granules) {  // unpin: the bucket (or every bucket) goes back to the balancer
    ShareTable& t = comm->shares[op];
    if (bucket == FLX_BUCKET_ALL) {
      t.fallback = Granules{{FLX_GRANULE_TOTAL, 0, 0}};
      t.fallback_pinned = false;
      t.entries.clear();
    } else {
      t.entries.erase({(int)op, bucket});
    }
    return flxSuccess;
  }
  Granules g{{granules[0], granules[1], granules[2]}};
  int sum = 0;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) {
    if (g[p] < 0) return fail(flxInvalidArgument, "negative share on path %d", p);
    sum += g[p];
  }
  if (sum != FLX_GRANULE_TOTAL)
    return fail(flxInvalidArgument, "shares sum to %d, expected %d", sum, FLX_GRANULE_TOTAL);
  const int mask = path_mask();
  for (int p = 1; p < FLX_NUM_PATHS; ++p)
    if (g[p] > 0 && !(mask & (1 << p)))
      return fail(flxInvalidArgument, "path %d is not available on this box", p);
  ShareTable& t = comm->shares[op];
  if (bucket == FLX_BUCKET_ALL) {
    t.fallback = g;
    t.fallback_pinned = true;  // the user fixed every bucket: no autotuning
    t.entries.clear();
  } else {
    if (bucket < -1 || bucket > 63) return fail(flxInvalidArgument, "bad bucket %d", bucket);
    t.entries[{(int)op, bucket}] = g;
  }
  return flxSuccess;
}

flxResult_t flxGetShares(flxComm_t comm, flxCollOp_t op, int bucket, int granules[3]) {
  FLX_TRY(validate_comm(comm));
  if (op < flxCollAllReduce || op > flxCollAllToAll)
    return fail(flxInvalidArgument, "bad collective op %d", (int)op);
  if (!granules) return fail(flxInvalidArgument, "null granules");
  const ShareTable& t = comm->shares[op];
  Granules g = t.fallback;
  auto it = t.entries.find({(int)op, bucket});
  if (bucket != FLX_BUCKET_ALL && it != t.entries.end())
    g = it->second;
  else if (bucket != FLX_BUCKET_ALL && !t.fallback_pinned)
    tuner_of(comm)->current(op, bucket, &g);  // the balancer's split, if it tuned this bucket
  for (int p = 0; p < FLX_NUM_PATHS; ++p) granules[p] = g[p];
  return flxSuccess;
}

flxResult_t flxGetPathTimes(flxComm_t comm, float ms[3]) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  if (!ms) return fail(flxInvalidArgument, "null ms");
  if (comm->world) {
    const uint64_t calls = world_calls(comm->world, comm->local);
    if (calls == 0) return fail(flxInvalidUsage, "no collective has run on this comm");
    return world_read_timing(comm->world, comm->local, calls - 1, ms);
  }
  Clique* c = comm->clique;
  if (c->calls == 0) return fail(flxInvalidUsage, "no collective has run on this comm");
  return read_timing(c, c->calls - 1, ms);
}

flxResult_t flxGetPathTimesHistory(flxComm_t comm, int max_calls, float* ms, int* n_out) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  if (!ms || !n_out || max_calls < 0) return fail(flxInvalidArgument, "bad history arguments");
  const uint64_t calls =
      comm->world ? world_calls(comm->world, comm->local) : comm->clique->calls;
  const uint64_t avail = std::min<uint64_t>(calls, Clique::kTimingSlots);
  const uint64_t n = std::min<uint64_t>(avail, (uint64_t)max_calls);
  for (uint64_t i = 0; i < n; ++i) {
    if (comm->world)
      FLX_TRY(world_read_timing(comm->world, comm->local, calls - n + i, ms + 3 * i));
    else
      FLX_TRY(read_timing(comm->clique, calls - n + i, ms + 3 * i));
  }
  *n_out = (int)n;
  return flxSuccess;
}

flxResult_t flxGetPathBytes(flxComm_t comm, size_t bytes[3]) {
  FLX_TRY(validate_comm(comm));
  if (!bytes) return fail(flxInvalidArgument, "null bytes");
  const auto last = comm->world ? world_last_bytes(comm->world, comm->local)
                                : comm->clique->last_bytes;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) bytes[p] = last[p];
  return flxSuccess;
}

flxResult_t flxGetAlignment(flxComm_t comm, flxCollOp_t op, size_t* alignment) {
  FLX_TRY(validate_comm(comm));
  if (!alignment) return fail(flxInvalidArgument, "null alignment");
  *alignment = alignment_for(comm, op);
  return flxSuccess;
}

flxResult_t flxSetTiming(flxComm_t comm, int enabled) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  comm->timing = enabled != 0;
  return flxSuccess;
}

flxResult_t flxSetNvlinkCtas(flxComm_t comm, int nctas) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  if (nctas < 0 || nctas > 65535) return fail(flxInvalidArgument, "bad nctas %d", nctas);
  if (comm->nvlink_ctas != nctas) tuner_of(comm)->reset();  // measured rates are void
  comm->nvlink_ctas = nctas;
  if (comm->world) world_set_nctas(comm->world, nctas);
  return flxSuccess;
}

flxResult_t flxSetStaging(flxComm_t comm, size_t chunk_bytes, int buffers) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  if (buffers != 1 && buffers != 2)
    return fail(flxInvalidArgument, "buffers must be 1 or 2 (staging.py:41-42)");
  if (chunk_bytes % 4096) return fail(flxInvalidArgument, "chunk_bytes must be a multiple of 4096");
  if (comm->chunk_bytes != chunk_bytes || comm->buffers != buffers) tuner_of(comm)->reset();
  comm->chunk_bytes = chunk_bytes;
  comm->buffers = buffers;
  return flxSuccess;
}

flxResult_t flxGetPathMask(flxComm_t comm, int* mask) {
  FLX_TRY(validate_comm(comm));
  if (!mask) return fail(flxInvalidArgument, "null mask");
  *mask = path_mask();
  return flxSuccess;
}

flxResult_t flxCommDebugPeer(flxComm_t comm, int peer, int host_region, int write, void* buf,
                             size_t bytes) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  if (!comm->world) return fail(flxInvalidUsage, "not a multi-rank communicator");
  if (!buf && bytes) return fail(flxInvalidArgument, "null buffer");
  return world_debug_peer(comm->world, comm->local, peer, host_region, write, buf, bytes);
}

flxResult_t flxCommGetNvls(flxComm_t comm, int* on, char* reason, size_t reason_len) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  if (!on) return fail(flxInvalidArgument, "null on");
  const char* why = "NVLS needs a multi-GPU world (one process per GPU, FLX_NVLS=1)";
  *on = 0;
  if (comm->world) why = world_nvls_status(comm->world, on);
  if (reason && reason_len) snprintf(reason, reason_len, "%s", why);
  return flxSuccess;
}

flxResult_t flxGetLaunchCount(unsigned long long* count) {
  if (!count) return fail(flxInvalidArgument, "null count");
  *count = g_launches.load();
  return flxSuccess;
}

}  // extern "C"

// ------------------------------------------------------ in-library balancer
extern "C" {

flxResult_t flxSetAutoTune(flxComm_t comm, int enabled) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  comm->autotune = enabled != 0;
  return flxSuccess;
}

flxResult_t flxSetTunerConfig(flxComm_t comm, const flxTunerConfig* s1,
                              const flxBalancerConfig* s2, size_t min_bytes) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  if (s1 && !tune::valid(*s1)) return fail(flxInvalidArgument, "bad tuner config");
  if (s2 && (!tune::valid(*s2) || s2->window > 32))
    return fail(flxInvalidArgument, "bad balancer config (window must be 1..32)");
  if (s1) comm->tune_s1 = *s1;
  if (s2) comm->tune_s2 = *s2;
  if (min_bytes) comm->tune_min_bytes = min_bytes;
  tuner_of(comm)->reset();
  return flxSuccess;
}

flxResult_t flxSetLinkProfile(flxComm_t comm, const flxLinkProfile* profile) {
  flx::CtxGuard ctx_guard;  // the caller's context is restored on return
  FLX_TRY(validate_comm(comm));
  if (profile && !(profile->bandwidth[flxPathNvlink] > 0))
    return fail(flxInvalidArgument, "the link profile needs a positive NVLink bandwidth");
  comm->have_profile = profile != nullptr;
  if (profile) comm->profile = *profile;
  tuner_of(comm)->reset();
  return flxSuccess;
}

flxResult_t flxGetTuneInfo(flxComm_t comm, flxCollOp_t op, int bucket, flxTuneInfo* info) {
  FLX_TRY(validate_comm(comm));
  if (!info || op < flxCollAllReduce || op > flxCollAllToAll)
    return fail(flxInvalidArgument, "bad arguments");
  tuner_of(comm)->info(op, bucket, info);
  return flxSuccess;
}

flxResult_t flxGetTuneTrace(flxComm_t comm, flxCollOp_t op, int bucket, flxTuneRecord* records,
                            int max_records, int* n) {
  FLX_TRY(validate_comm(comm));
  if (!n || max_records < 0 || (max_records && !records) || op < flxCollAllReduce ||
      op > flxCollAllToAll)
    return fail(flxInvalidArgument, "bad arguments");
  *n = tuner_of(comm)->trace(op, bucket, records, max_records);
  return flxSuccess;
}

flxResult_t flxGetTuneEvaluations(flxComm_t comm, flxCollOp_t op, int bucket,
                                  flxEvalRecord* records, int max_records, int* n) {
  FLX_TRY(validate_comm(comm));
  if (!n || max_records < 0 || (max_records && !records) || op < flxCollAllReduce ||
      op > flxCollAllToAll)
    return fail(flxInvalidArgument, "bad arguments");
  *n = tuner_of(comm)->evaluations(op, bucket, records, max_records);
  return flxSuccess;
}

}  // extern "C"
