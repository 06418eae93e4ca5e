// Multi-rank NVLink-path kernels: one launch per rank per call, CTA b of
// rank r exchanging with CTA b of every peer over NVSwitch through
// peer-mapped (CUDA IPC) scratch buffers and release/acquire flags.
//
// Two-shot AllReduce = reduce-scatter + all-gather in one launch, per round:
//   1 push   rank r stores its chunk c to peer c's inbox[r]           (NVLink write)
//   2 reduce rank r folds inbox[0..N) (own chunk read in place) in rank
//            order -> recv chunk r and its own outbox                  (local HBM)
//   3 pull   rank r loads every peer's outbox into recv chunk c         (NVLink read)
// Slot protocols (AllGather / ReduceScatter / AllToAll): push, wait, land or
// fold, free.  One-shot variants of all four (rank_oneshot) for small slices:
// push into the peers' double-buffered one-shot inboxes, one wait, finish locally.
// Flags (per receiving rank): arrive/free/ready/pulled[src][cta], monotone
// per-CTA epochs kept on the device (cta_epochs), compared cyclically; every
// CTA owns one fixed region of each slot (cta_sub).  The fold rule is
// kernels.cuh's (bit-identical to the virtual-rank path and the CPU oracle).
//
// Non-template kernels are `static` (this header is included by several
// translation units: world.cu and the per-dtype launch units rank_launch_*.cu).
// The same device code runs (a) per GPU with grid = nctas, (b) in loopback
// (all ranks on one GPU, grid = nctas x nranks, cooperative launch so every
// CTA is co-resident and the spin-waits cannot deadlock).
#pragma once

#include "kernels.cuh"

namespace flx {

constexpr int kMaxCtas = 64;  // also the number of regions per slot (cta_sub)

// Phase-timing hook for tools/rank_phases.cu (compiled out in the library).
#ifndef FLX_PHASE
#define FLX_PHASE(i)
#endif
// Flag kinds, each [src][cta] in the RECEIVING rank's block:
//   kArrive  src pushed its data into my inbox[src] for epoch e
//   kFree    src finished reading the inbox slot I pushed into (epoch e) —
//            set by EVERY protocol every round, so "kFree >= e-1" is a valid
//            reuse guard whatever collective ran before
//   kReady   (AllReduce) src's reduced outbox for epoch e is readable
//   kPulled  (AllReduce) src finished pulling my outbox of epoch e
enum FlagKind { kArrive = 0, kFree = 1, kReady = 2, kPulled = 3 };
constexpr int kFlagKinds = 4;
constexpr size_t kFlagWords = (size_t)kFlagKinds * kMaxRanks * kMaxCtas;
// Per-CTA epoch state, private to the rank, after the flag words:
//   [4*cta + 0] rounds run so far by CTA cta (round k of the next call uses
//               epoch state + 1 + k)
//   [4*cta + 1] epoch of the last two-shot AllReduce round (guards outbox
//               reuse through kPulled; 0: none)
//   [4*cta + 2] epoch of the last round that used the main inbox slots
//               (guards them through kFree; one-shot rounds do not touch them)
// Kept on the device and advanced by the kernel itself, so a launch carries
// no host-side epoch and can be captured into a CUDA graph and replayed.
// Every rank runs the same sequence of collectives with the same grid, so
// CTA b's state is identical on every rank; a CTA that sits out a call lags
// the same way everywhere.
constexpr size_t kStateWords = 4 * kMaxCtas;

struct RankArgs {
  const char* send;
  char* recv;
  char* scratch[kMaxRanks];    // every rank's scratch base, as mapped in this rank
  uint32_t* flags[kMaxRanks];  // every rank's flag block, as mapped in this rank
  int rank;
  int nranks;
  size_t bytes;        // NVLink slice: per-rank message bytes (AR) / send bytes (AG)
  size_t rank_stride;  // AllGather: distance between rank blocks in recv
  size_t slot;         // inbox slot capacity (bytes) per source rank
  size_t small_slot;   // one-shot inbox capacity per source rank and parity
  int oneshot;         // AllReduce: run the one-shot protocol (bytes fit small_slot)
  int ll;              // one-shot in the LL format (flag in every 64-bit word; rank_oneshot_ll)
  int bulk;            // copy phases as TMA bulk copies (cta_copy_bulk; FLX_BULK=0: off)
  uint32_t* abort_word;  // host-mapped; set on a wait timeout
  long long spin_limit;  // clock64 cycles a wait may spin before aborting (FLX_TIMEOUT_S)
};

// This CTA's epoch state (in its own rank's flag block).
struct CtaEpochs {
  uint32_t* state;
  uint32_t first;      // epoch of round 0 of this call
  uint32_t last_ar;    // epoch of the last two-shot AllReduce round before this call
  uint32_t last_main;  // epoch of the last main-slot round before this call
};

__device__ __forceinline__ CtaEpochs cta_epochs(const RankArgs& a, int cta) {
  __shared__ uint32_t s_st[3];
  uint32_t* st = a.flags[a.rank] + kFlagWords + 4 * (size_t)cta;
  if (threadIdx.x < 3) s_st[threadIdx.x] = st[threadIdx.x];
  __syncthreads();
  // Epoch 0 is never a call's first epoch: the LL packet area is zeroed at
  // init, so an LL round tagged 0 (after 2^32 rounds) would accept
  // never-written packets.  Skipping by 2 keeps the parity alternation the
  // one-shot regions rely on; every rank skips identically.
  uint32_t first = s_st[0] + 1;
  if (first == 0) first = 2;
  return CtaEpochs{st, first, s_st[1], s_st[2]};
}

// After the call's rounds (not reached when a wait aborted): `last_ar` /
// `last_main` are the values to carry forward.
__device__ __forceinline__ void cta_epochs_done(const CtaEpochs& ep, uint32_t rounds,
                                                uint32_t last_ar, uint32_t last_main) {
  if (threadIdx.x == 0 && rounds > 0) {
    ep.state[0] = ep.first - 1 + rounds;
    ep.state[1] = last_ar;
    ep.state[2] = last_main;
  }
}

struct LoopbackArgs {
  RankArgs r[kMaxRanks];
};

__device__ __forceinline__ uint32_t* flag_at(uint32_t* block, int kind, int src, int cta) {
  return block + ((size_t)kind * kMaxRanks + src) * kMaxCtas + cta;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Inter-rank data written during the kernel: bypass L1 (.cg) so a later round
// never sees a stale line.
__device__ __forceinline__ uint4 ld_cg(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Publish this CTA's prior global stores: bar.sync orders every thread's
// stores before the flag stores, and st.release.sys is cumulative, so a rank
// that acquires a flag sees all of them.  Lane i of warp 0 signals peer
// (r+1+i) mod n in its flag block, slot [kind][r][cta] — the N-1 peers in
// parallel; with kind2 >= 0, lanes 16.. signal kind2 the same way.  The
// target address is computed per lane: no per-peer pointer array (which
// would live in local memory).
__device__ __forceinline__ void cta_signal_peers(const RankArgs& a, int cta, int kind,
                                                 uint32_t epoch, int kind2 = -1) {
  __syncthreads();
  const int lane = threadIdx.x;
  const int i = lane & 15;
  const int k = lane < 16 ? kind : kind2;
  if (lane < 32 && k >= 0 && i < a.nranks - 1) {
    const int c = (a.rank + 1 + i) % a.nranks;
    st_release_sys(flag_at(a.flags[c], k, a.rank, cta), epoch);
  }
}

// Flags are compared cyclically ((int)(flag - epoch) >= 0) so epochs may wrap;
// a spin limit (FLX_TIMEOUT_S, default 600 s) sets the host-mapped abort word
// instead of hanging the GPU
// when a peer died.
// Warp 0 waits, one flag per lane, until every peer p != skip has published:
// lanes 0..15 watch flag(kind1, p) >= e1, lanes 16..31 flag(kind2, p) >= e2
// (kind2 < 0: unused).  One parallel poll instead of N-1 sequential ones.
__device__ __forceinline__ bool cta_wait_peers(uint32_t* block, int n, int skip, int cta,
                                               int kind1, uint32_t e1, int kind2, uint32_t e2,
                                               const RankArgs& a) {
  __shared__ int ok;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int src = lane & 15;
    const int kind = lane < 16 ? kind1 : kind2;
    const uint32_t e = lane < 16 ? e1 : e2;
    const bool active = src < n && src != skip && kind >= 0;
    const uint32_t* f = active ? flag_at(block, kind, src, cta) : nullptr;
    const long long t0 = clock64();
    uint32_t spins = 0;
    int good = 1;
    while (true) {
      const bool ready = !active || (int)(ld_acquire_sys(f) - e) >= 0;
      if (__all_sync(0xffffffffu, ready)) break;
      if ((++spins & 4095) == 0) {  // the abort word is host memory: poll it rarely
        int bad = 0;
        if (lane == 0) bad = *(volatile uint32_t*)a.abort_word || clock64() - t0 > a.spin_limit;
        if (__shfl_sync(0xffffffffu, bad, 0)) {
          if (lane == 0) atomicExch(a.abort_word, 1u);
          good = 0;
          break;
        }
      }
    }
    if (lane == 0) ok = good;
  }
  __syncthreads();
  return ok;
}

__device__ __forceinline__ bool aligned16_dev(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

// CTA-wide copy of n bytes (vectorised when both ends are 16 B aligned).
// kCopyUnroll 16 B loads per thread are in flight before the stores: a remote
// (NVLink) load costs ~2 us, so 512 threads x 8 x 16 B = 64 KB per CTA in
// flight is what sustains ~30 GB/s per CTA on the pull phase.
constexpr int kCopyUnroll = 4;

__device__ __forceinline__ void cta_copy(char* dst, const char* src, size_t n, bool coherent) {
  if (aligned16_dev(dst) && aligned16_dev(src)) {
    const size_t nv = n >> 4;
    const size_t step = blockDim.x;
    size_t v = threadIdx.x;
    for (; v + (kCopyUnroll - 1) * step < nv; v += kCopyUnroll * step) {
      uint4 w[kCopyUnroll];
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u) {
        const char* p = src + ((v + u * step) << 4);
        w[u] = coherent ? ld_cg(p) : ld_stream(p);
      }
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u)
        *reinterpret_cast<uint4*>(dst + ((v + u * step) << 4)) = w[u];
    }
    for (; v < nv; v += step) {
      const uint4 w = coherent ? ld_cg(src + (v << 4)) : ld_stream(src + (v << 4));
      *reinterpret_cast<uint4*>(dst + (v << 4)) = w;
    }
    for (size_t i = (nv << 4) + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  } else if (aligned16_dev(src)) {
    // aligned source, misaligned destination (AllGather / AllToAll blocks of
    // a ragged per-rank count): aligned 16 B stores of funnel-shifted source
    // vectors (kernels.cuh shift_bytes), bytewise head and tail only
    const size_t h = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
    const size_t body = n > h ? (n - h) >> 4 : 0;
    for (size_t j = threadIdx.x; j < body; j += blockDim.x) {
      const uint4 x = coherent ? ld_cg(src + (j << 4)) : ld_stream(src + (j << 4));
      // the last window's second vector may reach past the piece: clamp it
      const uint4 y = ld_vec_clamped(src + ((j + 1) << 4), n - ((j + 1) << 4), coherent);
      *reinterpret_cast<uint4*>(dst + h + (j << 4)) = shift_bytes(x, y, (uint32_t)h);
    }
    const size_t nh = n < h ? n : h, tail0 = h + (body << 4);
    for (size_t t = threadIdx.x; t < nh + (n - min(n, tail0)); t += blockDim.x) {
      const size_t i = t < nh ? t : tail0 + (t - nh);
      dst[i] = coherent ? *(volatile const char*)(src + i) : src[i];
    }
  } else {
    for (size_t i = threadIdx.x; i < n; i += blockDim.x)
      dst[i] = coherent ? *(volatile const char*)(src + i) : src[i];
  }
}

// A copy segment of a multi-peer phase: dst <- src, len bytes.
struct CopySeg {
  char* dst;
  const char* src;
  size_t len;
};

// Bulk-copy (TMA) form of a whole push / pull / land phase (RankArgs::bulk,
// the default; FLX_BULK=0 selects the register copies of cta_copy): the N-1
// segments stream as one pipeline of kBulkTile tiles through a ring of
// kBulkStages shared-memory stages — cp.async.bulk global -> smem behind an
// mbarrier (complete_tx), then cp.async.bulk smem -> global — driven by one
// thread, so the bytes in flight ((kBulkStages-1) tiles of loads + one store,
// ~80 KB per CTA) sit in dynamic shared memory instead of registers.  The 16 B
// aligned body of every segment goes through the pipeline while the other
// threads copy the ragged tails.  Proxy fences order the flag acquires
// (generic proxy) before the bulk reads and the bulk writes before the CTA's
// flag release.  Loopback A/B (profiles/r2/loopback_bulk_copy_ab.jsonl): 16 KB
// x 6 stages beats the register copies by 4-9 % (fp32, N = 8/4/2); rings that
// fit the 48 KB static limit (8 KB x 5, 4 KB x 10, 16 KB x 2) lose.
#ifndef FLX_BULK_TILE
#define FLX_BULK_TILE 16384
#endif
#ifndef FLX_BULK_STAGES
#define FLX_BULK_STAGES 6
#endif
constexpr uint32_t kBulkTile = FLX_BULK_TILE;
constexpr int kBulkStages = FLX_BULK_STAGES;

__device__ __forceinline__ void fence_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

struct BulkSmem {
  __align__(128) unsigned char buf[kBulkStages][kBulkTile];
  uint64_t full[kBulkStages];
  char* dst[kBulkStages];
  uint32_t len[kBulkStages];
};
// one dynamic allocation per kernel, shared by every phase's instantiation
__device__ __forceinline__ BulkSmem& bulk_smem() {
  extern __shared__ __align__(128) unsigned char flx_bulk_dyn[];
  return *reinterpret_cast<BulkSmem*>(flx_bulk_dyn);
}

template <typename SegFn>
__device__ void cta_copy_bulk(SegFn seg, int nseg, bool coherent) {
  bool ok = true;
  for (int i = 0; i < nseg; ++i) {
    const CopySeg g = seg(i);
    ok = ok && aligned16_dev(g.dst) && aligned16_dev(g.src);
  }
  if (!ok) {
    for (int i = 0; i < nseg; ++i) {
      const CopySeg g = seg(i);
      cta_copy(g.dst, g.src, g.len, coherent);
    }
    return;
  }
  BulkSmem& sm = bulk_smem();
  auto& buf = sm.buf;
  auto& full = sm.full;
  auto& sdst = sm.dst;
  auto& slen = sm.len;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBulkStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_global();
    int ps = 0;      // producer cursor: segment, byte offset in its body
    size_t po = 0;
    auto produce = [&](int stage) -> bool {
      for (; ps < nseg; ++ps, po = 0) {
        const CopySeg g = seg(ps);
        const size_t body = g.len & ~(size_t)15;
        if (po < body) {
          const uint32_t len = (uint32_t)min((size_t)kBulkTile, body - po);
          mbar_expect_tx(&full[stage], len);
          bulk_load(buf[stage], g.src + po, len, &full[stage]);
          sdst[stage] = g.dst + po;
          slen[stage] = len;
          po += len;
          return true;
        }
      }
      return false;
    };
    uint32_t issued = 0;
    while (issued < (uint32_t)kBulkStages && produce((int)issued)) ++issued;
    for (uint32_t t = 0; t < issued; ++t) {
      const int s = (int)(t % kBulkStages);
      mbar_wait(&full[s], (t / kBulkStages) & 1);
      bulk_store(sdst[s], buf[s], slen[s]);
      bulk_commit();
      if (t >= 1) {  // the previous tile's store has read its stage: refill it
        bulk_wait_read<1>();
        if (produce((int)((t - 1) % kBulkStages))) ++issued;
      }
    }
    bulk_wait_all();
    fence_async_global();
    for (int s = 0; s < kBulkStages; ++s)
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
  }
  for (int i = 0; i < nseg; ++i) {  // ragged tails (< 16 B per segment)
    const CopySeg g = seg(i);
    for (size_t j = (g.len & ~(size_t)15) + threadIdx.x; j < g.len; j += blockDim.x)
      g.dst[j] = coherent ? *(volatile const char*)(g.src + j) : g.src[j];
  }
  __syncthreads();
}
constexpr size_t kRankDynSmem = sizeof(BulkSmem);  // dynamic smem of launches with a.bulk

// vectors per thread per source in the fold: 4 for 32/64-bit types; 2 for
// 16-bit ones, whose fp32 accumulators are twice as many per vector (keeps the
// kernels inside 64 registers, 2 CTAs per SM)
template <typename T>
constexpr int fold_unroll() { return sizeof(T) >= 4 ? 4 : 2; }

// CTA-wide fold of n bytes: src(0..nsrc) -> dst0 (and dst1 when non-null),
// fold rule of kernels.cuh.  `src(p)` returns source p's pointer; it is
// evaluated per use (a select and a multiply-add), so no per-source pointer
// array is kept — arrays indexed by a runtime rank live in local memory.
template <typename T, int OP, typename Src>
__device__ __forceinline__ void cta_fold(char* dst0, char* dst1, Src src, int nsrc, size_t n) {
  using A = typename AccT<T>::type;
  constexpr int kVec = 16 / sizeof(T);
  constexpr int kFoldUnroll = fold_unroll<T>();
  bool vec = aligned16_dev(dst0) && (!dst1 || aligned16_dev(dst1));
  for (int i = 0; i < nsrc; ++i) vec = vec && aligned16_dev(src(i));
  size_t done = 0;
  if (vec) {
    const size_t nv = n >> 4;
    const size_t step = blockDim.x;
    size_t v = threadIdx.x;
    // kFoldUnroll vectors per thread per source: with few sources (n = 2) one
    // vector per source left ~2 loads in flight per thread and the fold phase
    // latency-bound (bf16, whose unpack/repack lengthens each iteration, ran
    // 0.77x fp32).  Same rank order per element, so the result is unchanged.
    // 16-bit types with more than 4 sources keep one vector per source (the
    // unrolled body measured 0.94x there: 8 x 4 fp32 accumulators spill).
    const bool unrolled = sizeof(T) >= 4 || nsrc <= 4;
    for (; unrolled && v + (kFoldUnroll - 1) * step < nv; v += kFoldUnroll * step) {
      A acc[kFoldUnroll][kVec];
      uint4 w[kFoldUnroll];
      {
        const char* s0 = src(0);
#pragma unroll
        for (int u = 0; u < kFoldUnroll; ++u) w[u] = ld_cg(s0 + ((v + u * step) << 4));
      }
#pragma unroll
      for (int u = 0; u < kFoldUnroll; ++u) load_acc<T>(acc[u], w[u]);
      for (int i = 1; i < nsrc; ++i) {
        const char* si = src(i);
#pragma unroll
        for (int u = 0; u < kFoldUnroll; ++u) w[u] = ld_cg(si + ((v + u * step) << 4));
#pragma unroll
        for (int u = 0; u < kFoldUnroll; ++u) fold_into<T, OP>(acc[u], w[u]);
      }
#pragma unroll
      for (int u = 0; u < kFoldUnroll; ++u) {
        const uint4 out = pack_acc<T>(acc[u]);
        *reinterpret_cast<uint4*>(dst0 + ((v + u * step) << 4)) = out;
        if (dst1) *reinterpret_cast<uint4*>(dst1 + ((v + u * step) << 4)) = out;
      }
    }
    for (; v < nv; v += step) {  // one vector per thread, sources streamed in order
      A acc[kVec];
      load_acc<T>(acc, ld_cg(src(0) + (v << 4)));
      for (int i = 1; i < nsrc; ++i) fold_into<T, OP>(acc, ld_cg(src(i) + (v << 4)));
      const uint4 out = pack_acc<T>(acc);
      *reinterpret_cast<uint4*>(dst0 + (v << 4)) = out;
      if (dst1) *reinterpret_cast<uint4*>(dst1 + (v << 4)) = out;
    }
    done = nv << 4;
  }
  for (size_t i = done / sizeof(T) + threadIdx.x; i < n / sizeof(T); i += blockDim.x) {
    A acc = to_acc<T>(*(volatile const T*)(src(0) + i * sizeof(T)));
    for (int s = 1; s < nsrc; ++s)
      acc = apply_op<OP>(acc, to_acc<T>(*(volatile const T*)(src(s) + i * sizeof(T))));
    const T out = from_acc<T>(acc);
    *reinterpret_cast<T*>(dst0 + i * sizeof(T)) = out;
    if (dst1) *reinterpret_cast<T*>(dst1 + i * sizeof(T)) = out;
  }
}

__device__ __forceinline__ size_t ceil16(size_t x) { return (x + 15) & ~(size_t)15; }

// [lo, hi) of CTA `cta`'s part of a span of `len` bytes split over `nctas`.
__device__ __forceinline__ void cta_part(size_t len, int nctas, int cta, size_t* lo, size_t* hi) {
  const size_t part = ceil16((len + nctas - 1) / nctas);
  *lo = min(len, (size_t)cta * part);
  *hi = min(len, *lo + part);
}

// CTA cta owns the same region [cta*sub, cta*sub + sub) of every inbox slot
// and of the outbox, sub = slot / kMaxCtas, in every round of every protocol:
// it depends neither on the message length nor on the grid size, so the
// per-CTA flags guard exactly the bytes that CTA pair writes and reads (with
// length- or grid-dependent offsets, CTA b could overwrite bytes a slower
// peer CTA b' is still reading from an earlier round).  The round capacity is
// sub * nctas per slot, which keeps every CTA part <= sub.
__device__ __forceinline__ size_t cta_sub(size_t slot) {
  return (slot / (size_t)kMaxCtas) & ~(size_t)15;
}

// Every protocol: wait until peer c freed the inbox slot I push into
// (kFree >= e-1), push, announce (kArrive = e); the receiver consumes its
// inbox and answers kFree = e.

// Two-shot rounds.  CTA b owns part b of every rank's chunk for the WHOLE call
// (chunk c = [c*chunk, (c+1)*chunk) of the message, reduced by rank c) and
// walks it in rounds of `round` bytes per chunk part, each round a complete
// push -> fold -> pull with its own epoch.  Large messages take several
// rounds, and odd CTAs start with a half-length round: their phases then run
// half a round out of step with the even CTAs', so while one half of the CTAs
// folds (local HBM only) the other half keeps NVLink busy pushing or pulling —
// the link no longer idles for the whole fold phase.  Every rank derives the
// same schedule for CTA b from (bytes, n, nctas, b), so CTA b's rounds and
// epochs agree across ranks; per-CTA epochs let CTAs run different counts.
constexpr size_t kRoundMin = 128 << 10;  // shortest full round per chunk part
#ifndef FLX_ROUNDS_PER_CALL
#define FLX_ROUNDS_PER_CALL 4  // tools/rank_timeline.cu compares 1 (round-1 schedule)
#endif
constexpr size_t kRoundsPerCall = FLX_ROUNDS_PER_CALL;  // target rounds for large messages

template <typename T, int OP>
__device__ void rank_allreduce(const RankArgs& a, int cta, int nctas) {
  const int r = a.rank, n = a.nranks;
  const size_t sub = cta_sub(a.slot);
  const size_t mine = (size_t)cta * sub;  // this CTA's region in every slot
  const size_t outbox = a.slot * n;       // outbox follows the n inbox slots
  const size_t chunk = ceil16((a.bytes + n - 1) / n);
  const size_t maxpart = ceil16((chunk + nctas - 1) / nctas);  // a full chunk's part
  // a round is at most one region (sub <= slot / 64), so it fits 32 bits
  const uint32_t round = (uint32_t)min(sub, max(kRoundMin, ceil16((maxpart + kRoundsPerCall - 1) /
                                                                kRoundsPerCall)));
#ifndef FLX_STAGGER
#define FLX_STAGGER 1  // tools/rank_timeline.cu builds both ways to compare
#endif
  const bool stagger = FLX_STAGGER && (cta & 1) && maxpart >= 2 * kRoundMin;
  FLX_PHASE(0);
  const CtaEpochs ep = cta_epochs(a, cta);
  uint32_t prev_outbox = ep.last_ar, prev_main = ep.last_main;
  uint32_t k = 0;
  for (size_t at = 0; at < maxpart; ++k) {
    const uint32_t e = ep.first + k;
    const uint32_t len =
        (uint32_t)min(maxpart - at, (size_t)((k == 0 && stagger) ? ((round / 2 + 15) & ~15u) : round));
    // this round's piece of CTA b's part of rank c's chunk, as a message
    // offset and length — recomputed per use instead of kept in per-peer
    // arrays (which would live in local memory)
    // (full chunks share `maxpart`; only the ragged last chunk divides again)
    auto piece = [&](int c) {
      const size_t off = min(a.bytes, (size_t)c * chunk);
      const size_t clen = min(a.bytes - off, chunk);
      const size_t p = clen == chunk ? maxpart : ceil16((clen + nctas - 1) / nctas);
      const size_t b0 = (size_t)cta * p;
      const size_t lo = min(clen, b0 + at), hi = min(min(clen, b0 + p), lo + len);
      return make_ulonglong2(off + lo, hi - lo);  // {message offset, bytes}
    };
    // 1) push my chunk c into peer c's inbox slot r (this CTA's region)
    if (!cta_wait_peers(a.flags[r], n, r, cta, kFree, prev_main, -1, 0, a)) return;
    FLX_PHASE(1);
    if (a.bulk) {
      cta_copy_bulk([&](int i) {
        const int c = (r + 1 + i) % n;
        const ulonglong2 pc = piece(c);
        return CopySeg{a.scratch[c] + (size_t)r * a.slot + mine, a.send + pc.x, pc.y};
      }, n - 1, false);
    } else {
      for (int s = 1; s < n; ++s) {
        const int c = (r + s) % n;
        const ulonglong2 pc = piece(c);
        cta_copy(a.scratch[c] + (size_t)r * a.slot + mine, a.send + pc.x, pc.y, false);
      }
    }
    cta_signal_peers(a, cta, kArrive, e);
    FLX_PHASE(2);
    // 2) every push landed, and every peer pulled my previous outbox
    if (!cta_wait_peers(a.flags[r], n, r, cta, kArrive, e, kPulled, prev_outbox, a)) return;
    FLX_PHASE(3);
    {
      const ulonglong2 pr = piece(r);
      const char* own = a.send + pr.x;
      const char* inbox = a.scratch[r] + mine;
      const size_t slot = a.slot;
      cta_fold<T, OP>(a.recv + pr.x, a.scratch[r] + outbox + mine,
                      [=](int p) { return p == r ? own : inbox + (size_t)p * slot; }, n, pr.y);
    }
    // inbox slots consumed (kFree) and outbox readable (kReady), to every peer
    cta_signal_peers(a, cta, kFree, e, kReady);
    FLX_PHASE(4);
    // 3) pull every peer's reduced chunk
    if (!cta_wait_peers(a.flags[r], n, r, cta, kReady, e, -1, 0, a)) return;
    FLX_PHASE(5);
    if (a.bulk) {
      cta_copy_bulk([&](int i) {
        const int c = (r + 1 + i) % n;
        const ulonglong2 pc = piece(c);
        return CopySeg{a.recv + pc.x, a.scratch[c] + outbox + mine, pc.y};
      }, n - 1, true);
    } else {
      for (int s = 1; s < n; ++s) {
        const int c = (r + s) % n;
        const ulonglong2 pc = piece(c);
        cta_copy(a.recv + pc.x, a.scratch[c] + outbox + mine, pc.y, true);
      }
    }
    cta_signal_peers(a, cta, kPulled, e);
    FLX_PHASE(6);
    prev_outbox = prev_main = e;
    at += len;
  }
  cta_epochs_done(ep, k, prev_outbox, prev_main);
}

// One-shot protocols for small slices (RankArgs::oneshot): one release and one
// wait per call.  Every rank pushes its pieces into the peers' small inboxes
// (parity e & 1, slot = source rank, this CTA's region), signals kArrive(e),
// waits for every peer's kArrive(e), then finishes locally:
//   KIND 0 AllReduce      push my part of the whole message to every peer,
//                         fold the n copies in rank order into recv
//   KIND 1 AllGather      push my slice to every peer, land each peer's slice
//                         in its recv block
//   KIND 2 ReduceScatter  push block c to peer c, fold my block's n copies
//   KIND 3 AllToAll       push block c to peer c, land peer p's block in recv
//                         block p
// The two-shot AllReduce spends three signal hops and the slot protocols two
// (kArrive, then kFree); a signal costs ~1.5-2 us (tools/rank_phases.cu).
// Reuse of the parity region needs no flag: its last readers ran round e-2,
// and in round e-1 this CTA awaited every peer's kArrive(e-1), which that peer
// signalled after finishing round e-2 (every protocol awaits kArrive from
// every peer every round).  The main slots are untouched, so last_main stays.
template <typename T, int OP, int KIND>
__device__ void rank_oneshot_ll(const RankArgs& a, int cta, int nctas);

template <typename T, int OP, int KIND>
__device__ void rank_oneshot(const RankArgs& a, int cta, int nctas) {
  if (a.ll) {
    rank_oneshot_ll<T, OP, KIND>(a, cta, nctas);
    return;
  }
  FLX_PHASE(0);
  const int r = a.rank, n = a.nranks;
  const CtaEpochs ep = cta_epochs(a, cta);
  const uint32_t e = ep.first;
  const size_t mine = (size_t)cta * cta_sub(a.small_slot);
  const size_t region = a.slot * (n + 1) + (size_t)(e & 1) * n * a.small_slot;
  const size_t stride = a.rank_stride;
  size_t lo, hi;
  cta_part(a.bytes, nctas, cta, &lo, &hi);
  auto inbox = [&](int holder, int src) {
    return a.scratch[holder] + region + (size_t)src * a.small_slot + mine;
  };
  FLX_PHASE(1);
  {
    for (int s = 1; s < n; ++s) {
      const int c = (r + s) % n;
      const char* piece = (KIND == 0 || KIND == 1) ? a.send + lo : a.send + (size_t)c * stride + lo;
      cta_copy(inbox(c, r), piece, hi - lo, false);
    }
    if (KIND == 1) {
      char* own = a.recv + (size_t)r * stride + lo;
      if (own != a.send + lo) cta_copy(own, a.send + lo, hi - lo, false);
    } else if (KIND == 3) {
      cta_copy(a.recv + (size_t)r * stride + lo, a.send + (size_t)r * stride + lo, hi - lo, false);
    }
    cta_signal_peers(a, cta, kArrive, e);
  }
  FLX_PHASE(2);
  if (!cta_wait_peers(a.flags[r], n, r, cta, kArrive, e, -1, 0, a)) return;
  FLX_PHASE(3);
  if (KIND == 0 || KIND == 2) {
    const char* own = KIND == 0 ? a.send + lo : a.send + (size_t)r * stride + lo;
    const char* box = a.scratch[r] + region + mine;
    const size_t ss = a.small_slot;
    cta_fold<T, OP>(a.recv + lo, nullptr,
                    [=](int p) { return p == r ? own : box + (size_t)p * ss; }, n, hi - lo);
  } else {
    for (int s = 1; s < n; ++s) {
      const int p = (r - s + n) % n;
      cta_copy(a.recv + (size_t)p * stride + lo, inbox(r, p), hi - lo, true);
    }
  }
  FLX_PHASE(4);
  cta_epochs_done(ep, 1, ep.last_ar, ep.last_main);
}

// ---- LL one-shot: the epoch travels inside every 64-bit word of the data ----
//
// The one-shot above pays two sys-scope operations per call: the release
// signal after the push (a fence that drains every outstanding store, ~1.5-2
// us, tools/flag_pingpong.cu) and the acquire wait.  For slices whose CTA part
// fits kLLRegion / 2, the push instead stores 32-byte packets: 16 B of data as
// four 64-bit words {data32 | epoch << 32}, written with plain (volatile)
// 64-bit-element vector stores.  Each 64-bit element is single-copy atomic, so
// a reader that sees the epoch in a word's high half sees that word's data:
// no fence, no flag, the receiver polls the packets themselves (NCCL's LL
// protocol, with 64-bit elements so the PTX model guarantees it).
//
// The packets live in their own area after the one-shot inboxes,
// [2 parities][N sources][kMaxCtas regions of kLLRegion], zeroed at init and
// only ever written with LL packets, so a stale word carries an older epoch
// (epochs start at 1 and are unique per CTA) and is never mistaken for the
// current one.  Parity reuse: round e overwrites what peer CTA b read in
// round e-2; in round e-1 this CTA received every peer's packets (an empty
// part still sends one packet), which that peer wrote in a later kernel than
// its round e-2 reads.  Every rank computes the same parts (same bytes, same
// grid), so sender and receiver agree on the packet count.
constexpr size_t kLLRegion = 32768;  // packet bytes per (parity, source, CTA): 16 KiB of data
constexpr size_t kLLSlot = kLLRegion * kMaxCtas;

__device__ __forceinline__ void st_ll(char* p, const uint4& d, uint32_t e) {
  const uint64_t f = (uint64_t)e << 32;
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(f | d.x), "l"(f | d.y)
               : "memory");
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p + 16), "l"(f | d.z),
               "l"(f | d.w)
               : "memory");
}

// Poll one packet until its four words carry epoch e (false: timed out or
// another wait aborted; the abort word is host memory, polled rarely).
__device__ __forceinline__ bool ld_ll(const char* p, uint32_t e, uint4* out, const RankArgs& a,
                                      long long t0) {
  uint32_t spins = 0;
  while (true) {
    uint64_t w0, w1, w2, w3;
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];"
                 : "=l"(w2), "=l"(w3)
                 : "l"(p + 16)
                 : "memory");
    if ((uint32_t)(w0 >> 32) == e && (uint32_t)(w1 >> 32) == e && (uint32_t)(w2 >> 32) == e &&
        (uint32_t)(w3 >> 32) == e) {
      *out = make_uint4((uint32_t)w0, (uint32_t)w1, (uint32_t)w2, (uint32_t)w3);
      return true;
    }
    if ((++spins & 4095) == 0 &&
        (*(volatile uint32_t*)a.abort_word || clock64() - t0 > a.spin_limit)) {
      atomicExch(a.abort_word, 1u);
      return false;
    }
  }
}

// m (<= 16) bytes of user memory at any alignment, zero-padded to 16.  The
// word of byte i is picked with selects, not an indexed array (a runtime index
// into a register array would put the vector in local memory).
__device__ __forceinline__ uint4 ld_user(const char* p, size_t m) {
  if (m == 16 && aligned16_dev(p)) return *reinterpret_cast<const uint4*>(p);
  uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
  for (size_t i = 0; i < m; ++i) {
    const uint32_t b = (uint32_t)(uint8_t)p[i] << (8 * (i & 3));
    const size_t k = i >> 2;
    w0 |= k == 0 ? b : 0u;
    w1 |= k == 1 ? b : 0u;
    w2 |= k == 2 ? b : 0u;
    w3 |= k == 3 ? b : 0u;
  }
  return make_uint4(w0, w1, w2, w3);
}

__device__ __forceinline__ void st_user(char* p, const uint4& v, size_t m) {
  if (m == 16 && aligned16_dev(p)) {
    *reinterpret_cast<uint4*>(p) = v;
    return;
  }
  for (size_t i = 0; i < m; ++i) {
    const size_t k = i >> 2;
    const uint32_t w = k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
    p[i] = (char)(w >> (8 * (i & 3)));
  }
}

template <typename T, int OP, int KIND>
__device__ void rank_oneshot_ll(const RankArgs& a, int cta, int nctas) {
  using A = typename AccT<T>::type;
  constexpr int kVec = 16 / sizeof(T);
  FLX_PHASE(0);
  const int r = a.rank, n = a.nranks;
  const CtaEpochs ep = cta_epochs(a, cta);
  const uint32_t e = ep.first;
  const size_t area = a.slot * (n + 1) + 2 * (size_t)n * a.small_slot +
                      (size_t)(e & 1) * n * kLLSlot + (size_t)cta * kLLRegion;
  const size_t stride = a.rank_stride;
  size_t lo, hi;
  cta_part(a.bytes, nctas, cta, &lo, &hi);
  const size_t len = hi - lo;
  const size_t nvec = (len + 15) >> 4;
  const size_t npk = nvec ? nvec : 1;  // an empty part still proves progress with one packet
  auto inbox = [&](int holder, int src) {
    return a.scratch[holder] + area + (size_t)src * kLLSlot;
  };
  auto valid = [&](size_t v) { return v < nvec ? min((size_t)16, len - 16 * v) : (size_t)0; };
  FLX_PHASE(1);
  for (int s = 1; s < n; ++s) {
    const int c = (r + s) % n;
    const char* piece = (KIND == 0 || KIND == 1) ? a.send + lo : a.send + (size_t)c * stride + lo;
    char* dst = inbox(c, r);
    for (size_t v = threadIdx.x; v < npk; v += blockDim.x)
      st_ll(dst + 32 * v, ld_user(piece + 16 * v, valid(v)), e);
  }
  if (KIND == 1) {
    char* own = a.recv + (size_t)r * stride + lo;
    if (own != a.send + lo) cta_copy(own, a.send + lo, len, false);
  } else if (KIND == 3) {
    cta_copy(a.recv + (size_t)r * stride + lo, a.send + (size_t)r * stride + lo, len, false);
  }
  FLX_PHASE(2);
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  const long long t0 = clock64();
  bool ok = true;
  if (KIND == 0 || KIND == 2) {
    const char* own = KIND == 0 ? a.send + lo : a.send + (size_t)r * stride + lo;
    for (size_t v = threadIdx.x; ok && v < npk; v += blockDim.x) {
      const size_t m = valid(v);
      A acc[kVec];
      for (int p = 0; p < n; ++p) {  // the fixed rank-order fold (kernels.cuh rule)
        uint4 w;
        if (p == r) w = ld_user(own + 16 * v, m);
        else if (!(ok = ld_ll(inbox(r, p) + 32 * v, e, &w, a, t0))) break;
        if (p == 0) load_acc<T>(acc, w);
        else fold_into<T, OP>(acc, w);
      }
      if (ok && m) st_user(a.recv + lo + 16 * v, pack_acc<T>(acc), m);
    }
  } else {
    for (int s = 1; ok && s < n; ++s) {
      const int p = (r - s + n) % n;
      for (size_t v = threadIdx.x; v < npk; v += blockDim.x) {
        uint4 w;
        if (!(ok = ld_ll(inbox(r, p) + 32 * v, e, &w, a, t0))) break;
        const size_t m = valid(v);
        if (m) st_user(a.recv + (size_t)p * stride + lo + 16 * v, w, m);
      }
    }
  }
  if (!ok) bad = 1;
  __syncthreads();
  FLX_PHASE(3);
  if (!bad) cta_epochs_done(ep, 1, ep.last_ar, ep.last_main);
}

// After consuming my inbox slots for epoch e: tell every source (kFree = e).
__device__ __forceinline__ void free_all(const RankArgs& a, int cta, uint32_t e) {
  cta_signal_peers(a, cta, kFree, e);
}

// Staggered-round schedule of CTA `cta` over a span of `span` bytes shared by
// `nctas` CTAs (rank_allreduce's scheme for the slot protocols): the CTA owns
// [lo, lo + plen) of the span for the whole call and walks it in rounds of up
// to one region, ~kRoundsPerCall of them, odd CTAs starting with a half round
// so their land / fold phases overlap the even CTAs' pushes.  Every rank
// computes the same plan for CTA b, and every CTA loops to the full part
// length `maxpart` (empty pieces included), so rounds and epochs agree.
struct RoundPlan {
  size_t lo, plen, maxpart;
  uint32_t round;
  bool stagger;
  __device__ __forceinline__ uint32_t len(size_t at, uint32_t k) const {
    const uint32_t want = (k == 0 && stagger) ? ((round / 2 + 15) & ~15u) : round;
    return (uint32_t)min(maxpart - at, (size_t)want);
  }
  // this round's piece of the CTA's part: {offset in the span, bytes}
  __device__ __forceinline__ ulonglong2 piece(size_t at, uint32_t len) const {
    const size_t a0 = min(plen, at), a1 = min(plen, at + len);
    return make_ulonglong2(lo + a0, a1 - a0);
  }
};

__device__ __forceinline__ RoundPlan round_plan(size_t span, int nctas, int cta, size_t sub) {
  RoundPlan p;
  p.maxpart = ceil16((span + nctas - 1) / nctas);
  p.lo = min(span, (size_t)cta * p.maxpart);
  p.plen = min(span, p.lo + p.maxpart) - p.lo;
  p.round = (uint32_t)min(sub, max(kRoundMin, ceil16((p.maxpart + kRoundsPerCall - 1) /
                                                     kRoundsPerCall)));
  p.stagger = FLX_STAGGER && (cta & 1) && p.maxpart >= 2 * kRoundMin;
  return p;
}

// Slot-protocol phases (this round's piece pc = {offset, bytes} of CTA `mine`'s
// region), as one bulk pipeline (a.bulk) or register copies.
// Land: peer p's push in my inbox slot p -> recv block p (AllGather / AllToAll).
static __device__ __forceinline__ void land_all(const RankArgs& a, int r, int n, size_t mine,
                                                ulonglong2 pc) {
  if (a.bulk) {
    cta_copy_bulk([&](int i) {
      const int p = (r - 1 - i + n) % n;
      return CopySeg{a.recv + (size_t)p * a.rank_stride + pc.x,
                     a.scratch[r] + (size_t)p * a.slot + mine, pc.y};
    }, n - 1, true);
    return;
  }
  for (int s = 1; s < n; ++s) {
    const int p = (r - s + n) % n;
    cta_copy(a.recv + (size_t)p * a.rank_stride + pc.x, a.scratch[r] + (size_t)p * a.slot + mine,
             pc.y, true);
  }
}

// Push block c of send to peer c's inbox slot r (ReduceScatter / AllToAll);
// with `own`, my own block also lands in recv block r (AllToAll).
static __device__ __forceinline__ void push_blocks(const RankArgs& a, int r, int n, size_t mine,
                                                   ulonglong2 pc, bool own) {
  const size_t mo = (size_t)r * a.rank_stride + pc.x;
  if (a.bulk) {
    cta_copy_bulk([&](int i) {
      if (i == n - 1) return CopySeg{a.recv + mo, a.send + mo, own ? pc.y : 0};
      const int c = (r + 1 + i) % n;
      return CopySeg{a.scratch[c] + (size_t)r * a.slot + mine,
                     a.send + (size_t)c * a.rank_stride + pc.x, pc.y};
    }, n, false);
    return;
  }
  for (int s = 1; s < n; ++s) {
    const int c = (r + s) % n;
    cta_copy(a.scratch[c] + (size_t)r * a.slot + mine, a.send + (size_t)c * a.rank_stride + pc.x,
             pc.y, false);
  }
  if (own) cta_copy(a.recv + mo, a.send + mo, pc.y, false);
}

static __device__ void rank_allgather(const RankArgs& a, int cta, int nctas) {
  const int r = a.rank, n = a.nranks;
  const size_t sub = cta_sub(a.slot);
  const size_t mine = (size_t)cta * sub;  // this CTA's region in every slot
  const RoundPlan plan = round_plan(a.bytes, nctas, cta, sub);
  const CtaEpochs ep = cta_epochs(a, cta);
  uint32_t prev_main = ep.last_main;
  uint32_t k = 0;
  for (size_t at = 0; at < plan.maxpart; ++k) {
    const uint32_t e = ep.first + k;
    const uint32_t len = plan.len(at, k);
    const ulonglong2 pc = plan.piece(at, len);  // {send offset, bytes}
    {  // push my piece into every peer's inbox slot r (this CTA's region)
      if (!cta_wait_peers(a.flags[r], n, r, cta, kFree, prev_main, -1, 0, a)) return;
      char* own = a.recv + (size_t)r * a.rank_stride;
      if (a.bulk) {  // n-1 pushes and my own block, one pipeline
        cta_copy_bulk([&](int i) {
          if (i == n - 1) return CopySeg{own + pc.x, a.send + pc.x, own != a.send ? pc.y : 0};
          const int c = (r + 1 + i) % n;
          return CopySeg{a.scratch[c] + (size_t)r * a.slot + mine, a.send + pc.x, pc.y};
        }, n, false);
      } else {
        for (int s = 1; s < n; ++s) {
          const int c = (r + s) % n;
          cta_copy(a.scratch[c] + (size_t)r * a.slot + mine, a.send + pc.x, pc.y, false);
        }
        if (own != a.send) cta_copy(own + pc.x, a.send + pc.x, pc.y, false);
      }
      cta_signal_peers(a, cta, kArrive, e);
    }
    if (!cta_wait_peers(a.flags[r], n, r, cta, kArrive, e, -1, 0, a)) return;
    land_all(a, r, n, mine, pc);
    free_all(a, cta, e);
    prev_main = e;
    at += len;
  }
  cta_epochs_done(ep, k, ep.last_ar, prev_main);
}

// ReduceScatter: a.bytes = NVLink part of each recv block, a.rank_stride = the
// block stride R in send.  Push block c to peer c, fold my block in rank order.
template <typename T, int OP>
__device__ void rank_reducescatter(const RankArgs& a, int cta, int nctas) {
  const int r = a.rank, n = a.nranks;
  const size_t sub = cta_sub(a.slot);
  const size_t mine = (size_t)cta * sub;  // this CTA's region in every slot
  const RoundPlan plan = round_plan(a.bytes, nctas, cta, sub);
  const CtaEpochs ep = cta_epochs(a, cta);
  uint32_t prev_main = ep.last_main;
  uint32_t k = 0;
  for (size_t at = 0; at < plan.maxpart; ++k) {
    const uint32_t e = ep.first + k;
    const uint32_t len = plan.len(at, k);
    const ulonglong2 pc = plan.piece(at, len);  // {offset in a block, bytes}
    {
      if (!cta_wait_peers(a.flags[r], n, r, cta, kFree, prev_main, -1, 0, a)) return;
      push_blocks(a, r, n, mine, pc, false);
      cta_signal_peers(a, cta, kArrive, e);
    }
    if (!cta_wait_peers(a.flags[r], n, r, cta, kArrive, e, -1, 0, a)) return;
    {
      const char* own = a.send + (size_t)r * a.rank_stride + pc.x;
      const char* inbox = a.scratch[r] + mine;
      const size_t slot = a.slot;
      cta_fold<T, OP>(a.recv + pc.x, nullptr,
                      [=](int p) { return p == r ? own : inbox + (size_t)p * slot; }, n, pc.y);
    }
    free_all(a, cta, e);
    prev_main = e;
    at += len;
  }
  cta_epochs_done(ep, k, ep.last_ar, prev_main);
}

// AllToAll: a.bytes = NVLink part of each block, a.rank_stride = block stride
// B (send and recv).  Push block c to peer c, copy my own block locally, then
// land every peer's push into recv block p.
static __device__ void rank_alltoall(const RankArgs& a, int cta, int nctas) {
  const int r = a.rank, n = a.nranks;
  const size_t sub = cta_sub(a.slot);
  const size_t mine = (size_t)cta * sub;  // this CTA's region in every slot
  const RoundPlan plan = round_plan(a.bytes, nctas, cta, sub);
  const CtaEpochs ep = cta_epochs(a, cta);
  uint32_t prev_main = ep.last_main;
  uint32_t k = 0;
  for (size_t at = 0; at < plan.maxpart; ++k) {
    const uint32_t e = ep.first + k;
    const uint32_t len = plan.len(at, k);
    const ulonglong2 pc = plan.piece(at, len);  // {offset in a block, bytes}
    {
      if (!cta_wait_peers(a.flags[r], n, r, cta, kFree, prev_main, -1, 0, a)) return;
      push_blocks(a, r, n, mine, pc, true);
      cta_signal_peers(a, cta, kArrive, e);
    }
    if (!cta_wait_peers(a.flags[r], n, r, cta, kArrive, e, -1, 0, a)) return;
    land_all(a, r, n, mine, pc);
    free_all(a, cta, e);
    prev_main = e;
    at += len;
  }
  cta_epochs_done(ep, k, ep.last_ar, prev_main);
}

static __global__ void __launch_bounds__(512, 2) rank_alltoall_kernel(const __grid_constant__ RankArgs a) {
  if (a.oneshot) rank_oneshot<float, kSum, 3>(a, blockIdx.x, gridDim.x);
  else rank_alltoall(a, blockIdx.x, gridDim.x);
}

static __global__ void __launch_bounds__(512, 2) loopback_alltoall_kernel(const __grid_constant__ LoopbackArgs a) {
  if (a.r[blockIdx.y].oneshot) rank_oneshot<float, kSum, 3>(a.r[blockIdx.y], blockIdx.x, gridDim.x);
  else rank_alltoall(a.r[blockIdx.y], blockIdx.x, gridDim.x);
}

template <typename T, int OP>
__global__ void __launch_bounds__(512, 2) rank_allreduce_kernel(const __grid_constant__ RankArgs a) {
  if (a.oneshot) rank_oneshot<T, OP, 0>(a, blockIdx.x, gridDim.x);
  else rank_allreduce<T, OP>(a, blockIdx.x, gridDim.x);
}

template <typename T, int OP>
__global__ void __launch_bounds__(512, 2) rank_reducescatter_kernel(const __grid_constant__ RankArgs a) {
  if (a.oneshot) rank_oneshot<T, OP, 2>(a, blockIdx.x, gridDim.x);
  else rank_reducescatter<T, OP>(a, blockIdx.x, gridDim.x);
}

static __global__ void __launch_bounds__(512, 2) rank_allgather_kernel(const __grid_constant__ RankArgs a) {
  if (a.oneshot) rank_oneshot<float, kSum, 1>(a, blockIdx.x, gridDim.x);
  else rank_allgather(a, blockIdx.x, gridDim.x);
}

// Loopback: blockIdx.y is the rank; cooperative launch (all CTAs co-resident).
template <typename T, int OP>
__global__ void __launch_bounds__(512, 2) loopback_allreduce_kernel(const __grid_constant__ LoopbackArgs a) {
  if (a.r[blockIdx.y].oneshot) rank_oneshot<T, OP, 0>(a.r[blockIdx.y], blockIdx.x, gridDim.x);
  else rank_allreduce<T, OP>(a.r[blockIdx.y], blockIdx.x, gridDim.x);
}

template <typename T, int OP>
__global__ void __launch_bounds__(512, 2) loopback_reducescatter_kernel(const __grid_constant__ LoopbackArgs a) {
  if (a.r[blockIdx.y].oneshot) rank_oneshot<T, OP, 2>(a.r[blockIdx.y], blockIdx.x, gridDim.x);
  else rank_reducescatter<T, OP>(a.r[blockIdx.y], blockIdx.x, gridDim.x);
}

static __global__ void __launch_bounds__(512, 2) loopback_allgather_kernel(const __grid_constant__ LoopbackArgs a) {
  if (a.r[blockIdx.y].oneshot) rank_oneshot<float, kSum, 1>(a.r[blockIdx.y], blockIdx.x, gridDim.x);
  else rank_allgather(a.r[blockIdx.y], blockIdx.x, gridDim.x);
}

}  // namespace flx
