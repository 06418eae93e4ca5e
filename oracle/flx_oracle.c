/*
 * flx_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU data-plane oracle.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * `--impl reference`) may load this library, and only as the checker or the
 * CPU baseline.  The product path (paper_2510_15882_b200) never calls it.
 *
 * What it restates.  The reference (linkstripe) never moves bytes; its
 * collective is the closed-form model `simulate_collective`
 * (pkg/src/linkstripe/collectives.py:136-186), which fixes the *contract*:
 *   - the message (per-rank `size` bytes, nccl-tests convention,
 *     collectives.py:4-7,49) is split per path by `partition`
 *     (collectives.py:93-114): floor(size*g/sum(g)) rounded down to
 *     `alignment`, remainder to NVLINK;
 *   - "each path independently runs the ring schedule on its slice"
 *     (collectives.py:145-153): the slice splits into N rank chunks
 *     (size/N per step, collectives.py:167); chunk c is reduced for rank c
 *     (reduce-scatter) and then circulated to every rank (all-gather) —
 *     2(N-1) steps for AllReduce, N-1 for AllGather (ring_steps,
 *     collectives.py:31-39).
 * The byte layout of the slices (PCIE at offset 0, then RDMA, then NVLINK,
 * which absorbs the remainder at its end so the secondary slices stay on the
 * alignment grid) and the reduction order are not defined by the reference
 * (SURVEY.md §8c); this build fixes them: every element is reduced entirely inside one path by the
 * left fold acc = x[0]; acc = op(acc, x[r]) for r = 1..N-1 in rank order,
 * accumulated in fp32 for fp16/bf16 (one final RNE rounding), in the native
 * type otherwise (integers wrap).  AllGather is a pure byte copy.
 *
 * Build: oracle/Makefile (gcc -O3 -fopenmp -ffp-contract=off; vectorised
 * across elements only, never across ranks, so the fold order is kept).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { I8 = 0, U8 = 1, I32 = 2, U32 = 3, I64 = 4, U64 = 5, F16 = 6, F32 = 7, F64 = 8, BF16 = 9 };
enum { SUM = 0, PROD = 1, MAX = 2, MIN = 3 };
/* slice order in a rank's message: pcie (1), rdma (2), nvlink (0) last */
static const uint64_t kOrder[3] = {1, 2, 0};

/* ------------------------------------------------------------ conversions */
static inline float bits_to_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static inline uint32_t f32_to_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

static inline float bf16_to_f32(uint16_t h) { return bits_to_f32((uint32_t)h << 16); }

/* round-to-nearest-even, NaN -> canonical 0x7FFF (cvt.rn.bf16.f32) */
static inline uint16_t f32_to_bf16(float f) {
  uint32_t u = f32_to_bits(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fff;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static inline float f16_to_f32(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000) << 16;
  uint32_t exp = (h >> 10) & 0x1f, man = h & 0x3ff;
  if (exp == 0) {
    if (man == 0) return bits_to_f32(sign);
    float v = (float)man * 5.9604644775390625e-08f; /* 2^-24, exact */
    return sign ? -v : v;
  }
  if (exp == 31) return bits_to_f32(sign | 0x7f800000u | (man << 13));
  return bits_to_f32(sign | ((exp + 112) << 23) | (man << 13));
}

/* round-to-nearest-even with subnormals and overflow to inf (cvt.rn.f16.f32) */
static inline uint16_t f32_to_f16(float f) {
  uint32_t u = f32_to_bits(f);
  uint16_t sign = (uint16_t)((u >> 16) & 0x8000);
  uint32_t a = u & 0x7fffffffu;
  if (a > 0x7f800000u) return 0x7fff;
  if (a >= 0x47800000u) return sign | 0x7c00; /* >= 65536 (and inf) */
  if (a < 0x38800000u) {                      /* below 2^-14: half subnormal / zero */
    float mag = bits_to_f32(a);
    float scaled = mag * 16777216.0f; /* / 2^-24, exact */
    /* nearbyint in the default RNE mode */
    float q = rintf(scaled);
    return sign | (uint16_t)q;
  }
  uint32_t odd = (a >> 13) & 1u;
  a += 0xc8000fffu + odd; /* rebias exponent (-112 << 23) and round */
  return sign | (uint16_t)(a >> 13);
}

/* -------------------------------------------------------------- the fold */
/* Blocked so the per-element work vectorises across elements while every
 * element keeps its left fold in rank order: the loop over ranks is outside
 * the loop over a block's elements, nothing is reassociated, and all sources
 * of a block are read before any destination is written (in-place safe). */
#define FOLD_BLOCK 2048

#define FOLD_INT(T, UT)                                                                     \
  static void fold_##T(const void* const* src, void* const* dst, int n, int ndst,           \
                       uint64_t i0, uint64_t i1, int op) {                                  \
    T acc[FOLD_BLOCK];                                                                      \
    for (uint64_t b = i0; b < i1; b += FOLD_BLOCK) {                                        \
      const int len = (int)(i1 - b < FOLD_BLOCK ? i1 - b : FOLD_BLOCK);                     \
      memcpy(acc, (const T*)src[0] + b, (size_t)len * sizeof(T));                           \
      for (int r = 1; r < n; ++r) {                                                         \
        const T* x = (const T*)src[r] + b;                                                  \
        if (op == SUM)                                                                      \
          for (int j = 0; j < len; ++j) acc[j] = (T)(UT)((UT)acc[j] + (UT)x[j]);            \
        else if (op == PROD)                                                                \
          for (int j = 0; j < len; ++j) acc[j] = (T)(UT)((UT)acc[j] * (UT)x[j]);            \
        else if (op == MAX)                                                                 \
          for (int j = 0; j < len; ++j) acc[j] = (x[j] > acc[j]) ? x[j] : acc[j];           \
        else                                                                                \
          for (int j = 0; j < len; ++j) acc[j] = (x[j] < acc[j]) ? x[j] : acc[j];           \
      }                                                                                     \
      for (int r = 0; r < ndst; ++r) memcpy((T*)dst[r] + b, acc, (size_t)len * sizeof(T)); \
    }                                                                                       \
  }

FOLD_INT(int8_t, uint8_t)
FOLD_INT(uint8_t, uint8_t)
FOLD_INT(int32_t, uint32_t)
FOLD_INT(uint32_t, uint32_t)
FOLD_INT(int64_t, uint64_t)
FOLD_INT(uint64_t, uint64_t)

#define FOLD_FLOAT(NAME, T, A, LOAD, STORE)                                                 \
  static void fold_##NAME(const void* const* src, void* const* dst, int n, int ndst,        \
                          uint64_t i0, uint64_t i1, int op) {                               \
    A acc[FOLD_BLOCK];                                                                      \
    T out[FOLD_BLOCK];                                                                      \
    for (uint64_t b = i0; b < i1; b += FOLD_BLOCK) {                                        \
      const int len = (int)(i1 - b < FOLD_BLOCK ? i1 - b : FOLD_BLOCK);                     \
      const T* s0 = (const T*)src[0] + b;                                                   \
      for (int j = 0; j < len; ++j) acc[j] = LOAD(s0[j]);                                   \
      for (int r = 1; r < n; ++r) {                                                         \
        const T* x = (const T*)src[r] + b;                                                  \
        if (op == SUM)                                                                      \
          for (int j = 0; j < len; ++j) acc[j] = acc[j] + LOAD(x[j]);                       \
        else if (op == PROD)                                                                \
          for (int j = 0; j < len; ++j) acc[j] = acc[j] * LOAD(x[j]);                       \
        else if (op == MAX)                                                                 \
          for (int j = 0; j < len; ++j) {                                                   \
            const A v = LOAD(x[j]);                                                         \
            acc[j] = (v > acc[j]) ? v : acc[j];                                             \
          }                                                                                 \
        else                                                                                \
          for (int j = 0; j < len; ++j) {                                                   \
            const A v = LOAD(x[j]);                                                         \
            acc[j] = (v < acc[j]) ? v : acc[j];                                             \
          }                                                                                 \
      }                                                                                     \
      for (int j = 0; j < len; ++j) out[j] = STORE(acc[j]);                                 \
      for (int r = 0; r < ndst; ++r) memcpy((T*)dst[r] + b, out, (size_t)len * sizeof(T));  \
    }                                                                                       \
  }

#define IDENT(x) (x)
FOLD_FLOAT(f32, float, float, IDENT, IDENT)
FOLD_FLOAT(f64, double, double, IDENT, IDENT)
FOLD_FLOAT(bf16, uint16_t, float, bf16_to_f32, f32_to_bf16)
FOLD_FLOAT(f16, uint16_t, float, f16_to_f32, f32_to_f16)

typedef void (*fold_fn)(const void* const*, void* const*, int, int, uint64_t, uint64_t, int);

static fold_fn pick(int dtype) {
  switch (dtype) {
    case I8: return fold_int8_t;
    case U8: return fold_uint8_t;
    case I32: return fold_int32_t;
    case U32: return fold_uint32_t;
    case I64: return fold_int64_t;
    case U64: return fold_uint64_t;
    case F16: return fold_f16;
    case F32: return fold_f32;
    case F64: return fold_f64;
    case BF16: return fold_bf16;
  }
  return 0;
}

int flxo_dtype_size(int dtype) {
  switch (dtype) {
    case I8: case U8: return 1;
    case F16: case BF16: return 2;
    case I32: case U32: case F32: return 4;
    case I64: case U64: case F64: return 8;
  }
  return 0;
}

/* partition (collectives.py:93-114) over paths {nvlink, pcie, rdma} */
int flxo_partition(uint64_t size, const int granules[3], uint64_t alignment, uint64_t out[3]) {
  if (alignment < 1) return -1;
  long long denom = 0;
  for (int p = 0; p < 3; ++p) {
    if (granules[p] < 0) return -1;
    denom += granules[p];
  }
  if (size > 0 && denom <= 0) return -1;
  uint64_t used = 0;
  for (int p = 0; p < 3; ++p) {
    unsigned __int128 raw = denom ? (unsigned __int128)size * (unsigned)granules[p] / denom : 0;
    out[p] = (uint64_t)raw / alignment * alignment;
    used += out[p];
  }
  out[0] += size - used;
  return 0;
}

static void set_threads(int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
}

/*
 * AllReduce over `nranks` simulated ranks: send[r]/recv[r] hold `count`
 * elements.  For every path slice, for every ring chunk c (owner rank c), the
 * chunk's elements are folded in rank order and the result lands in every
 * rank's recv (reduce-scatter to the owner, then all-gather).
 */
int flxo_allreduce(const void* const* send, void* const* recv, int nranks, uint64_t count,
                   int dtype, int op, const int granules[3], uint64_t alignment, int threads) {
  const int esz = flxo_dtype_size(dtype);
  fold_fn fold = pick(dtype);
  if (!esz || !fold || nranks < 1 || op < 0 || op > 3) return -1;
  uint64_t split[3];
  if (flxo_partition(count * esz, granules, alignment, split)) return -1;
  for (uint64_t k = 0, p = kOrder[0], at = 0; k < 3; at += split[p], p = kOrder[++k % 3]) {
    if (split[p] % esz) return -2; /* slice boundary inside an element */
    const uint64_t e0 = at / esz, elems = split[p] / esz;
    const uint64_t per = (elems + nranks - 1) / nranks; /* ring chunk per owner */
    set_threads(threads);
#pragma omp parallel for schedule(static)
    for (long long c = 0; c < (long long)nranks * 64; ++c) {
      /* owner = c / 64; each owner's chunk is cut in 64 parts for the threads */
      const uint64_t owner = (uint64_t)c / 64, part = (uint64_t)c % 64;
      uint64_t lo = owner * per, hi = lo + per;
      if (hi > elems) hi = elems;
      if (lo >= hi) continue;
      const uint64_t span = hi - lo, plo = lo + span * part / 64, phi = lo + span * (part + 1) / 64;
      fold(send, recv, nranks, nranks, e0 + plo, e0 + phi, op);
    }
  }
  return 0;
}

/*
 * AllGather: recv[q][r*sendcount + i] = send[r][i] for all q, r.  The per-rank
 * send bytes are partitioned per path; every path's slice of every rank's
 * block is copied (the ring's N-1 forwarding steps just move these bytes).
 */
int flxo_allgather(const void* const* send, void* const* recv, int nranks, uint64_t sendcount,
                   int dtype, const int granules[3], uint64_t alignment, int threads) {
  const int esz = flxo_dtype_size(dtype);
  if (!esz || nranks < 1) return -1;
  const uint64_t bytes = sendcount * esz;
  uint64_t split[3];
  if (flxo_partition(bytes, granules, alignment, split)) return -1;
  set_threads(threads);
  for (uint64_t k = 0, p = kOrder[0], at = 0; k < 3; at += split[p], p = kOrder[++k % 3]) {
    const uint64_t len = split[p];
    if (!len) continue;
#pragma omp parallel for collapse(2) schedule(static)
    for (int q = 0; q < nranks; ++q)
      for (int r = 0; r < nranks; ++r)
        memmove((char*)recv[q] + (uint64_t)r * bytes + at, (const char*)send[r] + at, len);
  }
  return 0;
}

/*
 * ReduceScatter (ring_steps N-1; the reduce-scatter half of the AllReduce
 * ring): recv[r][i] = fold_q send[q][r*recvcount + i].  The per-rank recv
 * block bytes are partitioned per path; each path's slice of every block is
 * folded in rank order.
 */
int flxo_reducescatter(const void* const* send, void* const* recv, int nranks,
                       uint64_t recvcount, int dtype, int op, const int granules[3],
                       uint64_t alignment, int threads) {
  const int esz = flxo_dtype_size(dtype);
  fold_fn fold = pick(dtype);
  if (!esz || !fold || nranks < 1 || nranks > 64 || op < 0 || op > 3) return -1;
  uint64_t split[3];
  if (flxo_partition(recvcount * esz, granules, alignment, split)) return -1;
  for (int p = 0; p < 3; ++p)
    if (split[p] % esz) return -2;
  set_threads(threads);
#pragma omp parallel for schedule(static)
  for (int r = 0; r < nranks; ++r) {
    const void* rows[64];
    void* dst[1] = {recv[r]};
    for (int q = 0; q < nranks; ++q)
      rows[q] = (const char*)send[q] + (uint64_t)r * recvcount * esz;
    for (uint64_t k = 0, p = kOrder[0], at = 0; k < 3; at += split[p], p = kOrder[++k % 3])
      if (split[p]) fold(rows, dst, nranks, 1, at / esz, (at + split[p]) / esz, op);
  }
  return 0;
}

/*
 * AllToAll (N-1 pairwise steps): recv[q][r*count + i] = send[r][q*count + i].
 * The per-block bytes are partitioned per path; every path moves its slice of
 * every block.
 */
int flxo_alltoall(const void* const* send, void* const* recv, int nranks, uint64_t count,
                  int dtype, const int granules[3], uint64_t alignment, int threads) {
  const int esz = flxo_dtype_size(dtype);
  if (!esz || nranks < 1) return -1;
  const uint64_t block = count * esz;
  uint64_t split[3];
  if (flxo_partition(block, granules, alignment, split)) return -1;
  set_threads(threads);
  for (uint64_t k = 0, p = kOrder[0], at = 0; k < 3; at += split[p], p = kOrder[++k % 3]) {
    if (!split[p]) continue;
#pragma omp parallel for collapse(2) schedule(static)
    for (int q = 0; q < nranks; ++q)
      for (int r = 0; r < nranks; ++r)
        memcpy((char*)recv[q] + (uint64_t)r * block + at,
               (const char*)send[r] + (uint64_t)q * block + at, split[p]);
  }
  return 0;
}

/* element conversions exported for the Python side of the tests */
float flxo_bf16_to_f32(uint16_t h) { return bf16_to_f32(h); }
uint16_t flxo_f32_to_bf16(float f) { return f32_to_bf16(f); }
float flxo_f16_to_f32(uint16_t h) { return f16_to_f32(h); }
uint16_t flxo_f32_to_f16(float f) { return f32_to_f16(f); }
