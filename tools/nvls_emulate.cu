// The NVLS AllReduce / AllGather kernels (csrc/nvls_kernels.cuh) executed with
// every multimem operation emulated by unicast loads / stores / reductions over
// every rank's buffer, all ranks on this GPU in one cooperative grid
// (FLX_NVLS_EMULATE).  This GPU is in no multicast fabric, so the switch path
// itself cannot run here; the emulation checks everything around it — the
// per-CTA partition, the per-CTA epochs across repeated calls, the two arrive
// barriers, staging and landing offsets, the AllGather stride — against a CPU
// fold in the same (rank) order: bit-exact.  One JSON line per case; exit 0
// iff all exact.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -o tools/bin/nvls_emulate tools/nvls_emulate.cu
#define FLX_NVLS_EMULATE 1
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#include "../paper_2510_15882_b200/csrc/nvls_kernels.cuh"

using namespace flx;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("{\"error\": \"%s: %s\"}\n", #x, cudaGetErrorString(e_));          \
      return false;                                                             \
    }                                                                           \
  } while (0)

static uint32_t lcg(uint32_t& s) { return s = s * 1664525u + 1013904223u; }

static float value(uint32_t& s) { return (float)((int)(lcg(s) >> 8) % 2001 - 1000) / 8.0f; }

static uint16_t to_bf16(float f) {  // round to nearest even (host)
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7fff + ((u >> 16) & 1);
  return (uint16_t)(u >> 16);
}
static float from_bf16(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

struct World {
  int n = 0, nctas = 0;
  std::vector<char*> send, recv, buf;
  std::vector<uint32_t*> state;
  uint32_t* abort_host = nullptr;
  uint32_t* abort_dev = nullptr;
  NvlsLoopArgs la;
};

static bool make(World& w, int n, size_t send_bytes, size_t recv_bytes, size_t buf_bytes) {
  w.n = n;
  int sms = 0, per_sm = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nvls_allreduce_loop_kernel<float>, 512, 0));
  w.nctas = std::min(kNvlsCtas, sms * per_sm / n);  // every CTA co-resident
  CK(cudaHostAlloc(&w.abort_host, 64, cudaHostAllocMapped));
  *w.abort_host = 0;
  CK(cudaHostGetDevicePointer(&w.abort_dev, w.abort_host, 0));
  memset(&w.la, 0, sizeof(w.la));
  for (int r = 0; r < n; ++r) {
    char *s, *d, *b;
    uint32_t* st;
    CK(cudaMalloc(&s, send_bytes));
    CK(cudaMalloc(&d, recv_bytes));
    CK(cudaMalloc(&b, kNvlsFlagBytes + buf_bytes));
    CK(cudaMemset(b, 0, kNvlsFlagBytes + buf_bytes));
    CK(cudaMalloc(&st, kNvlsCtas * sizeof(uint32_t)));
    CK(cudaMemset(st, 0, kNvlsCtas * sizeof(uint32_t)));
    w.send.push_back(s);
    w.recv.push_back(d);
    w.buf.push_back(b);
    w.state.push_back(st);
  }
  for (int r = 0; r < n; ++r) {
    NvlsArgs& a = w.la.r[r];
    a.send = w.send[r];
    a.recv = w.recv[r];
    a.uc = w.buf[r];
    a.mc = nullptr;  // no multicast mapping: the emulation addresses the peers directly
    a.state = w.state[r];
    a.rank = r;
    a.nranks = n;
    a.abort_word = w.abort_dev;
    a.spin_limit = 20000000000ll;
    for (int q = 0; q < n; ++q) a.peers[q] = w.buf[q];
  }
  return true;
}

static void destroy(World& w) {
  for (int r = 0; r < w.n; ++r) {
    cudaFree(w.send[r]);
    cudaFree(w.recv[r]);
    cudaFree(w.buf[r]);
    cudaFree(w.state[r]);
  }
  cudaFreeHost(w.abort_host);
}

// AllReduce: bytes per rank = n * chunk; `bf16` selects the element type
static bool allreduce_case(int n, size_t chunk, bool bf16, int calls) {
  const size_t bytes = (size_t)n * chunk, esz = bf16 ? 2 : 4, count = bytes / esz;
  World w;
  if (!make(w, n, bytes, bytes, bytes)) return false;
  for (int r = 0; r < n; ++r) w.la.r[r].bytes = bytes;
  bool ok = true;
  uint32_t seed = 12345u + (uint32_t)n * 7u + (uint32_t)chunk;
  std::vector<std::vector<float>> in(n, std::vector<float>(count));
  std::vector<char> host(bytes);
  for (int call = 0; call < calls && ok; ++call) {
    for (int r = 0; r < n; ++r) {
      for (size_t i = 0; i < count; ++i) {
        float v = value(seed);
        if (bf16) {
          const uint16_t h = to_bf16(v);
          v = from_bf16(h);
          memcpy(host.data() + 2 * i, &h, 2);
        } else {
          memcpy(host.data() + 4 * i, &v, 4);
        }
        in[r][i] = v;
      }
      CK(cudaMemcpy(w.send[r], host.data(), bytes, cudaMemcpyHostToDevice));
      CK(cudaMemset(w.recv[r], 0xff, bytes));
    }
    void* params[] = {&w.la};
    const void* fn = bf16 ? (const void*)nvls_allreduce_loop_kernel<__nv_bfloat16>
                          : (const void*)nvls_allreduce_loop_kernel<float>;
    CK(cudaLaunchCooperativeKernel(fn, dim3(w.nctas, n), dim3(512), params, 0, 0));
    CK(cudaDeviceSynchronize());
    if (*w.abort_host) {
      ok = false;
      break;
    }
    for (int r = 0; r < n && ok; ++r) {
      CK(cudaMemcpy(host.data(), w.recv[r], bytes, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < count; ++i) {
        float acc = in[0][i];  // rank-order fold, fp32 accumulation (the emulation's order)
        for (int q = 1; q < n; ++q) acc += in[q][i];
        bool same;
        if (bf16) {
          uint16_t got;
          memcpy(&got, host.data() + 2 * i, 2);
          same = got == to_bf16(acc);
        } else {
          float got;
          memcpy(&got, host.data() + 4 * i, 4);
          same = memcmp(&got, &acc, 4) == 0;
        }
        if (!same) {
          ok = false;
          break;
        }
      }
    }
  }
  printf("{\"op\": \"allreduce\", \"n\": %d, \"dtype\": \"%s\", \"chunk_bytes\": %zu, \"ctas\": %d, "
         "\"calls\": %d, \"exact\": %s}\n",
         n, bf16 ? "bf16" : "f32", chunk, w.nctas, calls, ok ? "true" : "false");
  destroy(w);
  return ok;
}

// AllGather: `bytes` sent per rank, recv blocks at `stride` (>= bytes)
static bool allgather_case(int n, size_t bytes, size_t stride, int calls) {
  World w;
  if (!make(w, n, bytes, (size_t)n * stride, (size_t)n * bytes)) return false;
  for (int r = 0; r < n; ++r) w.la.r[r].bytes = bytes;
  bool ok = true;
  uint32_t seed = 777u + (uint32_t)n;
  std::vector<std::vector<char>> in(n, std::vector<char>(bytes));
  std::vector<char> host((size_t)n * stride);
  for (int call = 0; call < calls && ok; ++call) {
    for (int r = 0; r < n; ++r) {
      for (size_t i = 0; i < bytes; ++i) in[r][i] = (char)(lcg(seed) >> 24);
      CK(cudaMemcpy(w.send[r], in[r].data(), bytes, cudaMemcpyHostToDevice));
      CK(cudaMemset(w.recv[r], 0x5a, (size_t)n * stride));
    }
    void* params[] = {&w.la, &stride};
    CK(cudaLaunchCooperativeKernel((const void*)nvls_allgather_loop_kernel, dim3(w.nctas, n),
                                   dim3(512), params, 0, 0));
    CK(cudaDeviceSynchronize());
    if (*w.abort_host) {
      ok = false;
      break;
    }
    for (int r = 0; r < n && ok; ++r) {
      CK(cudaMemcpy(host.data(), w.recv[r], (size_t)n * stride, cudaMemcpyDeviceToHost));
      for (int c = 0; c < n && ok; ++c) {
        ok = memcmp(host.data() + (size_t)c * stride, in[c].data(), bytes) == 0;
        // the gap between blocks (stride > bytes) is left untouched
        for (size_t i = bytes; ok && i < stride; ++i) ok = host[(size_t)c * stride + i] == 0x5a;
      }
    }
  }
  printf("{\"op\": \"allgather\", \"n\": %d, \"bytes\": %zu, \"stride\": %zu, \"ctas\": %d, "
         "\"calls\": %d, \"exact\": %s}\n",
         n, bytes, stride, w.nctas, calls, ok ? "true" : "false");
  destroy(w);
  return ok;
}

int main() {
  bool ok = true;
  for (int n : {2, 4, 8}) {
    // chunk lengths: one vector; 64 CTAs' parts with a 16 B remainder (the
    // floor-then-round partition left it unreduced); ragged; 1 MiB
    for (size_t chunk : {(size_t)16, (size_t)(64 * 256 + 16), (size_t)(16 * 1001), (size_t)(1 << 20)}) {
      ok = allreduce_case(n, chunk, false, 3) && ok;
      ok = allreduce_case(n, chunk, true, 2) && ok;
    }
    for (size_t bytes : {(size_t)16, (size_t)(64 * 256 + 16), (size_t)(1 << 20)}) {
      ok = allgather_case(n, bytes, bytes, 3) && ok;
      ok = allgather_case(n, bytes, bytes + 48, 2) && ok;
    }
  }
  return ok ? 0 : 1;
}
