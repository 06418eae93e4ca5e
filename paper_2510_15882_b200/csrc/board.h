// The balancer's cross-rank agreement board (host only, no CUDA): a region of
// the shared host segment where every rank publishes the values of one
// decision point and reads everyone else's.  Slot (rank, k mod kBoardSlots)
// holds [stamp = k+1][count][kBoardDoubles values]; a rank writes its values,
// then release-stores the stamp, then waits for every peer's stamp k+1 in the
// same slot index and takes the elementwise max.  Ranks reach decision points
// in the same order and none can publish k+1 before every rank published k+1...
// which each does only after it finished reading k — so a slot is never
// rewritten while a peer still reads it, with 2 or more slots (4 here).
// Factored out of world.cu so tools/board_test.cpp can run it across real
// processes on the CPU (tests/test_board.py).
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <thread>

namespace flx {

constexpr int kBoardSlots = 4;     // decision points in flight (ranks are <= 1 apart)
constexpr int kBoardDoubles = 62;  // values per slot (+ stamp + count = 64 x 8 B)
constexpr size_t kBoardSlotWords = 64;

struct Board {
  char* base = nullptr;            // board start (kMaxRanks x kBoardSlots slots)
  int nranks = 0;
  int me = 0;
  uint64_t* seq = nullptr;         // decision points agreed so far (private, same on all ranks)
  volatile uint32_t* abort_word = nullptr;  // may be null
  double timeout_s = 10.0;
};

inline size_t board_bytes(int max_ranks) {
  return (size_t)max_ranks * kBoardSlots * kBoardSlotWords * 8;
}

// 0: ok; 1: a peer never arrived (timeout / abort; *bad = its rank);
// 2: a peer published a different value count (*bad = its rank)
inline int board_agree_max(const Board& b, double* vals, int n, int* bad) {
  auto slot = [&](int r, uint64_t k) {
    return reinterpret_cast<uint64_t*>(b.base) +
           ((size_t)r * kBoardSlots + k % kBoardSlots) * kBoardSlotWords;
  };
  for (int at = 0; at < n; at += kBoardDoubles) {
    const int m = std::min(kBoardDoubles, n - at);
    const uint64_t k = (*b.seq)++;
    uint64_t* mine = slot(b.me, k);
    mine[1] = (uint64_t)m;
    memcpy(mine + 2, vals + at, sizeof(double) * m);
    __atomic_store_n(&mine[0], k + 1, __ATOMIC_RELEASE);
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < b.nranks; ++r) {
      if (r == b.me) continue;
      uint64_t* theirs = slot(r, k);
      while (__atomic_load_n(&theirs[0], __ATOMIC_ACQUIRE) != k + 1) {
        if ((b.abort_word && *b.abort_word) ||
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() >
                b.timeout_s) {
          if (b.abort_word) *b.abort_word = 1;
          *bad = r;
          return 1;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(20));
      }
      if ((int)theirs[1] != m) {
        *bad = r;
        return 2;
      }
      double v[kBoardDoubles];
      memcpy(v, theirs + 2, sizeof(double) * m);
      for (int i = 0; i < m; ++i) vals[at + i] = std::max(vals[at + i], v[i]);
    }
  }
  return 0;
}

}  // namespace flx
