// In-library two-stage balancer: Stage 1 and Stage 2 driven by the real
// collective's per-path CUDA-event times, per (collective, size bucket), inside
// every communicator (virtual-rank clique or multi-rank world).  See
// include/flexlink_tuner.h for the behaviour and autotune.cpp for the
// mechanics.
#pragma once

#include <deque>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "internal.h"
#include "tuner.h"

namespace flx {

// Where a tuner reads per-path times and agrees them across ranks.
struct TimingPort {
  virtual ~TimingPort() = default;
  // Per-path ms of call `seq` (max over this process's ranks), blocking until
  // the call finished.  Unused paths read 0.
  virtual flxResult_t read(uint64_t seq, float ms[FLX_NUM_PATHS]) = 0;
  // Elementwise max over every rank of the communicator, in place.  Every rank
  // reaches the same agree() calls in the same order (a rendezvous);
  // single-process communicators return at once.
  virtual flxResult_t agree_max(double* vals, int n) = 0;
  // Calls issued so far (= the sequence number of the next call).
  virtual uint64_t calls() const = 0;
  // Identity for the persisted share cache, e.g. "B200/virtual/n8".
  virtual std::string scope() const = 0;
  virtual bool cache_writer() const = 0;
};

struct TunePolicy {  // copied from the lead comm when a bucket is first tuned
  flxTunerConfig s1;
  flxBalancerConfig s2;
  bool have_profile = false;
  flxLinkProfile profile{};
  int nvlink_ctas = 0;
};

class AutoTuner {
 public:
  // Decide the shares of the next call of (op, bytes).  `tunable` = autotune
  // on, bucket not pinned, >= min bytes; `can_measure` = timed and not inside a
  // CUDA-graph capture (otherwise the current split is used, no step).
  // `fallback` is what the share table says (used when not tunable).
  // *measured tells after_call whether to record this call.
  flxResult_t before_call(TimingPort& port, const TunePolicy& pol, int op, size_t bytes,
                          bool tunable, bool can_measure, int path_mask,
                          const Granules& fallback, Granules* g, bool* measured);
  void after_call(int op, size_t bytes, uint64_t seq, const std::array<size_t, FLX_NUM_PATHS>& split,
                  bool measured);
  bool info(int op, int bucket, flxTuneInfo* out) const;
  int trace(int op, int bucket, flxTuneRecord* out, int max) const;
  int evaluations(int op, int bucket, flxEvalRecord* out, int max) const;
  bool current(int op, int bucket, Granules* g) const;
  // forget every bucket (a path setting changed: earlier measurements are void)
  void reset() {
    slots_.clear();
    unread_.clear();
  }

 private:
  struct Meas {
    uint64_t seq = 0;
    int mask = 0;          // paths that carried bytes
    bool read = false;     // local times fetched
    bool agreed = false;   // max over ranks applied
    double ms[FLX_NUM_PATHS] = {0, 0, 0};
    double bytes[FLX_NUM_PATHS] = {0, 0, 0};
  };
  using MeasPtr = std::shared_ptr<Meas>;
  struct Slot {
    int phase = flxTuneIdle;
    TunePolicy pol;
    Granules cur{{FLX_GRANULE_TOTAL, 0, 0}};
    int round_calls = 0;               // calls issued in the current round
    int repeats = 3;                   // measured calls per round (adapted after the baseline)
    std::vector<MeasPtr> round;        // its measured calls
    MeasPtr pending;                   // the call being issued
    flxTunerState st{};
    std::vector<flxTuneRecord> trace;
    bool converged = false, kept = false, from_cache = false;
    double nv_ms = 0, tuned_ms = 0, seed[FLX_NUM_PATHS] = {0, 0, 0};
    Granules stage1{{FLX_GRANULE_TOTAL, 0, 0}};
    // Stage 2
    int s2_active = 0;
    int s2_calls = 0;                  // stage-2 calls issued
    int s2_observed = 0;               // reports observed (lags s2_calls by `lag`)
    std::deque<MeasPtr> lagq;          // issued, not yet observed
    std::deque<MeasPtr> window;        // observed, newest last
    std::deque<flxEvalRecord> evals;  // the last kMaxEvals evaluation records
    int n_evals = 0;                  // every evaluation so far
    int moves = 0;
    int calls = 0;
  };
  flxResult_t decide_round(TimingPort& port, Slot& s, int path_mask);
  flxResult_t stage2_call(TimingPort& port, Slot& s);
  flxResult_t fetch(TimingPort& port, const std::vector<MeasPtr>& ms);
  flxResult_t harvest(TimingPort& port);
  void finish_stage1(Slot& s);
  void start_stage2(Slot& s, const Granules& g);
  bool cache_lookup(TimingPort& port, int op, int bucket, const Slot& s, Granules* g);
  void cache_store(TimingPort& port, int op, int bucket, const Slot& s);

  std::map<std::pair<int, int>, Slot> slots_;
  std::deque<MeasPtr> unread_;  // measured calls whose events are not read yet
};

// Process-wide tuning defaults (env FLX_AUTOTUNE, FLX_AUTOTUNE_MIN_KB).
bool autotune_default();
size_t autotune_min_bytes_default();

}  // namespace flx
