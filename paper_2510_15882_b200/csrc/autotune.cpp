// In-library two-stage balancer (see include/flexlink_tuner.h).
//
// Every eligible call of a (collective, size bucket) is one step of a small
// state machine.  Stage 1 works in ROUNDS of `warm` unmeasured + `repeats`
// measured calls with a fixed split; the decision for the next round is taken
// when its first call is issued: the round's CUDA-event times are read (the
// host waits for the last call of the round — Stage 1 is start-up profiling,
// the paper's ~10 s phase), agreed across ranks (max), reduced
// to per-path medians and fed to tune_step (tuner.py:134-175):
//
//   baseline  NVLink-only round: the guard's reference and the NVLink rate
//   probe     a round with kProbeGranules on PCIe: the PCIe rate.  The two
//             measured rates are the link profile initialize_shares seeds
//             from (tuner.py:81-107), unless flxSetLinkProfile installed one
//   stage 1   one tune_step per round until `stability_required` stable
//             rounds, an early exit (NVLink alone left) or the iteration cap
//             (then one more round measures the final split)
//   guard     keep the tuned split only if its total beat NVLink-only (the
//             Python tune_shares guard)
//
// Stage 2 (balancer.py:163-207) then observes EVERY call, with a lag: before
// issuing stage-2 call c it observes call c-`lag`, so reading that call's
// events never stalls the GPU queue (the host only waits when it is more than
// `lag` calls ahead); every invocation_period observations it evaluates the
// window's per-path medians (agreed across ranks) and moves a quantum.
// Decisions depend only on agreed values and the call sequence, so every rank
// of a world computes the same split for the same call.
#include <sys/stat.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>

#include "autotune.h"

namespace flx {

namespace {
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}
// round shape and lag (FLX_TUNE_WARM / FLX_TUNE_REPEATS / FLX_TUNE_LAG)
int warm_calls() { static const int v = std::max(0, env_int("FLX_TUNE_WARM", 1)); return v; }
int repeat_calls() { static const int v = std::max(1, env_int("FLX_TUNE_REPEATS", 3)); return v; }
// measured time a round should span (FLX_TUNE_ROUND_US): short calls get more
// repeats so the per-path medians fed to tune_step are not noise (a 50 us call
// carries a few us of event jitter, the order of the 5 % convergence threshold)
double round_target_ms() {
  static const double v = std::max(0, env_int("FLX_TUNE_ROUND_US", 2000)) * 1e-3;
  return v;
}
constexpr int kMaxRepeats = 16;
// 8: a Stage-2 evaluation reads calls at least 8 behind the one being issued, so
// the host blocks on their events only when it runs more than 8 collectives ahead
// of the GPU (PyTorch's eager loop queues a layer or more ahead)
int stage2_lag() { static const int v = std::max(0, env_int("FLX_TUNE_LAG", 8)); return v; }
constexpr int kProbeGranules = 100;  // PCIe share of the rate-probe round
constexpr size_t kMaxEvals = 256;

int loaded_mask(const Granules& g) {
  int m = 0;
  for (int p = 0; p < FLX_NUM_PATHS; ++p)
    if (g[p] > 0) m |= 1 << p;
  return m;
}
}  // namespace

bool autotune_default() {
  static const bool on = env_int("FLX_AUTOTUNE", 1) != 0;
  return on;
}

size_t autotune_min_bytes_default() {
  static const size_t v = (size_t)std::max(0, env_int("FLX_AUTOTUNE_MIN_KB", 16384)) << 10;
  return v;
}

// Read (blocking) every unread measurement, then max-agree the unagreed ones
// across ranks in one batch.
flxResult_t AutoTuner::fetch(TimingPort& port, const std::vector<MeasPtr>& ms) {
  std::vector<double> vals;
  std::vector<Meas*> todo;
  for (const MeasPtr& m : ms) {
    if (!m->read) {
      float t[FLX_NUM_PATHS];
      FLX_TRY(port.read(m->seq, t));
      for (int p = 0; p < FLX_NUM_PATHS; ++p) m->ms[p] = t[p];
      m->read = true;
    }
    if (!m->agreed) {
      todo.push_back(m.get());
      for (int p = 0; p < FLX_NUM_PATHS; ++p) vals.push_back(m->ms[p]);
    }
  }
  if (!todo.empty()) {
    FLX_TRY(port.agree_max(vals.data(), (int)vals.size()));
    for (size_t i = 0; i < todo.size(); ++i) {
      for (int p = 0; p < FLX_NUM_PATHS; ++p) todo[i]->ms[p] = vals[3 * i + p];
      todo[i]->agreed = true;
    }
  }
  return flxSuccess;
}

// Per-call timing events live in a 64-slot ring: read a measured call before
// its slot can be reused (only blocks when the host is ~48 calls ahead).
flxResult_t AutoTuner::harvest(TimingPort& port) {
  const uint64_t next = port.calls();
  while (!unread_.empty()) {
    MeasPtr& m = unread_.front();
    if (!m->read && m.use_count() > 1) {
      if (m->seq + 48 > next) break;
      float t[FLX_NUM_PATHS];
      FLX_TRY(port.read(m->seq, t));
      for (int p = 0; p < FLX_NUM_PATHS; ++p) m->ms[p] = t[p];
      m->read = true;
    }
    unread_.pop_front();
  }
  return flxSuccess;
}

void AutoTuner::start_stage2(Slot& s, const Granules& g) {
  s.phase = flxTuneStage2;
  s.cur = g;
  s.s2_active = loaded_mask(g);
  s.s2_calls = s.s2_observed = 0;
  s.lagq.clear();
  s.window.clear();
}

void AutoTuner::finish_stage1(Slot& s) {
  Granules tuned{{s.st.shares[0], s.st.shares[1], s.st.shares[2]}};
  s.kept = loaded_mask(tuned) != (1 << flxPathNvlink) && s.tuned_ms < s.nv_ms;
  s.stage1 = s.kept ? tuned : Granules{{FLX_GRANULE_TOTAL, 0, 0}};
  start_stage2(s, s.stage1);
}

flxResult_t AutoTuner::decide_round(TimingPort& port, Slot& s, int path_mask) {
  FLX_TRY(fetch(port, s.round));
  // per-path medians over the round's calls (PathTimingReport of the round)
  tune::Report rep;
  rep.mask = s.round.empty() ? 0 : s.round[0]->mask;
  double bytes[FLX_NUM_PATHS] = {0, 0, 0};
  for (int p = 0; p < FLX_NUM_PATHS; ++p) {
    if (!(rep.mask >> p & 1)) continue;
    std::vector<double> v;
    for (const MeasPtr& m : s.round) v.push_back(m->ms[p]);
    std::sort(v.begin(), v.end());
    const size_t n = v.size();
    rep.ms[p] = n % 2 ? v[n / 2] : (v[n / 2 - 1] + v[n / 2]) / 2;
    bytes[p] = s.round[0]->bytes[p];
  }
  double total = 0;
  for (int p = 0; p < FLX_NUM_PATHS; ++p)
    if (rep.mask >> p & 1) total = std::max(total, rep.ms[p]);
  s.round.clear();
  s.round_calls = 0;
  const int nv_pc = (1 << flxPathNvlink) | (1 << flxPathPcie);

  switch (s.phase) {
    case flxTuneBaseline: {
      s.nv_ms = total;
      // later rounds repeat enough calls to span round_target_ms() (agreed
      // value on every rank, so every rank uses the same round length)
      if (total > 0)
        s.repeats = std::max(repeat_calls(),
                             std::min(kMaxRepeats, (int)std::ceil(round_target_ms() / total)));
      if (rep.mask & 1) s.seed[flxPathNvlink] = bytes[0] / (rep.ms[0] * 1e-3);
      flxLinkProfile prof{};
      if (s.pol.have_profile) {
        prof = s.pol.profile;
      } else if ((path_mask & nv_pc) == nv_pc && total > 0) {
        s.phase = flxTuneProbe;
        s.cur = Granules{{FLX_GRANULE_TOTAL - kProbeGranules, kProbeGranules, 0}};
        return flxSuccess;
      } else {
        s.tuned_ms = s.nv_ms;
        s.converged = true;
        s.st = flxTunerState{{FLX_GRANULE_TOTAL, 0, 0}, 1, 0, 0, -1, 0};
        finish_stage1(s);
        return flxSuccess;
      }
      const int mask = path_mask & 3;  // RDMA is never available (flxGetPathMask)
      tune::Shares g;
      if (!tune::initialize_shares(prof, mask, &g)) {
        s.tuned_ms = s.nv_ms;
        s.st = flxTunerState{{FLX_GRANULE_TOTAL, 0, 0}, 1, 0, 0, -1, 0};
        finish_stage1(s);
        return flxSuccess;
      }
      for (int p = 0; p < FLX_NUM_PATHS; ++p) s.seed[p] = prof.bandwidth[p];
      s.st = flxTunerState{{g[0], g[1], g[2]}, mask, s.pol.s1.initial_step, 0, -1, 0};
      break;
    }
    case flxTuneProbe: {
      if (!(rep.mask >> flxPathPcie & 1) || rep.ms[flxPathPcie] <= 0) {
        // the probe share rounded to 0 PCIe bytes (message below the alignment)
        s.tuned_ms = s.nv_ms;
        s.st = flxTunerState{{FLX_GRANULE_TOTAL, 0, 0}, 1, 0, 0, -1, 0};
        finish_stage1(s);
        return flxSuccess;
      }
      s.seed[flxPathPcie] = bytes[flxPathPcie] / (rep.ms[flxPathPcie] * 1e-3);
      flxLinkProfile prof{};
      prof.bandwidth[flxPathNvlink] = s.seed[flxPathNvlink];
      prof.bandwidth[flxPathPcie] = s.seed[flxPathPcie];
      prof.contention = 0;  // measured rates already include the interference
      tune::Shares g;
      tune::initialize_shares(prof, nv_pc, &g);
      s.st = flxTunerState{{g[0], g[1], g[2]}, nv_pc, s.pol.s1.initial_step, 0, -1, 0};
      break;
    }
    case flxTuneStage1: {
      flxTuneRecord rec;
      FLX_TRY(tune::tune_step(&s.st, rep, s.pol.s1, &rec));
      s.trace.push_back(rec);
      if (s.st.stability_count >= s.pol.s1.stability_required) {
        s.converged = true;
        s.tuned_ms = total;  // a stable round ran the final split
        finish_stage1(s);
        return flxSuccess;
      }
      break;
    }
    case flxTuneGuard:
      s.tuned_ms = total;
      finish_stage1(s);
      return flxSuccess;
  }
  // next Stage-1 iteration (initial_tune's loop, tuner.py:211-225)
  s.phase = flxTuneStage1;
  if (s.st.active_mask == (1 << flxPathNvlink)) {  // early exit: NVLink alone is left
    flxTuneRecord rec;
    memset(&rec, 0, sizeof(rec));
    rec.iteration = s.st.iteration + 1;
    for (int p = 0; p < FLX_NUM_PATHS; ++p) rec.shares[p] = s.st.shares[p];
    rec.slowest = rec.fastest = rec.source = rec.target = -1;
    rec.step = s.st.step;
    rec.stability_count = s.st.stability_count;
    rec.action = flxTuneEarlyExit;
    s.trace.push_back(rec);
    s.converged = true;
    s.tuned_ms = s.nv_ms;
    finish_stage1(s);
    return flxSuccess;
  }
  if ((int)s.trace.size() >= s.pol.s1.max_iterations) {
    s.phase = flxTuneGuard;  // not converged: measure the final split once
  }
  s.cur = Granules{{s.st.shares[0], s.st.shares[1], s.st.shares[2]}};
  return flxSuccess;
}

flxResult_t AutoTuner::stage2_call(TimingPort& port, Slot& s) {
  if (__builtin_popcount(s.s2_active) < 2) return flxSuccess;  // nothing to balance
  s.s2_calls += 1;
  if (s.s2_calls - stage2_lag() < 1 || s.lagq.empty()) return flxSuccess;
  s.window.push_back(s.lagq.front());  // observe call s2_calls - lag
  s.lagq.pop_front();
  while ((int)s.window.size() > s.pol.s2.window) s.window.pop_front();
  s.s2_observed += 1;
  if (s.s2_observed % s.pol.s2.invocation_period) return flxSuccess;
  std::vector<MeasPtr> win(s.window.begin(), s.window.end());
  FLX_TRY(fetch(port, win));
  std::vector<tune::Report> reps(win.size());
  for (size_t i = 0; i < win.size(); ++i) {
    reps[i].mask = win[i]->mask;
    for (int p = 0; p < FLX_NUM_PATHS; ++p) reps[i].ms[p] = win[i]->ms[p];
  }
  tune::Shares sh{{s.cur[0], s.cur[1], s.cur[2]}};
  flxEvalRecord rec;
  tune::evaluate_apply(reps.data(), (int)reps.size(), s.s2_active, s.pol.s2, &sh, &rec);
  rec.call = s.s2_observed;
  if (rec.moved) s.moves += 1;
  s.n_evals += 1;
  s.cur = Granules{{sh[0], sh[1], sh[2]}};
  s.evals.push_back(rec);
  if (s.evals.size() > kMaxEvals) s.evals.pop_front();
  return flxSuccess;
}

// ---------------------------------------------------------- share cache
namespace {
std::string cache_key(const std::string& scope, int op, int bucket, int ctas) {
  std::ostringstream k;
  k << scope << "/op" << op << "/bucket" << bucket << "/ctas" << ctas;
  return k.str();
}
}  // namespace

bool AutoTuner::cache_lookup(TimingPort& port, int op, int bucket, const Slot& s, Granules* g) {
  const char* path = getenv("FLX_SHARE_CACHE");
  double hit = 0, v[FLX_NUM_PATHS] = {0, 0, 0};
  if (path) {
    std::ifstream in(path);
    const std::string key = cache_key(port.scope(), op, bucket, s.pol.nvlink_ctas);
    std::string line;
    while (std::getline(in, line)) {  // the last entry for a key wins
      std::istringstream ls(line);
      std::string k;
      int a, b, c;
      if (ls >> k >> a >> b >> c && k == key && a >= 0 && b >= 0 && c == 0 &&
          a + b == FLX_GRANULE_TOTAL) {
        hit = 1;
        v[0] = a;
        v[1] = b;
        v[2] = c;
      }
    }
  }
  // every rank must take the same branch: agree on (hit, g) and -(hit, g)
  double ag[8] = {hit, -hit, v[0], -v[0], v[1], -v[1], v[2], -v[2]};
  if (port.agree_max(ag, 8) != flxSuccess) return false;
  for (int i = 0; i < 8; i += 2)
    if (ag[i] != -ag[i + 1]) return false;  // ranks disagree: tune afresh
  if (ag[0] != 1) return false;
  *g = Granules{{(int)ag[2], (int)ag[4], (int)ag[6]}};
  return true;
}

void AutoTuner::cache_store(TimingPort& port, int op, int bucket, const Slot& s) {
  const char* path = getenv("FLX_SHARE_CACHE");
  if (!path || !port.cache_writer()) return;
  FILE* f = fopen(path, "a");
  if (!f) return;
  fprintf(f, "%s %d %d %d\n", cache_key(port.scope(), op, bucket, s.pol.nvlink_ctas).c_str(),
          s.stage1[0], s.stage1[1], s.stage1[2]);
  fclose(f);
}

// ----------------------------------------------------------- per call
flxResult_t AutoTuner::before_call(TimingPort& port, const TunePolicy& pol, int op, size_t bytes,
                                   bool tunable, bool can_measure, int path_mask,
                                   const Granules& fallback, Granules* g, bool* measured) {
  *measured = false;
  *g = fallback;
  const int bucket = size_bucket(bytes);
  if (!tunable) return flxSuccess;
  if (!can_measure) {  // capture / timing off: the current split, no tuning step
    auto it = slots_.find({op, bucket});
    if (it != slots_.end() && it->second.phase != flxTuneIdle) *g = it->second.cur;
    return flxSuccess;
  }
  FLX_TRY(harvest(port));
  if (__builtin_popcount(path_mask & 7) < 2) return flxSuccess;  // one path: nothing to split
  Slot& s = slots_[{op, bucket}];
  if (s.phase == flxTuneIdle) {
    s = Slot();
    s.pol = pol;
    s.repeats = repeat_calls();
    Granules cached;
    if (cache_lookup(port, op, bucket, s, &cached)) {
      s.from_cache = true;
      s.stage1 = cached;
      s.kept = loaded_mask(cached) != 1;
      start_stage2(s, cached);
    } else {
      s.phase = flxTuneBaseline;
      s.cur = Granules{{FLX_GRANULE_TOTAL, 0, 0}};
    }
  }
  s.calls += 1;
  if (s.phase != flxTuneStage2) {
    if (s.round_calls == warm_calls() + s.repeats) {
      FLX_TRY(decide_round(port, s, path_mask));
      if (s.phase == flxTuneStage2) cache_store(port, op, bucket, s);
    }
  }
  if (s.phase != flxTuneStage2) {
    *measured = s.round_calls >= warm_calls();
    s.round_calls += 1;
  } else {
    FLX_TRY(stage2_call(port, s));
    *measured = __builtin_popcount(s.s2_active) >= 2;
  }
  *g = s.cur;
  if (*measured) s.pending = std::make_shared<Meas>();
  return flxSuccess;
}

void AutoTuner::after_call(int op, size_t bytes, uint64_t seq,
                           const std::array<size_t, FLX_NUM_PATHS>& split, bool measured) {
  if (!measured) return;
  auto it = slots_.find({op, size_bucket(bytes)});
  if (it == slots_.end() || !it->second.pending) return;
  Slot& s = it->second;
  MeasPtr m = s.pending;
  s.pending.reset();
  m->seq = seq;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) {
    m->bytes[p] = (double)split[p];
    if (split[p] > 0) m->mask |= 1 << p;
  }
  if (s.phase == flxTuneStage2)
    s.lagq.push_back(m);
  else
    s.round.push_back(m);
  unread_.push_back(m);
}

// ------------------------------------------------------------ queries
bool AutoTuner::current(int op, int bucket, Granules* g) const {
  auto it = slots_.find({op, bucket});
  if (it == slots_.end() || it->second.phase == flxTuneIdle) return false;
  *g = it->second.cur;
  return true;
}

bool AutoTuner::info(int op, int bucket, flxTuneInfo* out) const {
  memset(out, 0, sizeof(*out));
  out->shares[0] = FLX_GRANULE_TOTAL;
  auto it = slots_.find({op, bucket});
  if (it == slots_.end()) return false;
  const Slot& s = it->second;
  out->phase = s.phase;
  out->stage1_iterations = (int)s.trace.size();
  out->converged = s.converged;
  out->kept_tuned = s.kept;
  out->from_cache = s.from_cache;
  out->nvlink_only_ms = s.nv_ms;
  out->tuned_ms = s.tuned_ms;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) {
    out->seed_bandwidth[p] = s.seed[p];
    out->stage1_shares[p] = s.stage1[p];
    out->shares[p] = s.cur[p];
  }
  out->stage2_calls = s.s2_calls;
  out->stage2_evaluations = s.n_evals;
  out->stage2_moves = s.moves;
  out->calls = s.calls;
  return true;
}

int AutoTuner::trace(int op, int bucket, flxTuneRecord* out, int max) const {
  auto it = slots_.find({op, bucket});
  if (it == slots_.end()) return 0;
  const auto& t = it->second.trace;
  const int n = std::min<int>(max, (int)t.size());
  for (int i = 0; i < n; ++i) out[i] = t[i];
  return n;
}

int AutoTuner::evaluations(int op, int bucket, flxEvalRecord* out, int max) const {
  auto it = slots_.find({op, bucket});
  if (it == slots_.end()) return 0;
  const auto& e = it->second.evals;
  const int n = std::min<int>(max, (int)e.size());
  for (int i = 0; i < n; ++i) out[i] = e[e.size() - n + i];
  return n;
}

}  // namespace flx
