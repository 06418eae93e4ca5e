// The balancer's arithmetic in C++: Stage 1 (Algorithm 1) and Stage 2
// (windowed medians), restated from the reference decision for decision so the
// in-library autotuner takes exactly the decisions the Python package does.
//
//   maxmin_rates          simcore.py:100-130
//   effective_bandwidths  simcore.py:242-261
//   initialize_shares     tuner.py:81-107
//   slowest_fastest / imbalance / tune_step   tuner.py:110-175
//   median_durations / window_gap / evaluate / apply_adjustment
//                         balancer.py:60-122
//
// Floating-point order follows the Python expressions operand for operand
// (left-to-right sums, (1000*r)/aggregate, (slow-fast)/fast) and the file is
// built with -ffp-contract=off, so every comparison sees the same doubles as
// the reference (tests/test_tuner_native.py replays the goldens).
#include <algorithm>
#include <cstring>
#include <new>

#include "internal.h"
#include "tuner.h"

namespace flx {
namespace tune {

flxTunerConfig default_stage1() { return flxTunerConfig{32, 0.05, 3, 100}; }
flxBalancerConfig default_stage2() { return flxBalancerConfig{10, 0.10, 10, 10}; }

bool valid(const flxTunerConfig& c) {
  return c.initial_step >= 1 && c.convergence_threshold > 0 && c.stability_required >= 1 &&
         c.max_iterations >= 1;
}
bool valid(const flxBalancerConfig& c) {
  return c.window >= 1 && c.gap_threshold > 0 && c.quantum >= 1 && c.invocation_period >= 1;
}

// Progressive filling.  Limits are every flow's own demand (in flow order),
// then the groups; members iterate in ascending flow order like a Python set
// of small ints.
void maxmin_rates(int nflows, const double* demands, int ngroups, const unsigned* members,
                  const double* caps, double* rates) {
  std::vector<unsigned> lim_members;
  std::vector<double> lim_caps;
  for (int f = 0; f < nflows; ++f) {
    rates[f] = 0.0;
    lim_members.push_back(1u << f);
    lim_caps.push_back(demands[f]);
  }
  for (int g = 0; g < ngroups; ++g) {
    lim_members.push_back(members[g]);
    lim_caps.push_back(caps[g]);
  }
  unsigned done = 0;
  const unsigned all = nflows >= 32 ? 0xffffffffu : ((1u << nflows) - 1);
  double level = 0.0;
  while ((done & all) != all) {
    bool found = false;
    double best_room = 0.0;
    unsigned best = 0;
    for (size_t l = 0; l < lim_members.size(); ++l) {
      const unsigned m = lim_members[l] & all;
      const unsigned live = m & ~done;
      if (!live) continue;
      double spent = 0.0;
      for (int f = 0; f < nflows; ++f)
        if ((m >> f & 1u) && (done >> f & 1u)) spent += rates[f];
      const double nlive = (double)__builtin_popcount(live);
      const double room = (lim_caps[l] - spent - level * nlive) / nlive;
      if (!found || room < best_room) {
        found = true;
        best_room = room;
        best = m;
      }
    }
    if (!found) break;
    level += std::max(best_room, 0.0);
    for (int f = 0; f < nflows; ++f)
      if ((best >> f & 1u) && !(done >> f & 1u)) {
        rates[f] = level;
        done |= 1u << f;
      }
  }
}

// Paths that leave the GPU through the shared PCIe interface (simcore.py:19).
constexpr int kContentionGroup = (1 << flxPathPcie) | (1 << flxPathRdma);

void effective_bandwidths(const flxLinkProfile& topo, int mask, double rates[FLX_NUM_PATHS]) {
  for (int p = 0; p < FLX_NUM_PATHS; ++p) rates[p] = (mask >> p & 1) ? topo.bandwidth[p] : 0.0;
  if (!topo.contention) return;
  const int sharing = mask & kContentionGroup;
  if (!sharing) return;
  double demands[FLX_NUM_PATHS];
  int flow_path[FLX_NUM_PATHS];
  int nflows = 0;
  for (int p = 0; p < FLX_NUM_PATHS; ++p)
    if (sharing >> p & 1) {
      flow_path[nflows] = p;
      demands[nflows++] = topo.bandwidth[p];
    }
  const unsigned group = (1u << nflows) - 1;
  double split[FLX_NUM_PATHS];
  maxmin_rates(nflows, demands, 1, &group, &topo.shared_bw, split);
  for (int i = 0; i < nflows; ++i) rates[flow_path[i]] = split[i];
}

bool initialize_shares(const flxLinkProfile& topo, int mask, Shares* out) {
  if (!(mask & (1 << flxPathNvlink))) return false;
  double rates[FLX_NUM_PATHS];
  effective_bandwidths(topo, mask, rates);
  double aggregate = 0.0;  // sum(rates.values()) in path order
  for (int p = 0; p < FLX_NUM_PATHS; ++p)
    if (mask >> p & 1) aggregate += rates[p];
  Shares g{{0, 0, 0}};
  int others = 0;
  for (int p = 1; p < FLX_NUM_PATHS; ++p)
    if (mask >> p & 1) {
      g[p] = (int)(FLX_GRANULE_TOTAL * rates[p] / aggregate);  // int() truncates
      others += g[p];
    }
  g[flxPathNvlink] = FLX_GRANULE_TOTAL - others;
  // single granules from the largest secondary (lowest kind on ties) until
  // NVLink is strictly the largest
  while (true) {
    int donor = -1;
    for (int p = 1; p < FLX_NUM_PATHS; ++p)
      if ((mask >> p & 1) && (donor < 0 || g[p] > g[donor])) donor = p;
    if (donor < 0 || g[flxPathNvlink] > g[donor]) break;
    g[donor] -= 1;
    g[flxPathNvlink] += 1;
  }
  *out = g;
  return true;
}

// slowest (max time, lowest kind on ties) and fastest (min time, lowest kind)
static bool slowest_fastest(const Report& r, int active, int* slow, int* fast) {
  *slow = *fast = -1;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) {
    if (!((active & r.mask) >> p & 1)) continue;
    if (*slow < 0 || r.ms[p] > r.ms[*slow]) *slow = p;
    if (*fast < 0 || r.ms[p] < r.ms[*fast]) *fast = p;
  }
  return *slow >= 0;
}

flxResult_t tune_step(flxTunerState* st, const Report& rep, const flxTunerConfig& cfg,
                      flxTuneRecord* rec) {
  int slow, fast;
  if (!slowest_fastest(rep, st->active_mask, &slow, &fast))
    return fail(flxInvalidArgument, "no active path has a timing sample");
  double gap = 0.0;
  if (__builtin_popcount(st->active_mask & rep.mask) > 1) {
    const double base = rep.ms[fast];
    if (base <= 0) return fail(flxInvalidArgument, "fastest path time must be positive");
    gap = (rep.ms[slow] - base) / base;
  }
  memset(rec, 0, sizeof(*rec));
  rec->source = rec->target = -1;
  const int it = st->iteration + 1;
  if (gap < cfg.convergence_threshold) {
    st->stability_count += 1;
    st->iteration = it;
    rec->action = flxTuneStable;
  } else {
    int step = st->step;
    if (st->prev_slowest >= 0 && slow != st->prev_slowest) step = std::max(step / 2, 1);
    const int toward =
        (slow != flxPathNvlink && (st->active_mask & (1 << flxPathNvlink))) ? flxPathNvlink : fast;
    const int amount = std::min(step, st->shares[slow]);
    st->shares[slow] -= amount;
    st->shares[toward] += amount;
    rec->action = flxTuneMove;
    rec->moved = amount;
    rec->source = slow;
    rec->target = toward;
    if (st->shares[slow] <= 0) {
      st->active_mask &= ~(1 << slow);
      rec->deactivated = 1;
    }
    st->step = step;
    st->stability_count = 0;
    st->prev_slowest = slow;
    st->iteration = it;
  }
  rec->iteration = it;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) {
    rec->shares[p] = st->shares[p];
    rec->durations[p] = (rep.mask >> p & 1) ? rep.ms[p] : 0.0;
  }
  rec->timed_mask = rep.mask;
  rec->imbalance = gap;
  rec->slowest = slow;
  rec->fastest = fast;
  rec->step = st->step;
  rec->stability_count = st->stability_count;
  return flxSuccess;
}

static double median(std::vector<double>& v) {
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  return n % 2 ? v[n / 2] : (v[n / 2 - 1] + v[n / 2]) / 2;
}

bool window_gap(const Report* win, int n, int active, double* gap, int* slow, int* fast) {
  double med[FLX_NUM_PATHS];
  int have = 0;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) {
    if (!(active >> p & 1)) continue;
    std::vector<double> samples;
    for (int i = 0; i < n; ++i)
      if (win[i].mask >> p & 1) samples.push_back(win[i].ms[p]);
    if (!samples.empty()) {
      med[p] = median(samples);
      have |= 1 << p;
    }
  }
  if (__builtin_popcount(have) < 2) return false;
  *slow = *fast = -1;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) {
    if (!(have >> p & 1)) continue;
    if (*slow < 0 || med[p] > med[*slow]) *slow = p;
    if (*fast < 0 || med[p] < med[*fast]) *fast = p;
  }
  if (med[*fast] <= 0) return false;
  *gap = (med[*slow] - med[*fast]) / med[*fast];
  return true;
}

void evaluate_apply(const Report* win, int n, int active, const flxBalancerConfig& cfg,
                    Shares* shares, flxEvalRecord* rec) {
  memset(rec, 0, sizeof(*rec));
  rec->source = rec->target = -1;
  double gap = 0.0;
  int slow = -1, fast = -1;
  rec->has_gap = window_gap(win, n, active, &gap, &slow, &fast);
  rec->gap = rec->has_gap ? gap : 0.0;
  if (rec->has_gap && gap > cfg.gap_threshold) {
    const int toward =
        (slow != flxPathNvlink && (active & (1 << flxPathNvlink))) ? flxPathNvlink : fast;
    rec->adjusted = 1;
    rec->source = slow;
    rec->target = toward;
    rec->granules = cfg.quantum;
    const int moved = std::min(cfg.quantum, (*shares)[slow]);
    if (moved > 0) {
      (*shares)[slow] -= moved;
      (*shares)[toward] += moved;
    }
    rec->moved = moved;
  }
  for (int p = 0; p < FLX_NUM_PATHS; ++p) rec->shares[p] = (*shares)[p];
}

}  // namespace tune
}  // namespace flx

using namespace flx;

// RuntimeBalancer (balancer.py + stage2.py): window of the last `window`
// reports, an evaluation every invocation_period observes.
struct flxBalancer {
  flxBalancerConfig cfg;
  tune::Shares shares;
  int active;
  std::vector<tune::Report> window;  // oldest first
  int calls = 0;
};

extern "C" {

flxResult_t flxTunerDefaults(flxTunerConfig* s1, flxBalancerConfig* s2) {
  if (s1) *s1 = tune::default_stage1();
  if (s2) *s2 = tune::default_stage2();
  return flxSuccess;
}

flxResult_t flxMaxMinRates(int nflows, const double* demands, int ngroups,
                           const unsigned* group_members, const double* group_caps,
                           double* rates) {
  if (nflows < 0 || nflows > 32 || ngroups < 0 || (nflows && (!demands || !rates)) ||
      (ngroups && (!group_members || !group_caps)))
    return fail(flxInvalidArgument, "bad max-min arguments");
  tune::maxmin_rates(nflows, demands, ngroups, group_members, group_caps, rates);
  return flxSuccess;
}

flxResult_t flxEffectiveBandwidths(const flxLinkProfile* topo, int mask,
                                   double rates[FLX_NUM_PATHS]) {
  if (!topo || !rates || mask < 0 || mask > 7) return fail(flxInvalidArgument, "bad arguments");
  tune::effective_bandwidths(*topo, mask, rates);
  return flxSuccess;
}

flxResult_t flxInitializeShares(const flxLinkProfile* topo, int mask,
                                int granules[FLX_NUM_PATHS]) {
  if (!topo || !granules || mask < 0 || mask > 7) return fail(flxInvalidArgument, "bad arguments");
  tune::Shares g;
  if (!tune::initialize_shares(*topo, mask, &g))
    return fail(flxInvalidArgument, "NVLINK must be present to initialize shares");
  for (int p = 0; p < FLX_NUM_PATHS; ++p) granules[p] = g[p];
  return flxSuccess;
}

flxResult_t flxTunerStateInit(const flxLinkProfile* topo, int mask, const flxTunerConfig* cfg,
                              flxTunerState* st) {
  if (!topo || !st) return fail(flxInvalidArgument, "bad arguments");
  const flxTunerConfig c = cfg ? *cfg : tune::default_stage1();
  if (!tune::valid(c)) return fail(flxInvalidArgument, "bad tuner config");
  tune::Shares g;
  if (!tune::initialize_shares(*topo, mask, &g))
    return fail(flxInvalidArgument, "NVLINK must be present to initialize shares");
  memset(st, 0, sizeof(*st));
  for (int p = 0; p < FLX_NUM_PATHS; ++p) st->shares[p] = g[p];
  st->active_mask = mask;
  st->step = c.initial_step;
  st->prev_slowest = -1;
  return flxSuccess;
}

flxResult_t flxTuneStep(flxTunerState* st, const double durations[FLX_NUM_PATHS], int timed_mask,
                        const flxTunerConfig* cfg, flxTuneRecord* rec) {
  if (!st || !durations || !rec) return fail(flxInvalidArgument, "bad arguments");
  const flxTunerConfig c = cfg ? *cfg : tune::default_stage1();
  if (!tune::valid(c)) return fail(flxInvalidArgument, "bad tuner config");
  tune::Report r;
  r.mask = timed_mask & 7;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) r.ms[p] = durations[p];
  return tune::tune_step(st, r, c, rec);
}

flxResult_t flxBalancerCreate(const int shares[FLX_NUM_PATHS], int active_mask,
                              const flxBalancerConfig* cfg, flxBalancer_t* out) {
  if (!shares || !out) return fail(flxInvalidArgument, "bad arguments");
  const flxBalancerConfig c = cfg ? *cfg : tune::default_stage2();
  if (!tune::valid(c)) return fail(flxInvalidArgument, "bad balancer config");
  auto* b = new (std::nothrow) flxBalancer();
  if (!b) return fail(flxSystemError, "out of memory");
  b->cfg = c;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) b->shares[p] = shares[p];
  b->active = active_mask & 7;
  *out = b;
  return flxSuccess;
}

flxResult_t flxBalancerObserve(flxBalancer_t b, const double durations[FLX_NUM_PATHS],
                               int timed_mask, int* evaluated, flxEvalRecord* rec) {
  if (!b || !durations || !evaluated || !rec) return fail(flxInvalidArgument, "bad arguments");
  tune::Report r;
  r.mask = timed_mask & 7;
  for (int p = 0; p < FLX_NUM_PATHS; ++p) r.ms[p] = durations[p];
  b->window.push_back(r);
  if ((int)b->window.size() > b->cfg.window) b->window.erase(b->window.begin());
  b->calls += 1;
  *evaluated = b->calls % b->cfg.invocation_period == 0;
  if (!*evaluated) return flxSuccess;
  tune::evaluate_apply(b->window.data(), (int)b->window.size(), b->active, b->cfg, &b->shares,
                       rec);
  rec->call = b->calls;
  return flxSuccess;
}

flxResult_t flxBalancerGetShares(flxBalancer_t b, int shares[FLX_NUM_PATHS]) {
  if (!b || !shares) return fail(flxInvalidArgument, "bad arguments");
  for (int p = 0; p < FLX_NUM_PATHS; ++p) shares[p] = b->shares[p];
  return flxSuccess;
}

flxResult_t flxBalancerDestroy(flxBalancer_t b) {
  delete b;
  return flxSuccess;
}

}  // extern "C"
