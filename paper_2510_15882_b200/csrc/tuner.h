// Balancer arithmetic shared by the C-ABI hooks (tuner.cpp) and the
// in-library autotuner (autotune.cpp).  Host only.
#pragma once

#include <array>
#include <vector>

#include "../../include/flexlink_tuner.h"

namespace flx {
namespace tune {

using Shares = std::array<int, FLX_NUM_PATHS>;

// One per-path timing report (PathTimingReport.durations): ms[p] valid where
// bit p of mask is set.
struct Report {
  double ms[FLX_NUM_PATHS] = {0, 0, 0};
  int mask = 0;
};

flxTunerConfig default_stage1();
flxBalancerConfig default_stage2();
bool valid(const flxTunerConfig& c);
bool valid(const flxBalancerConfig& c);

void maxmin_rates(int nflows, const double* demands, int ngroups, const unsigned* members,
                  const double* caps, double* rates);
void effective_bandwidths(const flxLinkProfile& topo, int mask, double rates[FLX_NUM_PATHS]);
// false when NVLink is not in `mask` (ValueError in the reference)
bool initialize_shares(const flxLinkProfile& topo, int mask, Shares* out);
// flxInvalidArgument when no active path is timed or the fastest time is <= 0
flxResult_t tune_step(flxTunerState* st, const Report& rep, const flxTunerConfig& cfg,
                      flxTuneRecord* rec);

// Stage 2 over a window of reports (oldest first).
bool window_gap(const Report* win, int n, int active, double* gap, int* slow, int* fast);
// evaluate + apply_adjustment for an evaluation call; fills rec (call left 0)
void evaluate_apply(const Report* win, int n, int active, const flxBalancerConfig& cfg,
                    Shares* shares, flxEvalRecord* rec);

}  // namespace tune
}  // namespace flx
