/* Host cost of the balancer's decisions inside libflexlink (csrc/tuner.cpp),
 * beside the reference algorithm's own Python (bench.py control_plane()):
 *   Stage 1: flxTunerStateInit + flxTuneStep to convergence (tuner.py:181-226's
 *            loop) seeded from the H800 three-path profile, path times from a
 *            closed-form model t_p = lat_p + (S * g_p / 1000) / obs_p with
 *            observed rates below the profile's (NVLink 190, PCIe 40, NIC
 *            6.25 GB/s: a box whose PCIe path reaches less than its nominal
 *            rate), the same model bench.py feeds to stage1.initial_tune;
 *   Stage 2: flxBalancerObserve once per call for 1000 calls, PCIe at 0.7x
 *            from call 31 (balancer.py:163-207 with a BandwidthShift).
 * One JSON line: per-decision nanoseconds and the decisions themselves (final
 * shares, iterations), which bench.py checks against the Python's.
 *   gcc -O2 -Iinclude tools/control_cost.c -Lpaper_2510_15882_b200 -lflexlink \
 *       -Wl,-rpath,$PWD/paper_2510_15882_b200 -o tools/bin/control_cost
 */
#include <stdio.h>
#include <time.h>

#include "flexlink_tuner.h"

static const double kLat[FLX_NUM_PATHS] = {5e-6, 1e-5, 1.5e-5};
static const double kObs[FLX_NUM_PATHS] = {190e9, 40e9, 6.25e9};

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + ts.tv_nsec * 1e-9;
}

static void model(const int* shares, int mask, double scale_pcie, double bytes, double* d) {
  for (int p = 0; p < FLX_NUM_PATHS; ++p) {
    d[p] = 0.0;
    if (!(mask >> p & 1)) continue;
    const double bw = p == 1 ? kObs[p] * scale_pcie : kObs[p];
    d[p] = kLat[p] + (bytes * shares[p] / 1000.0) / bw;
  }
}

int main(void) {
  flxLinkProfile topo = {{200e9, 64e9, 6.25e9}, 1, 64e9};
  const int all = 7;
  const double bytes = (double)(256ull << 20) * 2.0 * 7.0 / 8.0;
  flxTunerConfig cfg;
  flxBalancerConfig bcfg;
  flxTunerDefaults(&cfg, &bcfg);

  /* Stage 1 */
  flxTunerState st;
  int iters = 0;
  const int reps1 = 200000;
  double d[FLX_NUM_PATHS];
  flxTuneRecord rec;
  const double t0 = now_s();
  for (int rep = 0; rep < reps1; ++rep) {
    flxTunerStateInit(&topo, all, &cfg, &st);
    iters = 0;
    for (int i = 0; i < cfg.max_iterations; ++i) {
      if (st.active_mask == 1) break;
      model(st.shares, st.active_mask, 1.0, bytes, d);
      flxTuneStep(&st, d, st.active_mask, &cfg, &rec);
      ++iters;
      if (st.stability_count >= cfg.stability_required) break;
    }
  }
  const double stage1_s = (now_s() - t0) / reps1;

  /* Stage 2 */
  const int calls = 1000, reps2 = 2000;
  int final2[FLX_NUM_PATHS] = {0, 0, 0};
  int evals = 0, moves = 0;
  double t_obs = 0.0;
  for (int rep = 0; rep < reps2; ++rep) {
    flxBalancer_t b;
    if (flxBalancerCreate(st.shares, st.active_mask, &bcfg, &b) != flxSuccess) return 1;
    int shares[FLX_NUM_PATHS] = {st.shares[0], st.shares[1], st.shares[2]};
    evals = moves = 0;
    const double t1 = now_s();
    for (int c = 1; c <= calls; ++c) {
      model(shares, st.active_mask, c >= 31 ? 0.7 : 1.0, bytes, d);
      int evaluated = 0;
      flxEvalRecord er;
      flxBalancerObserve(b, d, st.active_mask, &evaluated, &er);
      if (evaluated) {
        ++evals;
        if (er.adjusted) ++moves;
        for (int p = 0; p < FLX_NUM_PATHS; ++p) shares[p] = er.shares[p];
      }
    }
    t_obs += now_s() - t1;
    flxBalancerGetShares(b, final2);
    flxBalancerDestroy(b);
  }
  printf("{\"stage1_us\": %.4f, \"stage1_iterations\": %d, \"tune_step_ns\": %.1f, "
         "\"stage1_shares\": [%d, %d, %d], \"observe_ns\": %.1f, \"stage2_calls\": %d, "
         "\"stage2_evaluations\": %d, \"stage2_moves\": %d, \"stage2_shares\": [%d, %d, %d]}\n",
         stage1_s * 1e6, iters, stage1_s * 1e9 / (iters ? iters : 1), st.shares[0], st.shares[1],
         st.shares[2], t_obs / ((double)reps2 * calls) * 1e9, calls, evals, moves, final2[0],
         final2[1], final2[2]);
  return 0;
}
