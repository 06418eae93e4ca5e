/*
 * flexlink_tuner.h — the two-stage load balancer of libflexlink.so.
 *
 * Two layers:
 *
 * 1. Balancer arithmetic (host only; callable without a GPU).  A C
 *    restatement of the reference's tuner and runtime balancer, decision for
 *    decision (goldens: tests/golden/control_plane.json, replayed through
 *    these entry points by tests/test_tuner_native.py):
 *      flxMaxMinRates          <- simcore.maxmin_rates       (simcore.py:100-130)
 *      flxEffectiveBandwidths  <- simcore.effective_bandwidths (simcore.py:242-261)
 *      flxInitializeShares     <- tuner.initialize_shares    (tuner.py:81-107)
 *      flxTuneStep             <- tuner.tune_step            (tuner.py:110-175)
 *      flxBalancer*            <- balancer.TimingWindow / window_gap / evaluate /
 *                                 apply_adjustment / run_dynamic's per-call loop
 *                                 (balancer.py:47-122,163-207)
 *
 * 2. In-library autotune (the paper's "no code changes" drop-in, PAPER.md:5,46,
 *    172,203): every communicator runs Stage 1 on the first calls of each
 *    (collective, size bucket) it sees and Stage 2 on every later call, from
 *    per-path CUDA-event times of the real collective — so an application that
 *    only calls ncclAllReduce / ncclAllGather through libflexlink_nccl.so gets
 *    striped traffic.  Per (op, bucket):
 *      baseline  `repeats` measured calls NVLink-only (also the guard's reference)
 *      probe     `repeats` calls with a small PCIe share: the measured per-link
 *                rates seed initialize_shares (unless flxSetLinkProfile gave a
 *                profile) — "stage 1 a static partition from measured
 *                per-link bandwidth"
 *      stage 1   Algorithm 1 (tune_step) once per round of `warm`+`repeats`
 *                calls, until stable or the iteration cap, then the guard:
 *                keep the tuned split only if it beat NVLink-only
 *      stage 2   RuntimeBalancer on every call, reading per-path times with a
 *                lag of `lag` calls (the host waits only if it runs more than
 *                `lag` calls ahead of the GPU; no per-call synchronisation)
 *    Multi-rank: the per-path times are max-reduced over ranks through the
 *    already-mapped shared host segment at each decision point, so every rank
 *    takes identical decisions.  Buckets the user pinned with flxSetShares are
 *    never tuned.  FLX_AUTOTUNE=0 turns the default off; FLX_AUTOTUNE_MIN_KB
 *    (default 16384) is the smallest per-rank message it tunes;
 *    FLX_SHARE_CACHE=<file> persists Stage-1 results per (GPU, mode, nranks,
 *    collective, bucket, NVLink CTA cap) and later comms start from them.
 */
#ifndef FLEXLINK_TUNER_H_
#define FLEXLINK_TUNER_H_

#include "flexlink.h"

#ifdef __cplusplus
extern "C" {
#endif

/* TopologySpec fields the balancer reads (topo.py:47-123).  bandwidth[p] is
 * LinkSpec.bandwidth_uni in B/s; 0 marks the path absent. */
typedef struct {
  double bandwidth[FLX_NUM_PATHS];
  int contention;   /* TopologySpec.path_contention */
  double shared_bw; /* TopologySpec.shared_interface_bw */
} flxLinkProfile;

/* TunerConfig (tuner.py:35-45) */
typedef struct {
  int initial_step;
  double convergence_threshold;
  int stability_required;
  int max_iterations;
} flxTunerConfig;

/* BalancerConfig (balancer.py:30-44) */
typedef struct {
  int window;
  double gap_threshold;
  int quantum;
  int invocation_period;
} flxBalancerConfig;

/* TunerState (tuner.py:48-55); prev_slowest = -1 for None */
typedef struct {
  int shares[FLX_NUM_PATHS];
  int active_mask;
  int step;
  int stability_count;
  int prev_slowest;
  int iteration;
} flxTunerState;

typedef enum { flxTuneStable = 0, flxTuneMove = 1, flxTuneEarlyExit = 2 } flxTuneAction_t;

/* TuneRecord (tuner.py:58-69); the action string of the reference is
 * "stable" | "move {moved} {source}->{target}[, deactivate {source}]" |
 * "early_exit". */
typedef struct {
  int iteration;
  int shares[FLX_NUM_PATHS];
  double durations[FLX_NUM_PATHS];
  int timed_mask;
  double imbalance;
  int slowest, fastest; /* -1: none (early exit) */
  int step;
  int stability_count;
  int action; /* flxTuneAction_t */
  int moved, source, target, deactivated;
} flxTuneRecord;

/* EvalRecord of one Stage-2 evaluation (balancer.py:135-142) */
typedef struct {
  int call;
  int has_gap;
  double gap;
  int adjusted; /* evaluate() returned an Adjustment */
  int source, target, granules, moved;
  int shares[FLX_NUM_PATHS];
} flxEvalRecord;

/* ---- arithmetic (host only) -------------------------------------------- */
flxResult_t flxTunerDefaults(flxTunerConfig* stage1, flxBalancerConfig* stage2);
/* Progressive-filling max-min fair rates.  group_members[g] is a bit mask of
 * flows (flow i = bit i, nflows <= 32). */
flxResult_t flxMaxMinRates(int nflows, const double* demands, int ngroups,
                           const unsigned* group_members, const double* group_caps,
                           double* rates);
flxResult_t flxEffectiveBandwidths(const flxLinkProfile* topo, int path_mask,
                                   double rates[FLX_NUM_PATHS]);
flxResult_t flxInitializeShares(const flxLinkProfile* topo, int path_mask,
                                int granules[FLX_NUM_PATHS]);
/* The Stage-1 start state: initialize_shares + every present path active. */
flxResult_t flxTunerStateInit(const flxLinkProfile* topo, int path_mask,
                              const flxTunerConfig* config, flxTunerState* state);
/* One Algorithm-1 iteration on a report whose paths are timed_mask. */
flxResult_t flxTuneStep(flxTunerState* state, const double durations[FLX_NUM_PATHS],
                        int timed_mask, const flxTunerConfig* config, flxTuneRecord* record);

/* Stage 2 as a per-call hook (RuntimeBalancer): observe() records a report
 * and, every invocation_period calls, evaluates the window and moves a
 * quantum.  *evaluated = 1 when this call was an evaluation (record filled). */
typedef struct flxBalancer* flxBalancer_t;
flxResult_t flxBalancerCreate(const int shares[FLX_NUM_PATHS], int active_mask,
                              const flxBalancerConfig* config, flxBalancer_t* balancer);
flxResult_t flxBalancerObserve(flxBalancer_t balancer, const double durations[FLX_NUM_PATHS],
                               int timed_mask, int* evaluated, flxEvalRecord* record);
flxResult_t flxBalancerGetShares(flxBalancer_t balancer, int shares[FLX_NUM_PATHS]);
flxResult_t flxBalancerDestroy(flxBalancer_t balancer);

/* ---- in-library autotune (must match on all ranks) -------------------- */
flxResult_t flxSetAutoTune(flxComm_t comm, int enabled);
/* NULL keeps the current value; min_bytes = 0 keeps it too. */
flxResult_t flxSetTunerConfig(flxComm_t comm, const flxTunerConfig* stage1,
                              const flxBalancerConfig* stage2, size_t min_bytes);
/* Seed Stage 1 from this profile (e.g. the probe's measured rates) instead of
 * the in-call probe round.  NULL restores the in-call probe. */
flxResult_t flxSetLinkProfile(flxComm_t comm, const flxLinkProfile* profile);

typedef enum {
  flxTuneIdle = 0,     /* never tuned (pinned, too small, or autotune off) */
  flxTuneBaseline = 1, /* measuring NVLink-only */
  flxTuneProbe = 2,    /* measuring the per-link rates */
  flxTuneStage1 = 3,
  flxTuneGuard = 4,    /* measuring the final Stage-1 split */
  flxTuneStage2 = 5
} flxTunePhase_t;

typedef struct {
  int phase; /* flxTunePhase_t */
  int stage1_iterations;
  int converged;
  int kept_tuned; /* guard: 1 = tuned split kept, 0 = NVLink-only */
  int from_cache;
  double nvlink_only_ms; /* median total, NVLink-only (baseline round) */
  double tuned_ms;       /* median total of the final Stage-1 split */
  double seed_bandwidth[FLX_NUM_PATHS]; /* B/s (per-rank message bytes / path time) */
  int stage1_shares[FLX_NUM_PATHS];
  int stage2_calls, stage2_evaluations, stage2_moves;
  int shares[FLX_NUM_PATHS]; /* what the next call of this bucket uses */
  int calls;                 /* calls of this bucket the tuner has seen */
} flxTuneInfo;

flxResult_t flxGetTuneInfo(flxComm_t comm, flxCollOp_t op, int bucket, flxTuneInfo* info);
/* Stage-1 trace (oldest first); *n = records written. */
flxResult_t flxGetTuneTrace(flxComm_t comm, flxCollOp_t op, int bucket, flxTuneRecord* records,
                            int max_records, int* n);
/* Stage-2 evaluations (oldest first, last 256 kept). */
flxResult_t flxGetTuneEvaluations(flxComm_t comm, flxCollOp_t op, int bucket,
                                  flxEvalRecord* records, int max_records, int* n);

#ifdef __cplusplus
}
#endif
#endif /* FLEXLINK_TUNER_H_ */
