"""ctypes face of the native balancer (``include/flexlink_tuner.h``).

Two uses:

* the balancer arithmetic compiled into ``libflexlink.so`` — the same Stage-1
  and Stage-2 decisions the in-library autotuner takes on every communicator —
  callable on any host (no GPU): :func:`initialize_shares`, :func:`tune_step`,
  :class:`NativeBalancer` ...  ``tests/test_tuner_native.py`` replays the
  reference's goldens through them;
* the autotuner's per-bucket state: :func:`tune_info`, :func:`tune_trace`,
  :func:`tune_evaluations` (used by :class:`~paper_2510_15882_b200.comm.Communicator`).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from .comm import _check, load_library
from .links import PathKind

__all__ = ["LinkProfile", "TunerConfigC", "BalancerConfigC", "TunerStateC", "TuneRecordC",
           "EvalRecordC", "TuneInfoC", "profile_from_topology", "maxmin_rates",
           "effective_bandwidths", "initialize_shares", "tuner_state", "tune_step",
           "NativeBalancer", "ACTIONS", "PHASES"]

D3 = ctypes.c_double * 3
I3 = ctypes.c_int * 3

ACTIONS = {0: "stable", 1: "move", 2: "early_exit"}
PHASES = {0: "idle", 1: "baseline", 2: "probe", 3: "stage1", 4: "guard", 5: "stage2"}


class LinkProfile(ctypes.Structure):
    _fields_ = [("bandwidth", D3), ("contention", ctypes.c_int), ("shared_bw", ctypes.c_double)]


class TunerConfigC(ctypes.Structure):
    _fields_ = [("initial_step", ctypes.c_int), ("convergence_threshold", ctypes.c_double),
                ("stability_required", ctypes.c_int), ("max_iterations", ctypes.c_int)]


class BalancerConfigC(ctypes.Structure):
    _fields_ = [("window", ctypes.c_int), ("gap_threshold", ctypes.c_double),
                ("quantum", ctypes.c_int), ("invocation_period", ctypes.c_int)]


class TunerStateC(ctypes.Structure):
    _fields_ = [("shares", I3), ("active_mask", ctypes.c_int), ("step", ctypes.c_int),
                ("stability_count", ctypes.c_int), ("prev_slowest", ctypes.c_int),
                ("iteration", ctypes.c_int)]


class TuneRecordC(ctypes.Structure):
    _fields_ = [("iteration", ctypes.c_int), ("shares", I3), ("durations", D3),
                ("timed_mask", ctypes.c_int), ("imbalance", ctypes.c_double),
                ("slowest", ctypes.c_int), ("fastest", ctypes.c_int), ("step", ctypes.c_int),
                ("stability_count", ctypes.c_int), ("action", ctypes.c_int),
                ("moved", ctypes.c_int), ("source", ctypes.c_int), ("target", ctypes.c_int),
                ("deactivated", ctypes.c_int)]

    def action_string(self) -> str:
        """The reference's TuneRecord.action text (tuner.py:150-175)."""
        if self.action == 0:
            return "stable"
        if self.action == 2:
            return "early_exit"
        s = f"move {self.moved} {PathKind(self.source).short}->{PathKind(self.target).short}"
        if self.deactivated:
            s += f", deactivate {PathKind(self.source).short}"
        return s


class EvalRecordC(ctypes.Structure):
    _fields_ = [("call", ctypes.c_int), ("has_gap", ctypes.c_int), ("gap", ctypes.c_double),
                ("adjusted", ctypes.c_int), ("source", ctypes.c_int), ("target", ctypes.c_int),
                ("granules", ctypes.c_int), ("moved", ctypes.c_int), ("shares", I3)]


class TuneInfoC(ctypes.Structure):
    _fields_ = [("phase", ctypes.c_int), ("stage1_iterations", ctypes.c_int),
                ("converged", ctypes.c_int), ("kept_tuned", ctypes.c_int),
                ("from_cache", ctypes.c_int), ("nvlink_only_ms", ctypes.c_double),
                ("tuned_ms", ctypes.c_double), ("seed_bandwidth", D3),
                ("stage1_shares", I3), ("stage2_calls", ctypes.c_int),
                ("stage2_evaluations", ctypes.c_int), ("stage2_moves", ctypes.c_int),
                ("shares", I3), ("calls", ctypes.c_int)]

    def as_dict(self) -> dict:
        return {"phase": PHASES.get(self.phase, self.phase),
                "stage1_iterations": self.stage1_iterations, "converged": bool(self.converged),
                "kept_tuned": bool(self.kept_tuned), "from_cache": bool(self.from_cache),
                "nvlink_only_ms": round(self.nvlink_only_ms, 4),
                "tuned_ms": round(self.tuned_ms, 4),
                "seed_gbs": [round(b / 1e9, 2) for b in self.seed_bandwidth],
                "stage1_shares": list(self.stage1_shares), "shares": list(self.shares),
                "stage2_calls": self.stage2_calls,
                "stage2_evaluations": self.stage2_evaluations,
                "stage2_moves": self.stage2_moves, "calls": self.calls}


_bound = False


def lib() -> ctypes.CDLL:
    global _bound
    L = load_library()
    if _bound:
        return L
    P, ci = ctypes.POINTER, ctypes.c_int
    sig = {
        "flxTunerDefaults": [P(TunerConfigC), P(BalancerConfigC)],
        "flxMaxMinRates": [ci, P(ctypes.c_double), ci, P(ctypes.c_uint), P(ctypes.c_double),
                           P(ctypes.c_double)],
        "flxEffectiveBandwidths": [P(LinkProfile), ci, P(ctypes.c_double)],
        "flxInitializeShares": [P(LinkProfile), ci, P(ci)],
        "flxTunerStateInit": [P(LinkProfile), ci, P(TunerConfigC), P(TunerStateC)],
        "flxTuneStep": [P(TunerStateC), P(ctypes.c_double), ci, P(TunerConfigC),
                        P(TuneRecordC)],
        "flxBalancerCreate": [P(ci), ci, P(BalancerConfigC), P(ctypes.c_void_p)],
        "flxBalancerObserve": [ctypes.c_void_p, P(ctypes.c_double), ci, P(ci), P(EvalRecordC)],
        "flxBalancerGetShares": [ctypes.c_void_p, P(ci)],
        "flxBalancerDestroy": [ctypes.c_void_p],
        "flxSetAutoTune": [ctypes.c_void_p, ci],
        "flxSetTunerConfig": [ctypes.c_void_p, P(TunerConfigC), P(BalancerConfigC),
                              ctypes.c_size_t],
        "flxSetLinkProfile": [ctypes.c_void_p, P(LinkProfile)],
        "flxGetTuneInfo": [ctypes.c_void_p, ci, ci, P(TuneInfoC)],
        "flxGetTuneTrace": [ctypes.c_void_p, ci, ci, P(TuneRecordC), ci, P(ci)],
        "flxGetTuneEvaluations": [ctypes.c_void_p, ci, ci, P(EvalRecordC), ci, P(ci)],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ci
    _bound = True
    return L


def _mask(paths) -> int:
    m = 0
    for p in paths:
        m |= 1 << int(p)
    return m


def profile_from_topology(topo) -> LinkProfile:
    """TopologySpec -> the native link profile (bandwidth_uni, contention, shared bw)."""
    prof = LinkProfile()
    for p in PathKind:
        if p in topo.links:
            prof.bandwidth[int(p)] = topo.link(p).bandwidth_uni
    prof.contention = 1 if topo.path_contention else 0
    prof.shared_bw = float(topo.shared_interface_bw or 0.0)
    return prof


def maxmin_rates(demands: dict[int, float], groups: list[tuple[set[int], float]]) -> dict:
    flows = list(demands)
    idx = {f: i for i, f in enumerate(flows)}
    d = (ctypes.c_double * max(1, len(flows)))(*[demands[f] for f in flows])
    members = (ctypes.c_uint * max(1, len(groups)))(
        *[sum(1 << idx[f] for f in m) for m, _ in groups])
    caps = (ctypes.c_double * max(1, len(groups)))(*[c for _, c in groups])
    out = (ctypes.c_double * max(1, len(flows)))()
    _check(lib().flxMaxMinRates(len(flows), d, len(groups), members, caps, out),
           "flxMaxMinRates")
    return {f: out[idx[f]] for f in flows}


def effective_bandwidths(topo, paths) -> dict[PathKind, float]:
    out = D3()
    _check(lib().flxEffectiveBandwidths(ctypes.byref(profile_from_topology(topo)), _mask(paths),
                                        out), "flxEffectiveBandwidths")
    return {PathKind(p): out[int(p)] for p in sorted(paths)}


def initialize_shares(topo, paths=None) -> dict[PathKind, int]:
    paths = tuple(sorted(paths)) if paths is not None else topo.present_paths
    out = I3()
    _check(lib().flxInitializeShares(ctypes.byref(profile_from_topology(topo)), _mask(paths), out),
           "flxInitializeShares")
    return {p: out[int(p)] for p in paths}


def config_c(cfg) -> TunerConfigC:
    return TunerConfigC(cfg.initial_step, cfg.convergence_threshold, cfg.stability_required,
                        cfg.max_iterations)


def balancer_config_c(cfg) -> BalancerConfigC:
    return BalancerConfigC(cfg.window, cfg.gap_threshold, cfg.quantum, cfg.invocation_period)


def tuner_state(topo, paths=None, cfg=None) -> TunerStateC:
    paths = tuple(sorted(paths)) if paths is not None else topo.present_paths
    st = TunerStateC()
    c = ctypes.byref(config_c(cfg)) if cfg is not None else None
    _check(lib().flxTunerStateInit(ctypes.byref(profile_from_topology(topo)), _mask(paths), c,
                                   ctypes.byref(st)), "flxTunerStateInit")
    return st


def tune_step(state: TunerStateC, durations: dict, cfg=None) -> TuneRecordC:
    d = D3()
    for k, v in durations.items():
        d[int(k)] = v
    rec = TuneRecordC()
    c = ctypes.byref(config_c(cfg)) if cfg is not None else None
    _check(lib().flxTuneStep(ctypes.byref(state), d, _mask(durations), c, ctypes.byref(rec)),
           "flxTuneStep")
    return rec


@dataclass
class NativeEval:
    call: int
    gap: float | None
    moved: int
    source: int | None
    target: int | None
    shares: dict[int, int]


class NativeBalancer:
    """RuntimeBalancer in C (flxBalancer*): observe one report per call."""

    def __init__(self, shares: dict, active, config=None):
        g = I3(*[int(shares.get(PathKind(p), 0)) for p in range(3)])
        h = ctypes.c_void_p()
        c = ctypes.byref(balancer_config_c(config)) if config is not None else None
        _check(lib().flxBalancerCreate(g, _mask(active), c, ctypes.byref(h)), "flxBalancerCreate")
        self.handle = h
        self.active = tuple(sorted(active))

    def observe(self, durations: dict) -> NativeEval | None:
        d = D3()
        for k, v in durations.items():
            d[int(k)] = v
        ev = ctypes.c_int()
        rec = EvalRecordC()
        _check(lib().flxBalancerObserve(self.handle, d, _mask(durations), ctypes.byref(ev),
                                        ctypes.byref(rec)), "flxBalancerObserve")
        if not ev.value:
            return None
        return NativeEval(rec.call, rec.gap if rec.has_gap else None, rec.moved,
                          rec.source if rec.adjusted else None,
                          rec.target if rec.adjusted else None,
                          {p: rec.shares[p] for p in self.active})

    def shares(self) -> list[int]:
        g = I3()
        _check(lib().flxBalancerGetShares(self.handle, g), "flxBalancerGetShares")
        return list(g)

    def __del__(self):
        try:
            if self.handle:
                lib().flxBalancerDestroy(self.handle)
        except Exception:
            pass
