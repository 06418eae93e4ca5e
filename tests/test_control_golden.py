"""Control-plane parity: replay the reference's recorded outputs through this package.

tests/golden/control_plane.json was produced by tests/golden/make_goldens.py
importing the unmodified reference (linkstripe).  Every float is compared
exactly: the restatement performs the same arithmetic in the same order.
"""

import json
from pathlib import Path

import pytest

import paper_2510_15882_b200 as fl
from paper_2510_15882_b200 import stage2, units
from paper_2510_15882_b200.links import LinkSpec, PathKind, TopologySpec

G = json.loads((Path(__file__).parent / "golden" / "control_plane.json").read_text())


def topo(d):
    links = {}
    for k, (bw, lat, chunk, ovh) in d["links"].items():
        kind = PathKind(int(k))
        links[kind] = LinkSpec(kind, bw, base_latency=lat, staging_chunk=chunk,
                               per_chunk_overhead=ovh)
    return TopologySpec(n_gpus=d["n_gpus"], links=links, path_contention=d["contention"],
                        shared_interface_bw=d["shared"], name=d["name"])


def kd(d):
    return {PathKind(int(k)): v for k, v in d.items()}


def sj(d):
    return {str(int(k)): v for k, v in sorted(d.items())}


TOPOS = [topo(t) for t in G["topologies"]]


def test_partition_matches_reference():
    for case in G["partition"]:
        got = fl.partition(case["size"], kd(case["granules"]), case["alignment"])
        assert sj(got) == case["out"], case


def test_partition_native_c_matches_reference(oracle_lib):
    for case in G["partition"]:
        g = [case["granules"].get(str(i), 0) for i in range(3)]
        want = [case["out"].get(str(i), 0) for i in range(3)]
        assert oracle_lib.partition(case["size"], g, case["alignment"]) == want


def test_ring_steps_buckets_presets_headroom():
    for op, n, steps in G["ring_steps"]:
        assert fl.ring_steps(fl.CollectiveOp(op), n) == steps
    for size, bucket in G["size_bucket"]:
        assert fl.size_bucket(size) == bucket
    for name, d in G["presets"].items():
        t = fl.preset(name)
        assert topo(d) == fl.TopologySpec(t.n_gpus, t.links, t.path_contention,
                                          t.shared_interface_bw, d["name"])
    for name, v in G["idle"].items():
        assert fl.idle_bw_opportunity(fl.preset(name)) == v


def test_maxmin_rates():
    for case in G["maxmin"]:
        demands = {int(k): v for k, v in case["demands"].items()}
        groups = [(set(m), c) for m, c in case["groups"]]
        got = fl.maxmin_rates(demands, groups)
        assert {str(k): v for k, v in got.items()} == case["rates"]


def test_effective_bandwidths_and_initial_shares():
    for t, eff, init in zip(TOPOS, G["effective"], G["initial_shares"]):
        assert sj(fl.effective_bandwidths(t, t.present_paths)) == eff
        assert sj(fl.initialize_shares(t).as_dict()) == init


def _noise(n):
    return None if n is None else fl.NoiseModel(n[0], seed=n[1])


def test_simulate_collective_model():
    for case in G["simulate"]:
        t = TOPOS[case["topo"]]
        spec = fl.CollectiveSpec(fl.CollectiveOp(case["op"]), case["n"], case["size"])
        rep = fl.simulate_collective(t, spec, fl.ShareDistribution(kd(case["shares"])),
                                     noise=_noise(case["noise"]))
        assert sj(rep.durations) == case["durations"]
        assert rep.total == case["total"] and rep.algbw == case["algbw"]


def _records(trace):
    return [{"iteration": r.iteration, "action": r.action, "imbalance": r.imbalance,
             "slowest": None if r.slowest is None else int(r.slowest),
             "fastest": None if r.fastest is None else int(r.fastest), "step": r.step,
             "stability_count": r.stability_count, "shares": sj(r.shares),
             "durations": sj(r.durations)} for r in trace.records]


def test_initial_tune_traces_match_reference():
    assert len(G["tune"]) > 300
    for case in G["tune"]:
        t = TOPOS[case["topo"]]
        spec = fl.CollectiveSpec(fl.CollectiveOp(case["op"]), case["n"], case["size"])
        final, trace = fl.initial_tune(t, spec, noise=_noise(case["noise"]))
        assert sj(final.as_dict()) == case["final"]
        assert trace.converged == case["converged"]
        assert _records(trace) == case["records"]


def test_initial_tune_injected_measurements():
    t3 = topo(G["adv_topo"])
    spec = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 64 << 20)
    calls = {"n": 0}

    def alternating(state):
        calls["n"] += 1
        flip = calls["n"] % 2 == 0
        d = {p: 1.0 for p in state.active}
        if PathKind.PCIE_STAGED in state.active:
            d[PathKind.PCIE_STAGED] = 2.0 if flip else 2.5
        if PathKind.RDMA_NIC in state.active:
            d[PathKind.RDMA_NIC] = 2.5 if flip else 2.0
        return fl.PathTimingReport.build(spec.op, 8, spec.size, d)

    def hostile(state):
        d = {p: (3.0 if p == PathKind.NVLINK else 1.0) for p in state.active}
        return fl.PathTimingReport.build(spec.op, 8, spec.size, d)

    for fn, key in ((alternating, "tune_alternating"), (hostile, "tune_hostile")):
        final, trace = fl.initial_tune(t3, spec, measure=fn)
        assert sj(final.as_dict()) == G[key]["final"]
        assert _records(trace) == G[key]["records"]
    cfg = fl.TunerConfig(initial_step=8, convergence_threshold=0.01, stability_required=2,
                         max_iterations=40)
    final, trace = fl.initial_tune(fl.preset("H800"), fl.CollectiveSpec(
        fl.CollectiveOp.ALLGATHER, 4, 128 << 20), cfg, alignment=4096)
    assert _records(trace) == G["tune_cfg"]["records"]


def test_run_dynamic_matches_reference():
    for case in G["dynamic"]:
        t = topo(case["topo"])
        shifts = tuple(stage2.BandwidthShift(a, PathKind(p), s, d) for a, p, s, d in case["shifts"])
        noise = fl.NoiseModel(*case["noise"]) if case["noise"] else None
        spec = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 256 << 20)
        res = fl.run_dynamic(t, spec, fl.ShareDistribution(kd(case["shares"])),
                             n_calls=case["n_calls"], shifts=shifts, noise=noise)
        assert sj(res.final_shares.as_dict()) == case["final"], case["name"]
        assert [r.total for r in res.reports] == case["totals"]
        got = [{"call": e.call, "gap": e.gap, "moved": e.moved,
                "source": None if e.adjustment is None else int(e.adjustment.source),
                "target": None if e.adjustment is None else int(e.adjustment.target),
                "shares": sj(e.shares)} for e in res.evaluations]
        assert got == case["evals"], case["name"]


def test_run_dynamic_measure_seam_reproduces_model():
    # the new measure= seam fed by the model itself gives the same run
    case = G["dynamic"][0]
    t = topo(case["topo"])
    shift = stage2.BandwidthShift(31, PathKind.PCIE_STAGED, 0.7)
    spec = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 256 << 20)

    def measure(call, shares):
        eff = t.with_scaled_bandwidth(PathKind.PCIE_STAGED, 0.7) if shift.applies(call) else t
        return fl.simulate_collective(eff, spec, shares, paths=(0, 1))

    res = fl.run_dynamic(t, spec, fl.ShareDistribution(kd(case["shares"])), n_calls=150,
                         measure=measure)
    assert sj(res.final_shares.as_dict()) == case["final"]


def test_pipeline_model_and_events():
    for c in G["pipeline"]:
        spec = fl.PipelineSpec(chunk_bytes=c["chunk"], bw_pd2h=c["a"], bw_h2cd=c["b"],
                               per_chunk_overhead=c["ovh"], buffers=c["buffers"])
        assert fl.pipeline_time(c["total"], spec) == c["closed"]
        assert fl.simulate_pipeline_events(c["total"], spec) == c["events"]


def test_protocol_exploration():
    for c in G["protocol"]:
        v = fl.explore_protocol(c["iterations"], buffers=c["buffers"], variant=c["variant"])
        assert v.ok == c["ok"] and v.states_explored == c["states"]
        assert v.deadlocks == c["deadlocks"]
        got = None if v.witness is None else [a.to_dict() for a in v.witness]
        assert got == c["witness"]


def test_optimum_references():
    for c in G["bruteforce"]:
        t = TOPOS[c["topo"]]
        spec = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, t.n_gpus, 64 << 20)
        r = fl.optimal_shares_bruteforce(t, spec, granularity=c["granularity"])
        assert sj(r.best_shares.as_dict()) == c["best"]
        assert r.best_time == c["time"] and r.evaluations == c["evaluations"]
    for c in G["closed_form"]:
        bws, lats = kd(c["bw"]), kd(c["lat"])
        if "error" in c["out"]:
            with pytest.raises(ValueError):
                fl.closed_form_shares(bws, lats, c["steps"], c["volume"])
        else:
            assert sj(fl.closed_form_shares(bws, lats, c["steps"], c["volume"])) == c["out"]


def test_units():
    for s, v in G["units"]["size"]:
        assert units.parse_size(s) == v
    for s, v in G["units"]["bw"]:
        assert units.parse_bandwidth(s) == v
    for s, v in G["units"]["time"]:
        assert units.parse_time(s) == v
