"""Behavioural tests of the linkstripe-compatible control plane.

These restate, test by test, what the reference suite pins for the hot path
(`pkg/tests/test_{units,topo,collectives,staging,tuner,balancer,oracle}.py`
and the acceptance gate `test_acceptance.py`), written against this package.
Exact reference outputs on large corpora are in test_control_golden.py.
"""

import io
import json
import math
import random

import pytest

import paper_2510_15882_b200 as fl
from paper_2510_15882_b200 import stage1, stage2, units
from paper_2510_15882_b200.links import LinkSpec, PathKind, TopologySpec, path_from_name
from paper_2510_15882_b200.pipeline import ExplorationBudgetExceeded, write_trace_jsonl
from paper_2510_15882_b200.striping import report_row, write_reports_csv

MIB = 1 << 20
NV, PC, RD = PathKind.NVLINK, PathKind.PCIE_STAGED, PathKind.RDMA_NIC


def three_path(nv=200e9, pcie=64e9, rdma=25e9, chunk=MIB, **kw):
    return TopologySpec(n_gpus=8, links={
        NV: LinkSpec(NV, nv), PC: LinkSpec(PC, pcie, staging_chunk=chunk),
        RD: LinkSpec(RD, rdma, staging_chunk=chunk)}, **kw)


def flat(nv=100e9, pcie=50e9, lat=0.0, chunk=MIB):
    return TopologySpec(n_gpus=8, links={
        NV: LinkSpec(NV, nv, base_latency=lat),
        PC: LinkSpec(PC, pcie, base_latency=lat, staging_chunk=chunk)})


def report(d, op=fl.CollectiveOp.ALLREDUCE, n=8, size=MIB):
    return fl.PathTimingReport.build(op, n, size, d)


# ------------------------------------------------------------------ units
def test_units_prefix_rules():
    assert units.parse_size("256M") == 256 * MIB
    assert units.parse_size("4MiB") == 4 * MIB
    assert units.parse_bandwidth("64 GB/s") == 64e9
    assert units.parse_bandwidth("800 Gb/s") == 100e9
    assert units.parse_time("5us") == pytest.approx(5e-6)
    assert units.format_size(4 * MIB) == "4M" and units.format_size(1000) == "1000"
    for bad in ("12 parsecs", "abc", "5 XB/s"):
        with pytest.raises(ValueError):
            units.parse_bandwidth(bad)
    with pytest.raises(ValueError):
        units.parse_size("3 furlongs")


# ------------------------------------------------------------------ links
def test_path_order_and_names():
    assert sorted([RD, NV, PC]) == [NV, PC, RD]
    assert path_from_name("PCIe_staged") == PC and path_from_name(" nic ".replace("nic", "rdma")) == RD
    with pytest.raises(ValueError):
        path_from_name("smoke-signals")


def test_linkspec_and_topology_validation():
    with pytest.raises(ValueError):
        LinkSpec(NV, 0)
    with pytest.raises(ValueError):
        LinkSpec(PC, 1e9)  # staged without a chunk
    with pytest.raises(ValueError):
        LinkSpec(NV, 1e9, staging_chunk=4096)
    with pytest.raises(ValueError):
        TopologySpec(n_gpus=1, links={NV: LinkSpec(NV, 1e9)})
    with pytest.raises(ValueError):
        TopologySpec(n_gpus=8, links={PC: LinkSpec(PC, 1e9, staging_chunk=1)})
    with pytest.raises(ValueError):
        TopologySpec(n_gpus=8, links={NV: LinkSpec(NV, 1e9), PC: LinkSpec(PC, 5e9, staging_chunk=1)},
                     path_contention=True, shared_interface_bw=1e9)


def test_presets_and_headroom():
    h800 = fl.preset("H800")
    assert h800.link(NV).bandwidth_uni == 200e9
    assert h800.link(PC).bandwidth_uni == 64e9 and h800.link(RD).bandwidth_uni == 6.25e9
    assert h800.path_contention and not fl.preset("GB300").path_contention
    assert fl.preset("h20").name == "H100"
    got = {k: round(fl.idle_bw_opportunity(fl.preset(k)) * 100)
           for k in ("H800", "H100", "A800", "GB200", "GB300")}
    assert got == {"H800": 32, "H100": 14, "A800": 16, "GB200": 22, "GB300": 33}
    assert round(fl.idle_bw_opportunity(fl.preset("B200")) * 100) == 7
    with pytest.raises(ValueError):
        fl.preset("Z9000")


def test_load_topology_yaml(tmp_path):
    p = tmp_path / "box.yaml"
    p.write_text("name: box\nn_gpus: 4\npath_contention: true\nshared_interface_bw: 64 GB/s\n"
                 "links:\n  nvlink: {bandwidth: 900 GB/s, latency: 5us}\n"
                 "  pcie: {bandwidth: 55 GB/s, latency: 10us, staging_chunk: 1M}\n")
    t = fl.load_topology(str(p))
    assert t.n_gpus == 4 and t.link(PC).staging_chunk == MIB and t.shared_interface_bw == 64e9
    assert fl.topology_for(str(p)).name == "box"
    bad = tmp_path / "bad.yaml"
    bad.write_text("- just a list\n")
    with pytest.raises(ValueError):
        fl.load_topology(str(bad))


def test_probe_yaml_round_trips_through_load_topology(tmp_path):
    from paper_2510_15882_b200.probe import topology_to_yaml

    topo = TopologySpec(n_gpus=8, links={
        NV: LinkSpec(NV, 712.5e9, base_latency=3.25e-6),
        PC: LinkSpec(PC, 49.56e9, base_latency=11.5e-6, staging_chunk=4 * MIB,
                     per_chunk_overhead=2e-6)}, path_contention=True,
        shared_interface_bw=57.2e9, name="probed")
    p = tmp_path / "probed.yaml"
    p.write_text(topology_to_yaml(topo))
    back = fl.load_topology(str(p))
    assert back.name == "probed" and back.n_gpus == 8 and back.path_contention
    for k in (NV, PC):
        assert back.link(k).bandwidth_uni == pytest.approx(topo.link(k).bandwidth_uni, rel=1e-9)
        assert back.link(k).base_latency == pytest.approx(topo.link(k).base_latency, rel=1e-6)
    assert back.link(PC).staging_chunk == 4 * MIB
    assert back.shared_interface_bw == pytest.approx(57.2e9)
    assert fl.initialize_shares(back).get(NV) > 900


def test_restricted_and_scaled_copies():
    t = fl.preset("H800")
    r = t.restricted([NV, PC])
    assert r.present_paths == (NV, PC) and t.present_paths == (NV, PC, RD)
    s = t.with_scaled_bandwidth(PC, 0.5)
    assert s.link(PC).bandwidth_uni == 32e9 and t.link(PC).bandwidth_uni == 64e9


# -------------------------------------------------------------- striping
def test_ring_steps_and_spec():
    assert fl.ring_steps(fl.CollectiveOp.ALLREDUCE, 8) == 14
    assert [fl.ring_steps(fl.CollectiveOp.ALLGATHER, n) for n in (2, 4, 8)] == [1, 3, 7]
    with pytest.raises(ValueError):
        fl.ring_steps(fl.CollectiveOp.ALLREDUCE, 1)
    with pytest.raises(ValueError):
        fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, -1)


def test_share_distribution_invariants_and_move():
    s = fl.ShareDistribution({NV: 900, PC: 100})
    with pytest.raises(ValueError):
        fl.ShareDistribution({NV: 900, PC: 99})
    with pytest.raises(ValueError):
        fl.ShareDistribution({NV: 1001, PC: -1})
    m = s.move(PC, NV, 250)  # clamps to what PCIe holds
    assert m.as_dict() == {NV: 1000, PC: 0} and s.get(PC) == 100
    assert m.loaded_paths == (NV,) and s.fraction(PC) == 0.1


def test_partition_sums_alignment_and_layout():
    for size in (0, 1, 4095, 256 * MIB, 640 * MIB + 3):
        for align in (1, 16, 8 * 4096):
            split = fl.partition(size, {NV: 854, PC: 146}, align)
            assert sum(split.values()) == size
            assert split[PC] % align == 0
    assert fl.partition(256 * MIB, {NV: 854, PC: 146}, 4096) == {NV: 229244928, PC: 39190528}
    from paper_2510_15882_b200.striping import slice_offsets
    off = slice_offsets(1000, {NV: 700, PC: 200, RD: 100})
    assert off == {PC: (0, 200), RD: (200, 100), NV: (300, 700)}
    with pytest.raises(ValueError):
        fl.partition(10, {NV: 0})


def test_model_single_path_and_pcie_pipeline():
    t = flat(100e9, 50e9, lat=1e-6, chunk=MIB)
    spec = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 64 * MIB)
    r = fl.simulate_collective(t, spec, fl.ShareDistribution({NV: 1000}))
    assert r.durations[NV] == pytest.approx(14 * (8 * MIB / 100e9 + 1e-6))
    r2 = fl.simulate_collective(t, spec, fl.ShareDistribution({NV: 500, PC: 500}))
    step = 4 * MIB
    pipe = fl.pipeline_time(step, fl.PipelineSpec(chunk_bytes=MIB, bw_pd2h=50e9, bw_h2cd=50e9))
    assert r2.durations[PC] == pytest.approx(14 * (pipe + 1e-6))
    assert r2.total == max(r2.durations.values())
    zero = fl.simulate_collective(t, fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 0),
                                  fl.ShareDistribution({NV: 1000}))
    assert zero.algbw == 0.0


def test_noise_deterministic_and_buckets():
    t = flat()
    spec = fl.CollectiveSpec(fl.CollectiveOp.ALLGATHER, 8, 32 * MIB)
    sh = fl.ShareDistribution({NV: 800, PC: 200})
    a = fl.simulate_collective(t, spec, sh, noise=fl.NoiseModel(0.1, seed=4))
    b = fl.simulate_collective(t, spec, sh, noise=fl.NoiseModel(0.1, seed=4))
    c = fl.simulate_collective(t, spec, sh, noise=fl.NoiseModel(0.1, seed=5))
    assert a == b and a != c
    table = fl.ShareTable()
    table.set(fl.CollectiveOp.ALLREDUCE, 256 * MIB, sh)
    assert table.get(fl.CollectiveOp.ALLREDUCE, 300 * MIB) == sh
    assert table.get(fl.CollectiveOp.ALLREDUCE, 600 * MIB) is None
    assert fl.size_bucket(256 * MIB) == 28 and fl.size_bucket(640 * MIB) == 29


def test_report_rows_csv():
    r = report({NV: 2.0, PC: 1.0})
    row = report_row(r, fl.ShareDistribution({NV: 900, PC: 100}))
    assert row["total_s"] == 2.0 and row["nvlink_share"] == 900 and row["rdma_s"] == ""
    buf = io.StringIO()
    write_reports_csv([row], buf)
    assert buf.getvalue().startswith("op,n_gpus,size")


# ----------------------------------------------------------------- stage 1
def test_initialize_shares_rules():
    assert fl.initialize_shares(three_path()).as_dict() == {NV: 693, PC: 221, RD: 86}
    t = three_path(pcie=64e9, rdma=25e9, path_contention=True, shared_interface_bw=64e9)
    g = fl.initialize_shares(t).as_dict()
    assert g[NV] > g[PC] > g[RD]
    even = three_path(nv=100e9, pcie=100e9, rdma=100e9)
    g = fl.initialize_shares(even).as_dict()
    assert g[NV] > max(g[PC], g[RD]) and sum(g.values()) == 1000
    with pytest.raises(ValueError):
        fl.initialize_shares(even, paths=(PC, RD))


def test_tune_step_branches():
    cfg = fl.TunerConfig()
    st = stage1.TunerState(shares=fl.ShareDistribution({NV: 700, PC: 200, RD: 100}),
                           active=frozenset({NV, PC, RD}), step=32)
    s1, rec = fl.tune_step(st, report({NV: 1.0, PC: 1.01, RD: 1.02}), cfg)
    assert rec.action == "stable" and s1.stability_count == 1 and s1.shares == st.shares
    s2, rec = fl.tune_step(st, report({NV: 1.0, PC: 2.0, RD: 1.5}), cfg)
    assert rec.action == "move 32 pcie->nvlink" and s2.shares.get(PC) == 168
    s3, rec = fl.tune_step(st, report({NV: 3.0, PC: 2.0, RD: 1.5}), cfg)
    assert rec.action == "move 32 nvlink->rdma"  # NVLink slowest -> fastest gets it
    s4, _ = fl.tune_step(s2, report({NV: 1.0, PC: 1.2, RD: 2.0}), cfg)
    assert s4.step == 16  # bottleneck changed -> halve
    tiny = stage1.TunerState(shares=fl.ShareDistribution({NV: 995, PC: 5}),
                             active=frozenset({NV, PC}), step=32)
    s5, rec = fl.tune_step(tiny, report({NV: 1.0, PC: 3.0}), cfg)
    assert PC not in s5.active and rec.action.endswith("deactivate pcie")
    slow, fast = stage1.slowest_fastest(report({NV: 1.0, PC: 1.0, RD: 1.0}), {NV, PC, RD})
    assert (slow, fast) == (NV, NV)


def test_initial_tune_convergence_cap_early_exit():
    shares, trace = fl.initial_tune(three_path(), fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8,
                                                                    256 * MIB))
    assert trace.converged and trace.records[-1].stability_count == 3
    only = TopologySpec(n_gpus=8, links={NV: LinkSpec(NV, 1e9)})
    s, tr = fl.initial_tune(only, fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, MIB))
    assert tr.records[0].action == "early_exit" and s.as_dict() == {NV: 1000}

    def hostile(state):
        return report({p: (3.0 if p == NV else 1.0) for p in state.active})

    cfg = fl.TunerConfig(max_iterations=25)
    _, tr = fl.initial_tune(three_path(), fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, MIB),
                            cfg, measure=hostile)
    assert tr.iterations <= 25
    buf = io.StringIO()
    stage1.write_trace(tr, buf, "jsonl")
    assert json.loads(buf.getvalue().splitlines()[0])["iteration"] == 1


def _random_topology(seed):
    rng = random.Random(seed)
    nv_bw = rng.uniform(50e9, 400e9)
    links = {NV: LinkSpec(NV, nv_bw, base_latency=rng.uniform(0.0, 50e-6))}
    for kind in (PC, RD):
        if rng.random() < 0.8:
            links[kind] = LinkSpec(kind, nv_bw / rng.uniform(1.0, 10.0),
                                   base_latency=rng.uniform(0.0, 50e-6), staging_chunk=2 * MIB)
    return TopologySpec(n_gpus=rng.choice((2, 4, 8)), links=links), rng.choice(list(fl.CollectiveOp))


def test_acceptance_tuner_near_optimal():
    # reference acceptance 03: tuned time <= 1.05 x brute-force optimum on 20 topologies
    for seed in range(20):
        t, op = _random_topology(seed)
        spec = fl.CollectiveSpec(op, t.n_gpus, 32 * MIB)
        shares, _ = fl.initial_tune(t, spec)
        best = fl.optimal_shares_bruteforce(t, spec, granularity=10)
        assert fl.simulate_collective(t, spec, shares).total / best.best_time <= 1.05


def test_acceptance_symmetric_links_even_split():
    t = TopologySpec(n_gpus=8, links={
        NV: LinkSpec(NV, 100e9, base_latency=1e-6),
        PC: LinkSpec(PC, 100e9, base_latency=1e-6, staging_chunk=64 << 10),
        RD: LinkSpec(RD, 100e9, base_latency=1e-6, staging_chunk=64 << 10)})
    shares, trace = fl.initial_tune(t, fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 256 * MIB))
    assert trace.converged
    assert max(abs(v - 1000 / 3) for v in shares.as_dict().values()) <= 1.0


def test_acceptance_damping_under_alternating_bottleneck():
    t = TopologySpec(n_gpus=8, links={NV: LinkSpec(NV, 100e9),
                                      PC: LinkSpec(PC, 50e9, staging_chunk=MIB),
                                      RD: LinkSpec(RD, 25e9, staging_chunk=MIB)})
    spec = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 64 * MIB)
    calls = {"n": 0}

    def alternating(state):
        calls["n"] += 1
        flip = calls["n"] % 2 == 0
        d = {p: 1.0 for p in state.active}
        if PC in state.active:
            d[PC] = 2.0 if flip else 2.5
        if RD in state.active:
            d[RD] = 2.5 if flip else 2.0
        return report(d)

    _, trace = fl.initial_tune(t, spec, measure=alternating)
    steps = [r.step for r in trace.records]
    assert all(a >= b for a, b in zip(steps, steps[1:]))
    first_one = steps.index(1)
    slow = [r.slowest for r in trace.records]
    flips = sum(1 for a, b in zip(slow[:first_one + 1], slow[1:first_one + 1]) if a != b)
    assert flips <= math.ceil(math.log2(32))


def test_acceptance_offload_identity():
    # speedup over NVLink-only == 1000 / NVLink granules once converged (flat links)
    t = TopologySpec(n_gpus=8, links={NV: LinkSpec(NV, 100e9),
                                      PC: LinkSpec(PC, 50e9, staging_chunk=32 << 10)})
    spec = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 250 * MIB)
    shares, trace = fl.initial_tune(t, spec, fl.TunerConfig(convergence_threshold=0.01))
    assert trace.converged
    base = fl.simulate_collective(t, spec, fl.ShareDistribution({NV: 1000})).total
    tuned = fl.simulate_collective(t, spec, shares).total
    assert abs((base / tuned) / (1000 / shares.get(NV)) - 1) <= 0.01


# ----------------------------------------------------------------- stage 2
def test_balancer_window_median_and_evaluate():
    w = stage2.TimingWindow(3)
    for d in ({NV: 1.0, PC: 1.0}, {NV: 1.0, PC: 9.0}, {NV: 1.0, PC: 1.05}, {NV: 1.0, PC: 1.04}):
        stage2.record(w, report(d))
    assert len(w) == 3
    assert stage2.median_durations(w, [NV, PC]) == {NV: 1.0, PC: 1.05}
    cfg = fl.BalancerConfig()
    sh = fl.ShareDistribution({NV: 900, PC: 100})
    assert fl.evaluate(w, cfg, sh, [NV, PC]) is None  # 5% gap < 10%
    w2 = stage2.TimingWindow(10)
    stage2.record(w2, report({NV: 1.0, PC: 1.5}))
    adj = fl.evaluate(w2, cfg, sh, [NV, PC])
    assert (adj.source, adj.target, adj.granules) == (PC, NV, 10)
    w3 = stage2.TimingWindow(10)
    stage2.record(w3, report({NV: 2.0, PC: 1.0, RD: 1.5}))
    adj = fl.evaluate(w3, cfg, fl.ShareDistribution({NV: 800, PC: 100, RD: 100}), [NV, PC, RD])
    assert (adj.source, adj.target) == (NV, PC)
    single = stage2.TimingWindow(10)
    stage2.record(single, report({NV: 1.0}))
    assert fl.window_gap(single, [NV]) is None


def test_balancer_apply_clamp_and_shift_window():
    sh = fl.ShareDistribution({NV: 995, PC: 5})
    new, moved = fl.apply_adjustment(sh, stage2.Adjustment(PC, NV, 10, 0.5))
    assert moved == 5 and new.get(PC) == 0
    same, moved = fl.apply_adjustment(new, stage2.Adjustment(PC, NV, 10, 0.5))
    assert moved == 0 and same is new
    s = fl.BandwidthShift(at_call=10, path=PC, scale=0.5, duration=2)
    assert [s.applies(c) for c in (9, 10, 11, 12)] == [False, True, True, False]


DRIFT_BOX = TopologySpec(n_gpus=8, links={  # test_acceptance.py:257-262 YAML
    NV: LinkSpec(NV, 400e9, base_latency=5e-6),
    PC: LinkSpec(PC, 100e9, base_latency=10e-6, staging_chunk=MIB)}, name="drift-box")


def test_run_dynamic_drift_spike_no_reactivation():
    spec = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 64 * MIB)
    shares, _ = fl.initial_tune(DRIFT_BOX, spec)
    drift = fl.run_dynamic(DRIFT_BOX, spec, shares, n_calls=150,
                           shifts=(fl.BandwidthShift(31, PC, 0.7),))
    moves = [e for e in drift.evaluations if e.moved]
    assert 1 <= len(moves) <= 5
    assert drift.evaluations[-1].gap < fl.BalancerConfig().gap_threshold
    assert all(e.moved == 0 for e in drift.evaluations[-5:])
    spike = fl.run_dynamic(DRIFT_BOX, spec, shares, n_calls=40,
                           shifts=(fl.BandwidthShift(15, PC, 0.3, duration=1),))
    assert spike.adjustments_made == 0
    h800 = fl.preset("H800").restricted([NV, PC])
    big = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 256 * MIB)
    gone = fl.run_dynamic(h800, big, fl.ShareDistribution({NV: 1000, PC: 0}), n_calls=40,
                          active=(NV,))
    assert gone.final_shares.get(PC) == 0 and gone.adjustments_made == 0
    buf = io.StringIO()
    stage2.write_adjustment_log(drift, buf)
    assert len(buf.getvalue().splitlines()) == 15


def test_runtime_balancer_hook_matches_run_dynamic():
    spec = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 64 * MIB)
    shares, _ = fl.initial_tune(DRIFT_BOX, spec)
    shift = fl.BandwidthShift(31, PC, 0.7)
    ref = fl.run_dynamic(DRIFT_BOX, spec, shares, n_calls=150, shifts=(shift,))
    hook = fl.RuntimeBalancer(shares)
    for call in range(1, 151):
        eff = DRIFT_BOX.with_scaled_bandwidth(PC, 0.7) if shift.applies(call) else DRIFT_BOX
        hook.observe(fl.simulate_collective(eff, spec, hook.shares, paths=hook.active))
    assert hook.shares == ref.final_shares
    assert [e.moved for e in hook.evaluations] == [e.moved for e in ref.evaluations]


# ----------------------------------------------------------------- staging
def test_pipeline_closed_forms_and_double_buffer_gain():
    chunk, bw = 4 * MIB, float(1 << 35)
    t = chunk / bw
    for ovh in (0.0, 2.0 ** -10):
        for k in range(1, 33):
            two = fl.PipelineSpec(chunk_bytes=chunk, bw_pd2h=bw, bw_h2cd=bw,
                                  per_chunk_overhead=ovh, buffers=2)
            one = fl.PipelineSpec(chunk_bytes=chunk, bw_pd2h=bw, bw_h2cd=bw,
                                  per_chunk_overhead=ovh, buffers=1)
            assert fl.pipeline_time(k * chunk, two) == (k + 1) * t + k * ovh
            assert fl.simulate_pipeline_events(k * chunk, two) == (k + 1) * t + k * ovh
            assert fl.pipeline_time(k * chunk, one) == 2 * k * t + k * ovh
    assert fl.pipeline_time(0, two) == 0.0
    with pytest.raises(ValueError):
        fl.PipelineSpec(chunk_bytes=MIB, bw_pd2h=1, bw_h2cd=1, buffers=3)


def test_protocol_counter_safe_binary_stale(tmp_path):
    for buffers in (1, 2):
        for iters in (1, 2, 3, 4):
            assert fl.explore_protocol(iters, buffers=buffers, variant="counter").ok
    stale = fl.explore_protocol(2, buffers=1, variant="binary")
    assert not stale.ok and stale.witness[-1].action == "read"
    assert stale.witness[-1].value != stale.witness[-1].iteration
    assert len(stale.witness) == 8 and stale.verdict == "stale_read"
    assert fl.explore_protocol(1, buffers=1, variant="binary").ok  # needs reuse to fail
    with pytest.raises(ExplorationBudgetExceeded):
        fl.explore_protocol(4, buffers=2, budget=5)
    with pytest.raises(ValueError):
        fl.explore_protocol(0)
    buf = io.StringIO()
    write_trace_jsonl(stale.witness, buf)
    assert json.loads(buf.getvalue().splitlines()[-1])["action"] == "read"


# ----------------------------------------------------------------- optimum
def test_optimum_grid_ties_and_closed_form():
    t = flat(100e9, 50e9)
    spec = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 64 * MIB)
    r = fl.optimal_shares_bruteforce(t, spec, granularity=10)
    assert r.evaluations == 101
    nv = r.best_shares.get(NV)
    for nb in (nv - 10, nv + 10):  # never beaten by its grid neighbours
        if 0 <= nb <= 1000:
            t_nb = fl.simulate_collective(t, spec, fl.ShareDistribution({NV: nb, PC: 1000 - nb}))
            assert t_nb.total >= r.best_time
    with pytest.raises(ValueError):
        fl.optimal_shares_bruteforce(t, spec, granularity=7)
    cf = fl.closed_form_shares({NV: 100e9, PC: 50e9}, {NV: 0.0, PC: 0.0}, 14, 1e9)
    assert cf[NV] == 667 and cf[PC] == 333
    hopeless = fl.closed_form_shares({NV: 100e9, PC: 1e9}, {NV: 0.0, PC: 1.0}, 14, 1e6)
    assert hopeless == {NV: 1000, PC: 0}
    with pytest.raises(ValueError):
        fl.closed_form_shares({NV: 1e9}, {}, 1, 0)
