"""The native balancer (libflexlink.so, csrc/tuner.cpp) takes the reference's
decisions: tests/golden/control_plane.json replayed through the C entry points.

This is the arithmetic the in-library autotuner runs on every communicator
(csrc/autotune.cpp), so an application that only calls ncclAllReduce gets the
reference's Stage 1 (tuner.py:81-226) and Stage 2 (balancer.py:47-207)
decisions, bit for bit.  No GPU needed: these entry points are host code.
"""

import json
from pathlib import Path

import pytest

import paper_2510_15882_b200 as fl
from paper_2510_15882_b200 import stage2
from paper_2510_15882_b200.links import LinkSpec, PathKind, TopologySpec

G = json.loads((Path(__file__).parent / "golden" / "control_plane.json").read_text())


@pytest.fixture(scope="module")
def nt():
    from paper_2510_15882_b200 import comm, tuner_native

    try:
        comm.load_library()
    except Exception as e:  # the CPU suite builds the library first (test_library.py)
        pytest.skip(f"libflexlink.so not built: {e}")
    return tuner_native


def topo(d):
    links = {}
    for k, (bw, lat, chunk, ovh) in d["links"].items():
        kind = PathKind(int(k))
        links[kind] = LinkSpec(kind, bw, base_latency=lat, staging_chunk=chunk,
                               per_chunk_overhead=ovh)
    return TopologySpec(n_gpus=d["n_gpus"], links=links, path_contention=d["contention"],
                        shared_interface_bw=d["shared"], name=d["name"])


def sj(d):
    return {str(int(k)): v for k, v in sorted(d.items())}


TOPOS = [topo(t) for t in G["topologies"]]


def test_maxmin_rates_native(nt):
    for case in G["maxmin"]:
        demands = {int(k): v for k, v in case["demands"].items()}
        groups = [(set(m), c) for m, c in case["groups"]]
        assert {str(k): v for k, v in nt.maxmin_rates(demands, groups).items()} == case["rates"]


def test_effective_bandwidths_and_initial_shares_native(nt):
    for t, eff, init in zip(TOPOS, G["effective"], G["initial_shares"]):
        assert sj(nt.effective_bandwidths(t, t.present_paths)) == eff
        assert sj(nt.initialize_shares(t)) == init


def _replay(nt, t, records, cfg=None):
    """initial_tune's loop (tuner.py:211-225) with the recorded measurements fed
    to the native tune_step; every record must come out identical."""
    st = nt.tuner_state(t, cfg=cfg)
    for want in records:
        if st.active_mask == 1:  # NVLink alone: early exit, no measurement
            assert want["action"] == "early_exit"
            assert sj({PathKind(p): st.shares[p] for p in range(3)
                       if str(p) in want["shares"]}) == want["shares"]
            return
        d = {PathKind(int(k)): v for k, v in want["durations"].items()}
        rec = nt.tune_step(st, d, cfg)
        assert rec.action_string() == want["action"]
        assert rec.iteration == want["iteration"]
        assert rec.imbalance == want["imbalance"]
        assert rec.slowest == want["slowest"] and rec.fastest == want["fastest"]
        assert rec.step == want["step"] and rec.stability_count == want["stability_count"]
        assert {str(p): rec.shares[p] for p in range(3) if str(p) in want["shares"]} \
            == want["shares"]
    return st


def test_tune_step_replays_every_reference_trace(nt):
    assert len(G["tune"]) > 300
    for case in G["tune"]:
        st = _replay(nt, TOPOS[case["topo"]], case["records"])
        if st is not None:
            assert {str(p): st.shares[p] for p in range(3) if str(p) in case["final"]} \
                == case["final"]


def test_tune_step_injected_and_config_traces(nt):
    t3 = topo(G["adv_topo"])
    for key in ("tune_alternating", "tune_hostile"):
        _replay(nt, t3, G[key]["records"])
    cfg = fl.TunerConfig(initial_step=8, convergence_threshold=0.01, stability_required=2,
                         max_iterations=40)
    _replay(nt, fl.preset("H800"), G["tune_cfg"]["records"], cfg)


def test_native_balancer_replays_run_dynamic(nt):
    """run_dynamic (balancer.py:163-207): per-call reports from the golden-pinned
    model, decisions from the native window/evaluate/apply."""
    for case in G["dynamic"]:
        t = topo(case["topo"])
        shifts = tuple(stage2.BandwidthShift(a, PathKind(p), s, d) for a, p, s, d in case["shifts"])
        noise = fl.NoiseModel(*case["noise"]) if case["noise"] else None
        jitter = noise.stream() if noise else None
        spec = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 256 << 20)
        shares = fl.ShareDistribution({PathKind(int(k)): v for k, v in case["shares"].items()})
        active = shares.loaded_paths
        bal = nt.NativeBalancer(shares.as_dict(), active)
        evals = []
        for call in range(1, case["n_calls"] + 1):
            seen = t
            for sh in shifts:
                if sh.applies(call):
                    seen = seen.with_scaled_bandwidth(sh.path, sh.scale)
            cur = fl.ShareDistribution({PathKind(p): g for p, g in enumerate(bal.shares())
                                        if PathKind(p) in active or g})
            rep = fl.simulate_collective(seen, spec, cur, noise=noise, rng=jitter, paths=active)
            ev = bal.observe(rep.durations)
            if ev is not None:
                evals.append({"call": ev.call, "gap": ev.gap, "moved": ev.moved,
                              "source": ev.source, "target": ev.target,
                              "shares": {str(p): g for p, g in sorted(ev.shares.items())}})
        assert evals == case["evals"], case["name"]
        assert {str(int(p)): bal.shares()[int(p)] for p in active} == case["final"]


def test_native_rejects_bad_input(nt):
    from paper_2510_15882_b200.comm import FlexLinkArgumentError

    with pytest.raises(FlexLinkArgumentError):
        nt.initialize_shares(fl.preset("H800"), paths=(PathKind.PCIE_STAGED,))
    st = nt.tuner_state(fl.preset("H800"))
    with pytest.raises(FlexLinkArgumentError):
        nt.tune_step(st, {})
    with pytest.raises(FlexLinkArgumentError):
        nt.tune_step(st, {PathKind.NVLINK: 0.0, PathKind.PCIE_STAGED: 1.0})
