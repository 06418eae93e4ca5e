"""Alpha-beta calibration (paper_2510_15882_b200.calibration) reproduces the
reference's `calibrate` / `build_calibrated_topology` (bench.py:111-227) on its
H800 table and on 63 seeded synthetic row sets, float for float, and the
calibrated topology drives Stage 1 to the reference's reproduce_reference cells
(bench.py:318-355).  tests/golden/calibration.json: make_calibration_goldens.py."""

import json
from pathlib import Path

import pytest

from paper_2510_15882_b200 import calibration as C
from paper_2510_15882_b200.links import PathKind
from paper_2510_15882_b200.stage1 import TunerConfig, initial_tune
from paper_2510_15882_b200.striping import (CollectiveOp, CollectiveSpec, ShareDistribution,
                                            simulate_collective)

G = json.loads((Path(__file__).parent / "golden" / "calibration.json").read_text())


def rows(js):
    return [C.MeasuredRow(CollectiveOp(op), n, size, mode, bw, impr, pl, rl)
            for op, n, size, mode, bw, impr, pl, rl in js]


def fit_json(cal):
    return {
        "nvlink": [[op.value, n, f.bandwidth, f.latency,
                    [[s, r] for s, r in sorted(f.residuals.items())]]
                   for (op, n), f in sorted(cal.nvlink.items(), key=lambda kv: (kv[0][0].value,
                                                                                 kv[0][1]))],
        "secondary": [[op.value, n, mode, {str(int(k)): v for k, v in sorted(d.items())}]
                      for (op, n, mode), d in sorted(cal.secondary.items(),
                                                     key=lambda kv: (kv[0][0].value, kv[0][1],
                                                                     kv[0][2]))],
    }


def test_h800_table_is_the_references():
    assert rows(G["h800_rows"]) == list(C.H800_MEASUREMENTS)


def test_h800_fit_matches_reference_exactly():
    assert fit_json(C.calibrate(C.H800_MEASUREMENTS)) == G["h800_fit"]
    assert C.check_offload_identity() == G["offload_identity"]


def test_synthetic_fits_and_rejections_match_reference():
    for case in G["synthetic"]:
        rs = rows(case["rows"])
        if "error" in case:
            with pytest.raises(C.CalibrationError) as e:
                C.calibrate(rs)
            assert str(e.value) == case["error"]
        else:
            assert fit_json(C.calibrate(rs)) == case["fit"]


def test_calibrated_topologies_match_reference():
    cal = C.calibrate(C.H800_MEASUREMENTS)
    for op, n, mode, name, ng, cont, links in G["topologies"]:
        t = C.build_calibrated_topology(cal, CollectiveOp(op), n, mode)
        assert (t.name, t.n_gpus, t.path_contention) == (name, ng, cont)
        assert {str(int(k)): [v.bandwidth_uni, v.base_latency, v.staging_chunk,
                              v.per_chunk_overhead] for k, v in sorted(t.links.items())} == links


def test_calibrated_topology_seeds_stage1_to_the_reference_cells():
    """reproduce_reference: calibrate, build the topology, Stage 1, simulate."""
    cal = C.calibrate(C.H800_MEASUREMENTS)
    for op, n, size, mode, pub_bw, sim_bw, pub_off, sim_off, resid in G["reproduce"]:
        op = CollectiveOp(op)
        topo = C.build_calibrated_topology(cal, op, n, mode)
        spec = CollectiveSpec(op, n, size)
        shares, _ = initial_tune(topo, spec, TunerConfig())
        rep = simulate_collective(topo, spec, shares)
        assert rep.algbw / 1e9 == sim_bw
        assert (1000 - shares.get(PathKind.NVLINK)) / 10.0 == sim_off
        assert cal.nvlink[(op, n)].residuals[size] == resid
    base = C.build_calibrated_topology(cal, CollectiveOp.ALLREDUCE, 8, C.MODE_BASELINE)
    nv = simulate_collective(base, CollectiveSpec(CollectiveOp.ALLREDUCE, 8, 256 << 20),
                             ShareDistribution({PathKind.NVLINK: 1000}))
    assert abs(nv.algbw / 1e9 - 107) / 107 < 0.05  # the fit reproduces its baseline row
