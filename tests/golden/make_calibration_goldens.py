"""Generate tests/golden/calibration.json by running the REFERENCE's calibration
(`linkstripe.bench.calibrate` / `build_calibrated_topology` / `reproduce_reference`,
pkg/src/linkstripe/bench.py:111-355) on its own H800 table and on seeded
synthetic row sets.  Run in the build container (needs /root/reference):

    python tests/golden/make_calibration_goldens.py

tests/test_calibration.py replays the same inputs through
paper_2510_15882_b200.calibration.  The GPU box only reads the JSON."""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "calibration.json"
MIB = 1 << 20


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


def rows_json(rows):
    return [[r.op.value, r.n_gpus, r.size, r.mode, r.algbw, r.impr_pct, r.pcie_load,
             r.rdma_load] for r in rows]


def main():
    sys.path.insert(0, str(REF))
    import linkstripe.bench as B
    from linkstripe.collectives import CollectiveOp

    out = {"h800_rows": rows_json(B.H800_MEASUREMENTS),
           "h800_fit": fit_json(B.calibrate(B.H800_MEASUREMENTS))}
    cells = []
    for mode in (B.MODE_PCIE_ONLY, B.MODE_PCIE_RDMA):
        for c in B.reproduce_reference(mode=mode):
            cells.append([c.op.value, c.n_gpus, c.size, c.mode, c.published_bw, c.simulated_bw,
                          c.published_offload, c.simulated_offload, c.baseline_residual])
    out["reproduce"] = cells
    topos = []
    cal = B.calibrate(B.H800_MEASUREMENTS)
    for (op, n) in sorted(cal.nvlink, key=lambda k: (k[0].value, k[1])):
        for mode in (B.MODE_BASELINE, B.MODE_PCIE_ONLY, B.MODE_PCIE_RDMA):
            t = B.build_calibrated_topology(cal, op, n, mode)
            topos.append([op.value, n, mode, t.name, t.n_gpus, t.path_contention,
                          {str(int(k)): [v.bandwidth_uni, v.base_latency, v.staging_chunk,
                                         v.per_chunk_overhead]
                           for k, v in sorted(t.links.items())}])
    out["topologies"] = topos
    out["offload_identity"] = B.check_offload_identity()
    rng = random.Random(20261019)
    synth = []
    for case in range(60):
        op = rng.choice([CollectiveOp.ALLREDUCE, CollectiveOp.ALLGATHER])
        n = rng.choice([2, 4, 8])
        nsizes = rng.choice([1, 2, 3, 5])
        bw = rng.uniform(50, 900)
        lat = rng.uniform(0, 3e-5) if case % 7 else 0.0
        rows = []
        for mib in sorted(rng.sample([1, 2, 4, 8, 16, 32, 64, 128, 256, 512], nsizes)):
            size = mib * MIB
            steps = B.ring_steps(op, n)
            t = steps * (size / n / (bw * 1e9) + lat)
            meas = size / t / 1e9 * rng.uniform(0.97, 1.03)
            if case % 11 == 5:  # bandwidth falling with size: negative slope branch
                meas = bw * (1.0 - 0.05 * mib / 512)
            rows.append(B.MeasuredRow(op, n, size, B.MODE_BASELINE, meas))
            pl = rng.uniform(0, 30)
            rows.append(B.MeasuredRow(op, n, size, B.MODE_PCIE_ONLY, meas * 1.1, 0, pl))
            rows.append(B.MeasuredRow(op, n, size, B.MODE_PCIE_RDMA, meas * 1.15, 0, pl * 0.7,
                                      rng.uniform(0, 10)))
        try:
            synth.append({"rows": rows_json(rows), "fit": fit_json(B.calibrate(rows))})
        except B.CalibrationError as e:
            synth.append({"rows": rows_json(rows), "error": str(e)})
    # the reference's own rejection cases (test_bench.py:74-99 shapes)
    bad = [[B.MeasuredRow(CollectiveOp.ALLREDUCE, 2, 32 * MIB, B.MODE_BASELINE, 100),
            B.MeasuredRow(CollectiveOp.ALLREDUCE, 2, 64 * MIB, B.MODE_BASELINE, 1e9)],
           [B.MeasuredRow(CollectiveOp.ALLREDUCE, 2, 32 * MIB, B.MODE_PCIE_ONLY, 100, 0, 10)],
           [B.MeasuredRow(CollectiveOp.ALLREDUCE, 2, 32 * MIB, B.MODE_BASELINE, 100),
            B.MeasuredRow(CollectiveOp.ALLREDUCE, 2, 32 * MIB, B.MODE_PCIE_ONLY, 100, 0, 100)]]
    for rows in bad:
        try:
            synth.append({"rows": rows_json(rows), "fit": fit_json(B.calibrate(rows))})
        except B.CalibrationError as e:
            synth.append({"rows": rows_json(rows), "error": str(e)})
    out["synthetic"] = synth
    OUT.write_text(json.dumps(out))
    print(f"wrote {OUT} ({len(synth)} synthetic cases)")


if __name__ == "__main__":
    main()
