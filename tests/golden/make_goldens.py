"""Generate tests/golden/control_plane.json by running the REFERENCE (linkstripe).

Run in the build container, where /root/reference exists:

    python tests/golden/make_goldens.py

It imports the unmodified reference package from /root/reference/pkg/src and
records its outputs on a fixed corpus of inputs: partition splits, ring steps,
shared-interface rates, Stage-1 initial shares and full tuning traces (model and
injected measurements), Stage-2 evaluations under drift/spike/noise, pipeline
makespans, protocol exploration verdicts, optimum/closed-form splits, unit
parsing.  tests/test_control_golden.py replays the same inputs through
paper_2510_15882_b200 and demands identical results (floats compared exactly).
The GPU box never runs this script; it only reads the committed JSON.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "control_plane.json"
MIB = 1 << 20


def topo_to_json(t):
    return {"n_gpus": t.n_gpus, "contention": t.path_contention,
            "shared": t.shared_interface_bw, "name": t.name,
            "links": {str(int(k)): [v.bandwidth_uni, v.base_latency, v.staging_chunk,
                                    v.per_chunk_overhead] for k, v in sorted(t.links.items())}}


def topo_from_json(ls, d):
    links = {}
    for k, (bw, lat, chunk, ovh) in d["links"].items():
        kind = ls.PathKind(int(k))
        links[kind] = ls.LinkSpec(kind, bw, base_latency=lat, staging_chunk=chunk,
                                  per_chunk_overhead=ovh)
    return ls.TopologySpec(n_gpus=d["n_gpus"], links=links, path_contention=d["contention"],
                           shared_interface_bw=d["shared"], name=d["name"])


def g2j(shares_dict):
    return {str(int(k)): v for k, v in sorted(shares_dict.items())}


def records_to_json(trace):
    return [{"iteration": r.iteration, "action": r.action, "imbalance": r.imbalance,
             "slowest": None if r.slowest is None else int(r.slowest),
             "fastest": None if r.fastest is None else int(r.fastest), "step": r.step,
             "stability_count": r.stability_count, "shares": g2j(r.shares),
             "durations": {str(int(k)): v for k, v in sorted(r.durations.items())}}
            for r in trace.records]


def random_topo(ls, rng, contention=None):
    nv = rng.uniform(50e9, 900e9)
    links = {ls.PathKind.NVLINK: ls.LinkSpec(ls.PathKind.NVLINK, nv,
                                             base_latency=rng.uniform(0, 40e-6))}
    for kind in (ls.PathKind.PCIE_STAGED, ls.PathKind.RDMA_NIC):
        if rng.random() < 0.8:
            links[kind] = ls.LinkSpec(kind, nv / rng.uniform(1.0, 20.0),
                                      base_latency=rng.uniform(0, 40e-6),
                                      staging_chunk=rng.choice([64 << 10, MIB, 4 * MIB]),
                                      per_chunk_overhead=rng.choice([0.0, 1e-6, 3e-6]))
    cont = rng.random() < 0.5 if contention is None else contention
    shared = 0.0
    if cont:
        pcie = links.get(ls.PathKind.PCIE_STAGED)
        shared = (pcie.bandwidth_uni if pcie else nv / 10) * rng.uniform(1.0, 1.5)
    return ls.TopologySpec(n_gpus=rng.choice((2, 4, 8)), links=links, path_contention=cont,
                           shared_interface_bw=shared, name="rand")


def main():
    sys.path.insert(0, str(REF))
    import linkstripe as ls
    from linkstripe import balancer, bench, staging, tuner, units

    P = ls.PathKind
    rng = random.Random(20251015)
    out: dict = {"source": "linkstripe 0.1.0 (/root/reference/pkg/src), imported unmodified"}

    # ---- partition (collectives.py:93-114)
    cases = [(0, {0: 1000}, 1), (1, {0: 999, 1: 1}, 1), (256 * MIB, {0: 854, 1: 146}, 1),
             (256 * MIB, {0: 854, 1: 146}, 4096), (256 * MIB, {0: 854, 1: 146}, 8 * 4096),
             (640 * MIB, {0: 861, 1: 114, 2: 25}, 8 * 4096), (12345, {0: 0, 1: 500, 2: 500}, 7),
             (5000, {1: 1000}, 16), (4095, {0: 10, 1: 990}, 4096)]
    for _ in range(300):
        k = rng.randint(1, 3)
        g = [rng.randint(0, 1000) for _ in range(k)]
        g[0] += 1000 - sum(g) if sum(g) <= 1000 else 0
        if sum(g) != 1000 or min(g) < 0:
            a = rng.randint(0, 1000)
            b = rng.randint(0, 1000 - a)
            g = [1000 - a - b, a, b][:3]
        size = rng.choice([rng.randint(0, 10**6), rng.randint(0, 1 << 34), 256 * MIB])
        align = rng.choice([1, 2, 16, 4096, 8 * 4096, 3])
        cases.append((size, {i: g[i] for i in range(len(g))}, align))
    out["partition"] = [
        {"size": s, "granules": {str(k): v for k, v in g.items()}, "alignment": a,
         "out": {str(int(k)): v for k, v in
                 ls.partition(s, {P(k): v for k, v in g.items()}, a).items()}}
        for s, g, a in cases]

    # ---- ring steps / buckets / presets / headroom
    out["ring_steps"] = [[op.value, n, ls.ring_steps(op, n)] for op in ls.CollectiveOp
                         for n in (2, 3, 4, 8, 16)]
    out["size_bucket"] = [[s, ls.size_bucket(s)] for s in
                          (0, 1, 2, 3, 4095, 4096, 256 * MIB, 640 * MIB, (1 << 40) + 5)]
    out["presets"] = {name: topo_to_json(ls.preset(name)) for name in
                      ("H800", "H100", "H200", "H20", "A800", "GB200", "GB300")}
    out["idle"] = {name: ls.idle_bw_opportunity(ls.preset(name)) for name in
                   ("H800", "H100", "A800", "GB200", "GB300")}

    # ---- max-min fair split
    mm = []
    for _ in range(60):
        nflows = rng.randint(1, 5)
        demands = {i: rng.uniform(1, 100) for i in range(nflows)}
        groups = []
        for _ in range(rng.randint(0, 3)):
            members = sorted(rng.sample(range(nflows), rng.randint(1, nflows)))
            groups.append([members, rng.uniform(1, 150)])
        rates = ls.maxmin_rates(demands, [(set(m), c) for m, c in groups])
        mm.append({"demands": {str(k): v for k, v in demands.items()}, "groups": groups,
                   "rates": {str(k): v for k, v in rates.items()}})
    out["maxmin"] = mm

    # ---- topologies used below
    topos = [ls.preset(n) for n in ("H800", "H100", "A800", "GB200", "GB300")]
    topos += [ls.preset("H800").restricted(bench.MODE_PATHS[m]) for m in
              (bench.MODE_PCIE_ONLY, bench.MODE_BASELINE)]
    topos += [random_topo(ls, rng) for _ in range(40)]
    out["topologies"] = [topo_to_json(t) for t in topos]
    out["effective"] = [{str(int(k)): v for k, v in
                         ls.effective_bandwidths(t, t.present_paths).items()} for t in topos]
    out["initial_shares"] = [g2j(ls.initialize_shares(t).as_dict()) for t in topos]

    # ---- simulate_collective + initial_tune traces
    sims, tunes = [], []
    for ti, t in enumerate(topos):
        for op in ls.CollectiveOp:
            for size in (32 * MIB, 256 * MIB):
                n = t.n_gpus
                spec = ls.CollectiveSpec(op, n, size)
                for noise in (None, ls.NoiseModel(0.05, seed=ti)):
                    shares = ls.initialize_shares(t)
                    rep = ls.simulate_collective(t, spec, shares, noise=noise, alignment=1)
                    sims.append({"topo": ti, "op": op.value, "n": n, "size": size,
                                 "noise": None if noise is None else [noise.sigma, noise.seed],
                                 "shares": g2j(shares.as_dict()),
                                 "durations": {str(int(k)): v for k, v in
                                               sorted(rep.durations.items())},
                                 "total": rep.total, "algbw": rep.algbw})
                    final, trace = ls.initial_tune(t, spec, noise=noise)
                    tunes.append({"topo": ti, "op": op.value, "n": n, "size": size,
                                  "noise": None if noise is None else [noise.sigma, noise.seed],
                                  "final": g2j(final.as_dict()), "converged": trace.converged,
                                  "records": records_to_json(trace)})
    out["simulate"] = sims
    out["tune"] = tunes

    # injected measurements (tuner.py:178 seam): alternating + hostile
    t3 = ls.TopologySpec(n_gpus=8, links={
        P.NVLINK: ls.LinkSpec(P.NVLINK, 100e9),
        P.PCIE_STAGED: ls.LinkSpec(P.PCIE_STAGED, 50e9, staging_chunk=MIB),
        P.RDMA_NIC: ls.LinkSpec(P.RDMA_NIC, 25e9, staging_chunk=MIB)}, name="adv")
    out["adv_topo"] = topo_to_json(t3)
    spec = ls.CollectiveSpec(ls.CollectiveOp.ALLREDUCE, 8, 64 * MIB)
    calls = {"n": 0}

    def alternating(state):
        calls["n"] += 1
        flip = calls["n"] % 2 == 0
        d = {p: 1.0 for p in state.active}
        if P.PCIE_STAGED in state.active:
            d[P.PCIE_STAGED] = 2.0 if flip else 2.5
        if P.RDMA_NIC in state.active:
            d[P.RDMA_NIC] = 2.5 if flip else 2.0
        return ls.PathTimingReport.build(spec.op, 8, spec.size, d)

    final, trace = ls.initial_tune(t3, spec, measure=alternating)
    out["tune_alternating"] = {"final": g2j(final.as_dict()), "converged": trace.converged,
                               "records": records_to_json(trace)}

    def hostile(state):
        d = {p: (3.0 if p == P.NVLINK else 1.0) for p in state.active}
        return ls.PathTimingReport.build(spec.op, 8, spec.size, d)

    final, trace = ls.initial_tune(t3, spec, measure=hostile)
    out["tune_hostile"] = {"final": g2j(final.as_dict()), "converged": trace.converged,
                           "records": records_to_json(trace)}
    cfg = ls.TunerConfig(initial_step=8, convergence_threshold=0.01, stability_required=2,
                         max_iterations=40)
    final, trace = ls.initial_tune(ls.preset("H800"), ls.CollectiveSpec(
        ls.CollectiveOp.ALLGATHER, 4, 128 * MIB), cfg, alignment=4096)
    out["tune_cfg"] = {"final": g2j(final.as_dict()), "converged": trace.converged,
                       "records": records_to_json(trace)}

    # ---- Stage 2 (balancer.py:163-207)
    dyn = []
    drift_topo = ls.preset("H800").restricted(bench.MODE_PATHS[bench.MODE_PCIE_ONLY])
    scenarios = [
        ("drift", drift_topo, {0: 912, 1: 88}, [[31, 1, 0.7, None]], None, 150),
        ("spike", drift_topo, {0: 912, 1: 88}, [[15, 1, 0.3, 1]], None, 60),
        ("noise", ls.preset("H800"), {0: 800, 1: 150, 2: 50}, [], [0.08, 3], 200),
        ("nvslow", ls.preset("H800"), {0: 700, 1: 200, 2: 100}, [[5, 0, 0.2, None]], None, 120),
        ("drain", drift_topo, {0: 985, 1: 15}, [[1, 1, 0.05, None]], None, 100),
    ]
    for name, t, shares, shifts, noise, ncalls in scenarios:
        sh = tuple(balancer.BandwidthShift(a, P(p), s, d) for a, p, s, d in shifts)
        nm = ls.NoiseModel(*noise) if noise else None
        spec = ls.CollectiveSpec(ls.CollectiveOp.ALLREDUCE, 8, 256 * MIB)
        res = ls.run_dynamic(t, spec, ls.ShareDistribution({P(k): v for k, v in shares.items()}),
                             n_calls=ncalls, shifts=sh, noise=nm)
        dyn.append({"name": name, "topo": topo_to_json(t), "shares": {str(k): v for k, v in
                                                                       shares.items()},
                    "shifts": shifts, "noise": noise, "n_calls": ncalls,
                    "final": g2j(res.final_shares.as_dict()),
                    "totals": [r.total for r in res.reports],
                    "evals": [{"call": e.call, "gap": e.gap, "moved": e.moved,
                               "source": None if e.adjustment is None else int(e.adjustment.source),
                               "target": None if e.adjustment is None else int(e.adjustment.target),
                               "shares": g2j(e.shares)} for e in res.evaluations]})
    out["dynamic"] = dyn

    # ---- staging pipeline
    pipes = []
    for _ in range(80):
        spec = ls.PipelineSpec(chunk_bytes=rng.choice([4096, 64 << 10, MIB, 4 * MIB]),
                               bw_pd2h=rng.uniform(1e9, 64e9), bw_h2cd=rng.uniform(1e9, 64e9),
                               per_chunk_overhead=rng.choice([0.0, 2e-6, 1e-5]),
                               buffers=rng.choice([1, 2]))
        total = rng.choice([0, 1, 4095, rng.uniform(1, 64 * MIB), 40 * MIB])
        pipes.append({"chunk": spec.chunk_bytes, "a": spec.bw_pd2h, "b": spec.bw_h2cd,
                      "ovh": spec.per_chunk_overhead, "buffers": spec.buffers, "total": total,
                      "closed": ls.pipeline_time(total, spec),
                      "events": ls.simulate_pipeline_events(total, spec)})
    out["pipeline"] = pipes
    prot = []
    for variant in ("counter", "binary"):
        for buffers in (1, 2, 3):
            for iters in (1, 2, 3, 4, 5):
                v = ls.explore_protocol(iters, buffers=buffers, variant=variant)
                prot.append({"variant": variant, "buffers": buffers, "iterations": iters,
                             "ok": v.ok, "states": v.states_explored, "deadlocks": v.deadlocks,
                             "witness": None if v.witness is None else
                             [a.to_dict() for a in v.witness]})
    out["protocol"] = prot

    # ---- optimum references
    opt = []
    for ti in range(0, len(topos), 3):
        t = topos[ti]
        spec = ls.CollectiveSpec(ls.CollectiveOp.ALLREDUCE, t.n_gpus, 64 * MIB)
        gran = 10 if len(t.links) == 3 else 5
        r = ls.optimal_shares_bruteforce(t, spec, granularity=gran)
        opt.append({"topo": ti, "granularity": gran, "best": g2j(r.best_shares.as_dict()),
                    "time": r.best_time, "evaluations": r.evaluations})
    out["bruteforce"] = opt
    cf = []
    for _ in range(40):
        kinds = [P.NVLINK] + [k for k in (P.PCIE_STAGED, P.RDMA_NIC) if rng.random() < 0.8]
        bws = {k: rng.uniform(1e9, 900e9) for k in kinds}
        lats = {k: rng.uniform(0, 50e-6) for k in kinds}
        steps = rng.choice([1, 7, 14])
        vol = rng.choice([1e6, 64 * MIB * 14 / 8, 1e10])
        try:
            res = {str(int(k)): v for k, v in ls.closed_form_shares(bws, lats, steps, vol).items()}
        except ValueError as e:
            res = {"error": str(e)}
        cf.append({"bw": {str(int(k)): v for k, v in bws.items()},
                   "lat": {str(int(k)): v for k, v in lats.items()}, "steps": steps,
                   "volume": vol, "out": res})
    out["closed_form"] = cf

    # ---- unit parsing
    out["units"] = {
        "size": [[s, units.parse_size(s)] for s in ("256M", "4MiB", "1G", "512", "1.5K", "4 M")],
        "bw": [[s, units.parse_bandwidth(s)] for s in
               ("200 GB/s", "800 Gb/s", "64GB/s", "50 Gb/s", "1.5 TB/s", "400 kb/s", "12")],
        "time": [[s, units.parse_time(s)] for s in ("5us", "1.5 ms", "10µs", "2 s", "7ns", "3")],
    }
    OUT.write_text(json.dumps(out, indent=0, sort_keys=True))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
