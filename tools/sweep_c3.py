"""BASELINE config 3: AllReduce (or --op allgather) fp32/bf16 message-size sweep 1 MiB - 1 GiB at N = 2/4/8
(virtual ranks on one GPU), Stage 1 on the real path per size bucket (+ guard), per-link
traffic split and the Stage-1 trace.  One JSON line per cell."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.links import PathKind, preset  # noqa: E402
from paper_2510_15882_b200.stage1 import TunerConfig  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--ranks", default="2,4,8")
p.add_argument("--max-mib", type=int, default=1024)
p.add_argument("--steps", type=int, default=50)
p.add_argument("--warmup", type=int, default=20)
p.add_argument("--trace-dir", default="", help="write each cell's Stage-1 trace (reference "
               "JSONL schema, tuner.py:229-253) here")
p.add_argument("--nvlink-ctas", type=int, default=0)
p.add_argument("--op", choices=["allreduce", "allgather"], default="allreduce",
               help="allgather: S is the gathered size (S/N sent per rank), nccl-tests busbw")
p.add_argument("--loopback", action="store_true",
               help="the multi-GPU engine emulated on one GPU, NVLink path only (no tuning)")
p.add_argument("--inlib", action="store_true",
               help="the in-library balancer tunes every bucket (no Python Stage 1); "
                    "NVLink-only timed beside it; works with --loopback too")
a = p.parse_args()
topo = preset("B200").restricted([PathKind.NVLINK, PathKind.PCIE_STAGED])
for n in [int(x) for x in a.ranks.split(",")]:
    cl = flx.Clique(n, loopback=a.loopback)
    if a.nvlink_ctas:
        cl.set_nvlink_ctas(a.nvlink_ctas)
    if a.inlib:
        cl.set_tuner_config(min_bytes=1 << 20)
    for dt, esz, name in ((torch.float32, 4, "fp32"), (torch.bfloat16, 2, "bf16")):
        mib = 1
        while mib <= a.max_mib:
            S = mib << 20
            gather = a.op == "allgather"
            cop = CollectiveOp.ALLGATHER if gather else CollectiveOp.ALLREDUCE
            per = S // esz // n if gather else S // esz
            s = [torch.randn(per, device="cuda").to(dt) for _ in range(n)]
            r = [torch.empty(per * n if gather else per, device="cuda", dtype=dt) for _ in range(n)]
            run = (lambda: cl.all_gather(s, r)) if gather else (lambda: cl.all_reduce(s, r))
            nv_only_ms = info = None
            if a.inlib:
                nb = (per * esz)
                cl.set_shares(cop, (1000, 0, 0), nb)  # NVLink-only reference timing
                for _ in range(3):
                    run()
                torch.cuda.synchronize()
                q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                q0.record()
                for _ in range(10):
                    run()
                q1.record()
                torch.cuda.synchronize()
                nv_only_ms = q0.elapsed_time(q1) / 10
                cl.set_shares(cop, None, nb)  # hand the bucket to the in-library balancer
                k = 0
                while k < 400 and cl.tune_info(cop, nb)["phase"] not in ("stage2",) and not (
                        k >= 2 and cl.tune_info(cop, nb)["phase"] == "idle"):
                    run()
                    k += 1
                info = cl.tune_info(cop, nb)
                info["tuning_calls"] = k
                info["stage1_trace"] = [x["action"] for x in cl.tune_trace(cop, nb)]
                shares = flx.ShareDistribution({kd: info["shares"][int(kd)] for kd in PathKind
                                                if info["shares"][int(kd)] or kd == 0})
                trace = None
            elif a.loopback:
                shares, trace = flx.ShareDistribution({PathKind.NVLINK: 1000}), None
                cl.set_shares(cop, shares)
            else:
                shares, trace, tuned, base = flx.tune_shares(cl, topo, cop, s, r, TunerConfig(),
                                                             warmup=1, repeats=3)
            for _ in range(a.warmup):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                run()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / a.steps * 1e-3
            b = cl.path_bytes()
            print(json.dumps({
                "executor": "loopback" if a.loopback else "virtual", "op": a.op,
                "n": n, "dtype": name, "size_mib": mib, "ms": round(t * 1e3, 4),
                "busbw": round(S / t * ((n - 1) / n if gather else 2 * (n - 1) / n) / 1e9, 2),
                "shares": {k.short: shares.get(k) for k in PathKind},
                "traffic_pct": {k.short: round(100 * b[k] / (S // n if gather else S), 3)
                                for k in PathKind},
                "nvlink_only_ms": None if nv_only_ms is None else round(nv_only_ms, 4),
                "gain_pct": None if nv_only_ms is None else round(100 * (nv_only_ms / (t * 1e3) - 1), 2),
                "balancer": info,
                "stage1": None if trace is None else {
                    "iterations": trace.iterations, "tuned_ms": round(tuned * 1e3, 4),
                    "nvlink_only_ms": round(base * 1e3, 4),
                    "trace": [x.action for x in trace.records]}}), flush=True)
            if a.trace_dir and trace is not None:
                from paper_2510_15882_b200.stage1 import write_trace

                os.makedirs(a.trace_dir, exist_ok=True)
                tag = "ag_" if gather else ""
                with open(os.path.join(a.trace_dir, f"{tag}n{n}_{name}_{mib}MiB.jsonl"), "w") as fh:
                    write_trace(trace, fh, fmt="jsonl")
            del s, r
            mib *= 2
    cl.destroy()
