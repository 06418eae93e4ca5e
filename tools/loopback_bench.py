"""Time the one-process-per-GPU engine's rank kernels in loopback (all ranks on
this GPU, cooperative launch), NVLink-only split, AllReduce / AllGather /
ReduceScatter at 256 MiB per rank, several CTA counts.  One JSON line per cell.
HBM-bound here (every 'NVLink' byte is local HBM): algorithmic HBM bytes per
AllReduce call = (5n-2) * S (push 2(n-1)/n S r+w, fold (1+2/n) S, pull)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_15882_b200 import comm  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

MIB = 1 << 20
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists(
    "MEASURED_PEAKS.json") else 6545.0


def timed(fn, steps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8,4,2").split(",")]:
    for dt in (torch.float32, torch.bfloat16):
        count = 256 * MIB // (4 if dt == torch.float32 else 2)
        g = torch.Generator(device="cuda").manual_seed(n)
        x = [torch.randint(-64, 64, (count,), device="cuda", generator=g).to(dt) for _ in range(n)]
        y = [torch.empty_like(t) for t in x]
        exact = torch.stack([t.float() for t in x]).sum(0).to(dt)
        for ctas in (0, 18, 32, 36, 64):
            with comm.Clique(n, device=0, loopback=True) as w:
                w.set_shares(CollectiveOp.ALLREDUCE, (1000, 0, 0))
                if ctas:
                    w.set_nvlink_ctas(ctas)
                try:
                    ms = timed(lambda: w.all_reduce(x, y))
                except Exception as e:
                    print(json.dumps({"n": n, "ctas": ctas, "error": str(e)[:200]}))
                    continue
                ok = all(torch.equal(t, exact) for t in y)
                alg = (5 * n - 2) * 256 * MIB
                print(json.dumps({"op": "allreduce", "n": n, "dtype": str(dt)[6:], "ctas": ctas,
                                  "ms": round(ms, 4), "busbw": round(256 * MIB / ms / 1e6 * 2 * (n - 1) / n, 1),
                                  "hbm_frac": round(alg / (ms * 1e-3) / 1e9 / peak, 4),
                                  "exact": ok}), flush=True)
        del x, y
