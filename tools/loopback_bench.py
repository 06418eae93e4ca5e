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
    if len(sys.argv) > 2 and sys.argv[2] == "all":
        break  # only the slot protocols below
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


# AllGather / ReduceScatter / AllToAll through the same engine (fp32), 256 MiB
# sent per rank; HBM algorithmic bytes per call over all ranks:
#   AllGather (S sent): n(4(n-1)+2)S   ReduceScatter (B per block): n(3n-1)B
#   AllToAll (B per block): n(4n-2)B
if len(sys.argv) > 2 and sys.argv[2] == "all":
    for n in [int(x) for x in sys.argv[1].split(",")]:
        S = 256 * MIB
        B = S // n
        g = torch.Generator(device="cuda").manual_seed(n)
        x = [torch.randint(-64, 64, (S // 4,), device="cuda", generator=g).float() for _ in range(n)]
        with comm.Clique(n, device=0, loopback=True) as w:
            for op in (CollectiveOp.ALLGATHER, CollectiveOp.REDUCESCATTER, CollectiveOp.ALLTOALL):
                w.set_shares(op, (1000, 0, 0))
            ag = [torch.empty(n * S // 4, device="cuda") for _ in range(n)]
            rs = [torch.empty(B // 4, device="cuda") for _ in range(n)]
            a2a = [torch.empty_like(t) for t in x]
            for name, fn, alg, out_ok in (
                    ("allgather", lambda: w.all_gather(x, ag), n * (4 * (n - 1) + 2) * S,
                     lambda: all(torch.equal(t, torch.cat(x)) for t in ag)),
                    ("reducescatter", lambda: w.reduce_scatter(x, rs), n * (3 * n - 1) * B,
                     lambda: all(torch.equal(rs[r], torch.stack(x).sum(0)[r * B // 4:(r + 1) * B // 4])
                                 for r in range(n))),
                    ("alltoall", lambda: w.all_to_all(x, a2a), n * (4 * n - 2) * B,
                     lambda: all(torch.equal(a2a[r], torch.cat([x[q][r * B // 4:(r + 1) * B // 4]
                                                                for q in range(n)]))
                                 for r in range(n)))):
                ms = timed(fn)
                print(json.dumps({"op": name, "n": n, "send_mib": 256, "ms": round(ms, 4),
                                  "hbm_frac": round(alg / (ms * 1e-3) / 1e9 / peak, 4),
                                  "exact": bool(out_ok())}), flush=True)
            del ag, rs, a2a
