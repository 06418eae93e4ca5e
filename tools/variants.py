"""Time the virtual-rank fold / fan-out kernels and the PCIe path under the
current FLX_* environment (run once per variant).  One JSON line."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.links import PathKind  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

n, S = 8, 256 << 20
peak = 6551.4
cl = flx.Clique(n)
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("FLX_")}}


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for dt, name in ((torch.float32, "f32"), (torch.bfloat16, "bf16")):
    cnt = S // (4 if dt == torch.float32 else 2)
    s = [torch.randn(cnt, device="cuda").to(dt) for _ in range(n)]
    r = [torch.empty_like(x) for x in s]
    cl.set_shares(CollectiveOp.ALLREDUCE, (1000, 0, 0))
    ms = timeit(lambda: cl.all_reduce(s, r))
    h = cl.comms[0].path_times_history(20)
    kms = statistics.mean(x[PathKind.NVLINK] for x in h) * 1e3
    acc = s[0].float()
    for x in s[1:]:
        acc = acc + x.float()
    ok = all(torch.equal(o, acc.to(dt)) for o in r)
    out[f"allreduce_{name}"] = {"ms": round(ms, 4), "kernel_ms": round(kms, 4),
                                "hbm_frac": round(2 * n * S / (kms * 1e-3) / 1e9 / peak, 4),
                                "busbw": round(S / (ms * 1e-3) * 1.75 / 1e9, 1), "exact": ok}
    del s, r
ag = S // 2 // n
s = [torch.randn(ag, device="cuda").bfloat16() for _ in range(n)]
r = [torch.empty(ag * n, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
ms = timeit(lambda: cl.all_gather(s, r))
h = cl.comms[0].path_times_history(20)
kms = statistics.mean(x[PathKind.NVLINK] for x in h) * 1e3
ok = all(torch.equal(o, torch.cat(s)) for o in r)
out["allgather_bf16"] = {"ms": round(ms, 4), "kernel_ms": round(kms, 4),
                         "hbm_frac": round((n + n * n) * (S // n) / (kms * 1e-3) / 1e9 / peak, 4),
                         "busbw": round(S / (ms * 1e-3) * 7 / 8 / 1e9, 1), "exact": ok}
del s, r
# ReduceScatter fp32: each rank sends n blocks of S/n, receives one block
blk = S // 4 // n
s = [torch.randn(blk * n, device="cuda") for _ in range(n)]
r = [torch.empty(blk, device="cuda") for _ in range(n)]
cl.set_shares(CollectiveOp.REDUCESCATTER, (1000, 0, 0))
ms = timeit(lambda: cl.reduce_scatter(s, r))
h = cl.comms[0].path_times_history(20)
kms = statistics.mean(x[PathKind.NVLINK] for x in h) * 1e3
out["reducescatter_f32"] = {"ms": round(ms, 4), "kernel_ms": round(kms, 4),
                            "hbm_frac": round((n * S + S) / (kms * 1e-3) / 1e9 / peak, 4),
                            "busbw": round(S / (ms * 1e-3) * 7 / 8 / 1e9, 1)}
# AllToAll fp32: n blocks of S/n each way
r = [torch.empty_like(x) for x in s]
cl.set_shares(CollectiveOp.ALLTOALL, (1000, 0, 0))
ms = timeit(lambda: cl.all_to_all(s, r))
h = cl.comms[0].path_times_history(20)
kms = statistics.mean(x[PathKind.NVLINK] for x in h) * 1e3
out["alltoall_f32"] = {"ms": round(ms, 4), "kernel_ms": round(kms, 4),
                       "hbm_frac": round(2 * n * S / (kms * 1e-3) / 1e9 / peak, 4)}
del s, r
# PCIe-path cost in the capped (config-4 style) setting
cnt = S // 4
s = [torch.randn(cnt, device="cuda") for _ in range(n)]
r = [torch.empty_like(x) for x in s]
cl.set_nvlink_ctas(3)
for g in (0, 100, 200, 300):
    cl.set_shares(CollectiveOp.ALLREDUCE, (1000 - g, g, 0))
    ms = timeit(lambda: cl.all_reduce(s, r), reps=5)
    h = cl.comms[0].path_times_history(5)
    out[f"capped3_pcie{g}"] = {"ms": round(ms, 3),
                               "nv_ms": round(statistics.mean(x[PathKind.NVLINK] for x in h) * 1e3, 3),
                               "pcie_ms": round(statistics.mean(x[PathKind.PCIE_STAGED] for x in h) * 1e3, 3)}
print(json.dumps(out), flush=True)
cl.destroy()
