"""Stage 1 + Stage 2 on the multi-rank engine (loopback world): the NVLink-path
rank kernels capped to a few CTAs so the host-hub PCIe path carries a share,
then bench.run_stage2_drift's PCIe hog — the balancer must move granules off
PCIe while the hog runs and back after.  One JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.links import PathKind, preset  # noqa: E402
from paper_2510_15882_b200.stage1 import TunerConfig  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

n = int(os.environ.get("WS_RANKS", "4"))
ctas = int(os.environ.get("WS_CTAS", "1"))
cl = flx.Clique(n, loopback=True)
cl.set_nvlink_ctas(ctas)
cnt = bench.AR_BYTES // 4
g = torch.Generator(device="cuda").manual_seed(5)
sends = [torch.randint(-1024, 1024, (cnt,), device="cuda", generator=g).float() for _ in range(n)]
recvs = [torch.empty_like(s) for s in sends]
topo = preset("B200", n_gpus=max(n, 2)).restricted([PathKind.NVLINK, PathKind.PCIE_STAGED])
shares, trace, tuned, base = flx.tune_shares(cl, topo, CollectiveOp.ALLREDUCE, sends, recvs,
                                             TunerConfig(), warmup=1, repeats=3)
drift = bench.run_stage2_drift(cl, sends, recvs, shares, torch.cuda.current_stream(),
                               calls=160, hog_from=40, hog_to=100)
exact = torch.stack(sends).sum(0)
ok = all(torch.equal(r, exact) for r in recvs)
print(json.dumps({"executor": "loopback world", "n": n, "nvlink_ctas": ctas,
                  "stage1_shares": {k.short: shares.get(k) for k in PathKind},
                  "stage1_tuned_ms": round(tuned * 1e3, 3),
                  "stage1_nvlink_only_ms": round(base * 1e3, 3),
                  "stage1_trace": [r.action for r in trace.records], "stage2_drift": drift,
                  "result_exact": ok}))
cl.destroy()
