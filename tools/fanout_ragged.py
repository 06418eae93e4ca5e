"""AllGather fan-out time for a ragged per-rank count (rank blocks off the 16 B grid:
fanout_shift_kernel) vs the aligned count (fanout_once_kernel), 8 virtual ranks,
bf16, NVLink-only split; CUDA-event time per call.  One JSON line each."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_15882_b200 import comm  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

n = 8
for extra in (0, 3, 1, 7):
    count = (32 << 20) // 2 + extra  # 32 MiB (+extra bf16) per rank: 256 MiB gathered
    x = [torch.randn(count, device="cuda").bfloat16() for _ in range(n)]
    y = [torch.empty(n * count, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
    with comm.Clique(n) as c:
        c.set_autotune(False)
        c.set_shares(CollectiveOp.ALLGATHER, (1000, 0, 0))
        for _ in range(3):
            c.all_gather(x, y)
        ts = []
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(20):
            a.record()
            c.all_gather(x, y)  # NVLink-only: one fan-out kernel per call
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ok = all(torch.equal(t, torch.cat(x)) for t in y)
    ts.sort()
    print(json.dumps({"extra_elems": extra, "kernel": "fanout_once" if extra == 0 else "fanout_shift",
                      "median_ms": round(ts[len(ts) // 2], 4), "min_ms": round(ts[0], 4),
                      "exact": ok}), flush=True)
