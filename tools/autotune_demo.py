"""Print what the in-library balancer does on one GPU (virtual ranks), capped and
uncapped: phases, Stage-1 trace, guard, Stage-2 evaluations, and busbw before /
after.  Usage: python tools/autotune_demo.py [ctas] [MiB per rank] [calls]"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2510_15882_b200 import comm  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

ctas = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mib = int(sys.argv[2]) if len(sys.argv) > 2 else 64
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 150
n, count = 8, mib * (1 << 20) // 4
g = torch.Generator(device="cuda").manual_seed(1)
x = [torch.randint(-1024, 1024, (count,), device="cuda", generator=g).float() for _ in range(n)]
y = [torch.empty_like(t) for t in x]
with comm.Clique(n, device=0) as c:
    c.set_nvlink_ctas(ctas)
    t0 = time.perf_counter()
    phases = []
    for i in range(calls):
        c.all_reduce(x, y)
        ph = c.tune_info(CollectiveOp.ALLREDUCE, count * 4)["phase"]
        if not phases or phases[-1][1] != ph:
            phases.append((i, ph))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    info = c.tune_info(CollectiveOp.ALLREDUCE, count * 4)
    hist = c.comms[0].path_times_history(10)
    print(json.dumps({"ctas": ctas, "mib": mib, "calls": calls, "wall_s": round(wall, 3),
                      "phases": phases, "info": info,
                      "trace": [(r["action"], r["shares"], [None if d is None else round(d, 3)
                                                             for d in r["durations_ms"]])
                                for r in c.tune_trace(CollectiveOp.ALLREDUCE, count * 4)],
                      "evals": c.tune_evaluations(CollectiveOp.ALLREDUCE, count * 4)[-5:],
                      "last_ms": [[round(v * 1e3, 3) for v in h.values()] for h in hist]}))
    ok = all(torch.equal(t, torch.stack(x).sum(0)) for t in y)
    print("exact", ok)
