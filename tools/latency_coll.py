"""Per-call time of small collectives on the 8-rank loopback engine (timing
events off), one line per collective; run with FLX_ONESHOT_KB=0 to compare
against the slot (two-hop) protocols."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_15882_b200 import comm as flx  # noqa: E402

n, kib = 8, int(os.environ.get("LAT_KIB", "4"))
cl = flx.Clique(n, loopback=True)
cl.set_timing(False)
cnt = kib * 256
s = [torch.randn(n * cnt, device="cuda") for _ in range(n)]
full = [torch.empty_like(x) for x in s]
part = [torch.empty(cnt, device="cuda") for _ in range(n)]
ag_in = [x[:cnt] for x in s]
calls = {
    "allreduce": lambda: cl.all_reduce(ag_in, part),
    "allgather": lambda: cl.all_gather(ag_in, full),
    "reducescatter": lambda: cl.reduce_scatter(s, part),
    "alltoall": lambda: cl.all_to_all(s, full),
}
for name, fn in calls.items():
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(200):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"coll": name, "kib_per_rank": kib, "oneshot_kb": os.environ.get("FLX_ONESHOT_KB", "256"),
                      "us_per_call": round(e0.elapsed_time(e1) / 200 * 1e3, 2)}), flush=True)
cl.destroy()
