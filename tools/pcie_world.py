"""The multi-rank engine's host-hub PCIe path alone (shares 0/1000/0), 8-rank
loopback: ms per call and the per-link GB/s it sustains, per collective."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

n = int(os.environ.get("PW_RANKS", "8"))
MIB = 1 << 20
cl = flx.Clique(n, loopback=True)
for op in CollectiveOp:
    cl.set_shares(op, (0, 1000, 0))
S = int(os.environ.get("PW_MIB", "64")) * MIB  # per-rank message (AR / AG send / RS, A2A block x n)
cnt = S // 4
s = [torch.randn(cnt, device="cuda") for _ in range(n)]
full = [torch.empty(cnt * n, device="cuda") for _ in range(n)]
same = [torch.empty(cnt, device="cuda") for _ in range(n)]
part = [torch.empty(cnt // n, device="cuda") for _ in range(n)]
calls = {
    "allreduce": (lambda: cl.all_reduce(s, same), 2 * S),        # D2H S/n*(n-1)... per-rank bytes moved
    "allgather": (lambda: cl.all_gather(s, full), S * n),
    "reducescatter": (lambda: cl.reduce_scatter(s, part), S),
    "alltoall": (lambda: cl.all_to_all(s, same), S),
}
for name, (fn, _) in calls.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"coll": name, "n": n, "mib_per_rank": S // MIB, "ms": round(ms, 3),
                      "chunk_env": os.environ.get("FLX_PCIE_CHUNK_KB", "default")}), flush=True)
cl.destroy()
