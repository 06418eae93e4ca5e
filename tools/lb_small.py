"""8-rank loopback AllReduce (LB_BYTES per rank, default 4 KiB), repeated — for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_15882_b200 import comm as flx  # noqa: E402

n = int(os.environ.get("LB_RANKS", "8"))
cl = flx.Clique(n, loopback=True)
s = [torch.randn(int(os.environ.get("LB_BYTES", "4096")) // 4, device="cuda") for _ in range(n)]
r = [torch.empty_like(x) for x in s]
for _ in range(int(os.environ.get("LB_CALLS", "30"))):
    cl.all_reduce(s, r)
torch.cuda.synchronize()
cl.destroy()
print("ok")
