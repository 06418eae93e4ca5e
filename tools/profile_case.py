"""Small fixed-share workload for ncu: 8 virtual ranks, 256 MiB/rank fp32 AllReduce
(or bf16 AllGather, 256 MiB out) on cuda:0.  No tuning, so the launch list is short."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--op", default="allreduce",
               choices=["allreduce", "allgather", "reducescatter", "alltoall"])
p.add_argument("--steps", type=int, default=3)
p.add_argument("--shares", default="1000,0,0")
p.add_argument("--ranks", type=int, default=8)
p.add_argument("--mib", type=int, default=256)
p.add_argument("--loopback", action="store_true",
               help="the one-process-per-GPU engine (rank kernels), all ranks on this GPU")
p.add_argument("--ragged", action="store_true",
               help="odd element count per rank (AllGather blocks off the 16 B grid)")
a = p.parse_args()
n = a.ranks
shares = [int(x) for x in a.shares.split(",")]
clique = flx.Clique(n, loopback=a.loopback)
clique.set_autotune(False)  # fixed shares: a short, deterministic launch list
if a.op == "allreduce":
    count = a.mib * (1 << 20) // 4
    s = [torch.randn(count, device="cuda") for _ in range(n)]
    r = [torch.empty_like(x) for x in s]
    clique.set_shares(CollectiveOp.ALLREDUCE, shares)
    run = lambda: clique.all_reduce(s, r)  # noqa: E731
elif a.op in ("reducescatter", "alltoall"):  # fp32, a.mib MiB sent per rank
    count = a.mib * (1 << 20) // 4
    s = [torch.randn(count, device="cuda") for _ in range(n)]
    if a.op == "reducescatter":
        r = [torch.empty(count // n, device="cuda") for _ in range(n)]
        clique.set_shares(CollectiveOp.REDUCESCATTER, shares)
        run = lambda: clique.reduce_scatter(s, r)  # noqa: E731
    else:
        r = [torch.empty_like(x) for x in s]
        clique.set_shares(CollectiveOp.ALLTOALL, shares)
        run = lambda: clique.all_to_all(s, r)  # noqa: E731
else:
    count = a.mib * (1 << 20) // 2 // n + (3 if a.ragged else 0)
    s = [torch.randn(count, device="cuda").bfloat16() for _ in range(n)]
    r = [torch.empty(count * n, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
    clique.set_shares(CollectiveOp.ALLGATHER, shares)
    run = lambda: clique.all_gather(s, r)  # noqa: E731
for _ in range(a.steps):
    run()
torch.cuda.synchronize()
print("path ms", clique.path_times(), "bytes", clique.path_bytes())
clique.destroy()
