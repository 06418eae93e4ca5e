"""8-rank loopback AllReduce (LB_BYTES per rank, default 4 KiB; LB_DTYPE fp32|bf16), repeated —
for ncu.  LB_TIME=1 also prints the mean ms per call from CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_15882_b200 import comm as flx  # noqa: E402

n = int(os.environ.get("LB_RANKS", "8"))
cl = flx.Clique(n, loopback=True)
dt = {"fp32": torch.float32, "bf16": torch.bfloat16}[os.environ.get("LB_DTYPE", "fp32")]
nbytes = int(os.environ.get("LB_BYTES", "4096"))
s = [torch.randn(nbytes // dt.itemsize, device="cuda").to(dt) for _ in range(n)]
r = [torch.empty_like(x) for x in s]
for _ in range(int(os.environ.get("LB_CALLS", "30"))):
    cl.all_reduce(s, r)
torch.cuda.synchronize()
if os.environ.get("LB_TIME"):
    calls = 20
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(calls):
        cl.all_reduce(s, r)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / calls
    print(f"ranks={n} dtype={dt} bytes={nbytes} ms={ms:.4f} busbw={nbytes / ms / 1e6 * 2 * (n - 1) / n:.1f}")
cl.destroy()
print("ok")
