"""Diagnostic: per-path times of the 8-virtual-rank 256 MiB fp32 AllReduce vs PCIe granules,
NVLink-kernel CTA cap and staging chunk.  Prints one JSON line per cell."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.links import PathKind  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

n, count = 8, 64 << 20
s = [torch.randn(count, device="cuda") for _ in range(n)]
r = [torch.empty_like(x) for x in s]
cl = flx.Clique(n)


def cell(ctas, pcie, chunk, buffers=2, reps=10):
    cl.set_nvlink_ctas(ctas)
    cl.set_staging(chunk, buffers)
    cl.set_shares(CollectiveOp.ALLREDUCE, (1000 - pcie, pcie, 0))
    for _ in range(3):
        cl.all_reduce(s, r)
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(reps):
        cl.all_reduce(s, r)
    en.record()
    torch.cuda.synchronize()
    step = st.elapsed_time(en) / reps
    h = cl.comms[0].path_times_history(reps)
    nv = statistics.mean(x[PathKind.NVLINK] for x in h) * 1e3
    pc = statistics.mean(x[PathKind.PCIE_STAGED] for x in h) * 1e3
    b = cl.path_bytes()
    busbw = (count * 4) / (step * 1e-3) * 2 * (n - 1) / n / 1e9
    print(json.dumps({"ctas": ctas, "pcie_g": pcie, "chunk": chunk, "buffers": buffers,
                      "step_ms": round(step, 4), "nv_ms": round(nv, 4), "pcie_ms": round(pc, 4),
                      "pcie_bytes": b[PathKind.PCIE_STAGED], "busbw": round(busbw, 1)}), flush=True)


# raw PCIe copy bandwidth (pinned)
h = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
d = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record(); [fn() for _ in range(5)]; en.record(); torch.cuda.synchronize()
    print(json.dumps({"probe": name, "GBps": round(5 * (256 << 20) / (st.elapsed_time(en) * 1e-3) / 1e9, 2)}))
s2 = torch.cuda.Stream()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
h2 = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
d2 = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
st.record()
with torch.cuda.stream(s2):
    for _ in range(5):
        h2.copy_(d2, non_blocking=True)
for _ in range(5):
    d.copy_(h, non_blocking=True)
torch.cuda.current_stream().wait_stream(s2)
en.record(); torch.cuda.synchronize()
print(json.dumps({"probe": "bidir", "GBps_each": round(5 * (256 << 20) / (st.elapsed_time(en) * 1e-3) / 1e9, 2)}))

for ctas in (0, 16, 8, 4):
    for pcie in (0, 5, 10, 20, 40, 80):
        cell(ctas, pcie, 0)
for chunk in (256 << 10, 1 << 20, 4 << 20):
    cell(8, 40, chunk)
    cell(8, 40, chunk, buffers=1)
cl.destroy()
