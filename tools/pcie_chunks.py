"""Virtual-rank PCIe path alone (8 ranks x 256 MiB fp32 AllReduce, every byte
host-staged): per-direction rate vs staging chunk per rank and ring depth.
Bound: 2 GiB each way at the concurrent pinned rate (~49.6 GB/s)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_15882_b200 import comm  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

n, mib = 8, int(sys.argv[1]) if len(sys.argv) > 1 else 256
pcie = int(sys.argv[2]) if len(sys.argv) > 2 else 1000   # PCIe granules
ctas = int(sys.argv[3]) if len(sys.argv) > 3 else 0      # NVLink-path cap
count = mib << 18
x = [torch.ones(count, device="cuda") for _ in range(n)]
y = [torch.empty_like(t) for t in x]
c = comm.Clique(n)
c.set_autotune(False)
c.set_shares(CollectiveOp.ALLREDUCE, (1000 - pcie, pcie, 0))
c.set_nvlink_ctas(ctas)
for bufs in ((2, 1) if pcie == 1000 else (2,)):
    for ck in ((1, 2, 4, 8, 16, 32) if pcie == 1000 else (1, 2, 3, 4, 6, 8, 12, 16)):
        c.set_staging(ck << 20, bufs)
        for _ in range(2):
            c.all_reduce(x, y)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            c.all_reduce(x, y)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        print(json.dumps({"pcie_granules": pcie, "nvlink_ctas": ctas,
                          "buffers": bufs, "chunk_mib": ck, "ms": round(ms, 3),
                          "each_way_gbs": round(n * (mib << 20) / ms / 1e6, 2)}), flush=True)
