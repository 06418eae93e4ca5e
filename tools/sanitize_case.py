"""Small, odd-sized run of every collective in both executors (with PCIe shares)
for compute-sanitizer (memcheck / racecheck): exits 0 iff all results are exact."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("FLX_SLOT_MB", "1")
os.environ.setdefault("FLX_PCIE_STAGE_MB", "4")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

ok = True
for loopback in (False, True):
    for n, count in ((3, 70001), (4, 4099)):
        g = torch.Generator().manual_seed(n)
        host = [torch.randn(n * count, generator=g) for _ in range(n)]
        with flx.Clique(n, loopback=loopback) as c:
            for op in CollectiveOp:
                c.set_shares(op, (900, 100, 0))
            al = {op: c.comms[0].alignment(op) for op in CollectiveOp}
            s = [h.cuda() for h in host]
            r = [torch.empty_like(x) for x in s]
            c.all_reduce(s, r)
            want = oracle.allreduce([h.numpy() for h in host], 7, 0, (900, 100, 0),
                                    al[CollectiveOp.ALLREDUCE])
            ok &= all(np.array_equal(a.cpu().numpy(), b) for a, b in zip(r, want))
            sg = [x[:count] for x in s]
            rg = [torch.empty(n * count, device="cuda") for _ in range(n)]
            c.all_gather(sg, rg)
            want = oracle.allgather([h.numpy()[:count] for h in host], 7, (900, 100, 0),
                                    al[CollectiveOp.ALLGATHER])
            ok &= all(np.array_equal(a.cpu().numpy(), b) for a, b in zip(rg, want))
            rs = [torch.empty(count, device="cuda") for _ in range(n)]
            c.reduce_scatter(s, rs)
            want = oracle.reducescatter([h.numpy() for h in host], 7, 0, (900, 100, 0),
                                        al[CollectiveOp.REDUCESCATTER])
            ok &= all(np.array_equal(a.cpu().numpy(), b) for a, b in zip(rs, want))
            ra = [torch.empty_like(x) for x in s]
            c.all_to_all(s, ra)
            want = oracle.alltoall([h.numpy() for h in host], 7, (900, 100, 0),
                                   al[CollectiveOp.ALLTOALL])
            ok &= all(np.array_equal(a.cpu().numpy(), b) for a, b in zip(ra, want))
            torch.cuda.synchronize()
print("sanitize case exact:", ok)
sys.exit(0 if ok else 1)
