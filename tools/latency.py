"""Small-message cost per call (8 virtual ranks and 8-rank loopback), fp32 AllReduce."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_15882_b200 import comm as flx  # noqa: E402

for loop, timing in ((False, True), (False, False), (True, True), (True, False)):
    cl = flx.Clique(8, loopback=loop)
    cl.set_timing(timing)
    for kib in (4, 64, 1024, 4096):
        s = [torch.randn(kib * 256, device="cuda") for _ in range(8)]
        r = [torch.empty_like(x) for x in s]
        for _ in range(20):
            cl.all_reduce(s, r)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(200):
            cl.all_reduce(s, r)
        e1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / 200
        h = cl.comms[0].path_times_history(64)
        dev = sum(x[0] for x in h) / len(h) if h else 0
        print(json.dumps({"loopback": loop, "timing": timing, "kib": kib, "us_per_call": round(e0.elapsed_time(e1) / 200 * 1e3, 2),
                          "host_us_per_call": round(wall * 1e6, 2), "path_us": round(dev * 1e6, 2)}), flush=True)
    cl.destroy()
