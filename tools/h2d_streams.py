"""Pinned H2D of 8 x 256 MiB (the e2e step's inputs) over 1, 2, 4 or 8 streams:
does spreading the copies over more copy engines move more than one stream's
~55 GB/s through the one PCIe Gen5 link?  One JSON line per stream count."""
import json

import torch

n, mib = 8, 256
host = [torch.empty(mib << 20, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
dev = [torch.empty(mib << 20, dtype=torch.uint8, device="cuda") for _ in range(n)]
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    for _ in range(2):
        for i in range(n):
            with torch.cuda.stream(streams[i % k]):
                dev[i].copy_(host[i], non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    main = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(main)
    for rep in range(5):
        for i in range(n):
            with torch.cuda.stream(streams[i % k]):
                dev[i].copy_(host[i], non_blocking=True)
    for s in streams:
        main.wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(json.dumps({"streams": k, "ms_per_2GiB": round(ms, 3),
                      "GBps": round(n * (mib << 20) / ms / 1e6, 2)}), flush=True)
