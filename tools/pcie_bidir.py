"""PCIe copy-engine concurrency probe: H2D + D2H at once, 1..4 streams per
direction, 8 x 256 MiB each way (the e2e step's traffic)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

MIB = 1 << 20
n, size = 8, 256 * MIB
h_in = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
h_out = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
d_in = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(n)]
d_out = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(n)]


def run(k: int, up: bool, down: bool, split: int = 1) -> float:
    ups = [torch.cuda.Stream() for _ in range(k)]
    downs = [torch.cuda.Stream() for _ in range(k)]
    main = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(2):
        a.record(main)
        for s in ups + downs:
            s.wait_stream(main)
        piece = size // split
        j = 0
        for i in range(n):
            for p in range(split):
                sl = slice(p * piece, (p + 1) * piece)
                if up:
                    with torch.cuda.stream(ups[j % k]):
                        d_in[i][sl].copy_(h_in[i][sl], non_blocking=True)
                if down:
                    with torch.cuda.stream(downs[j % k]):
                        h_out[i][sl].copy_(d_out[i][sl], non_blocking=True)
                j += 1
        for s in ups + downs:
            main.wait_stream(s)
        b.record(main)
        torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    return round(n * size / (ms * 1e-3) / 1e9, 2)


out = {}
for k in (1, 2, 4):
    out[f"h2d_only_{k}s"] = run(k, True, False)
    out[f"d2h_only_{k}s"] = run(k, False, True)
    out[f"bidir_each_{k}s"] = run(k, True, True)
out["bidir_each_2s_split4"] = run(2, True, True, split=4)
print(json.dumps(out))
