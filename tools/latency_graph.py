"""Small-message AllReduce cost per call when the calls are replayed from a CUDA graph.

The eager numbers (`latency.py`) are host-issue bound: every call pays ctypes, the
group call and, with timing on, two timing-event records.  A serving engine captures
its tensor-parallel layers into CUDA graphs, so the cost it sees is the device-side
one.  This tool captures CALLS back-to-back AllReduces (8 virtual ranks, and 8-rank
loopback = the one-process-per-GPU kernels) into one graph, replays it REPS times
between CUDA events and reports us per call; the eager cost of the same call, timed
the same way, sits beside it.  Results are checked exact after the replays.
One JSON line per (executor, size).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

CALLS, REPS, N = 20, 50, 8


def per_call_us(fn, reps, calls_per_rep):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * calls_per_rep)


for loop in (False, True):
    cl = flx.Clique(N, loopback=loop)
    cl.set_shares(CollectiveOp.ALLREDUCE, (1000, 0, 0))
    for kib in (4, 64, 256, 1024, 4096):
        count = kib * 256
        g = torch.Generator(device="cuda").manual_seed(kib)
        s = [torch.randint(-64, 64, (count,), device="cuda", generator=g).float()
             for _ in range(N)]
        r = [torch.empty_like(x) for x in s]
        exact = torch.stack(s).sum(0)
        stream = torch.cuda.Stream()
        stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(stream):
            for _ in range(5):
                cl.all_reduce(s, r)
        torch.cuda.current_stream().wait_stream(stream)
        torch.cuda.synchronize()

        def eager():
            for _ in range(CALLS):
                cl.all_reduce(s, r)

        eager_us = per_call_us(eager, REPS, CALLS)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for _ in range(CALLS):
                cl.all_reduce(s, r)
        graph.replay()
        torch.cuda.synchronize()
        graph_us = per_call_us(graph.replay, REPS, CALLS)
        ok = all(torch.equal(x, exact) for x in r)
        del graph
        busbw = count * 4 / (graph_us * 1e-6) * 2 * (N - 1) / N / 1e9
        print(json.dumps({"executor": "loopback" if loop else "virtual", "ranks": N,
                          "kib_per_rank": kib, "graph_us_per_call": round(graph_us, 2),
                          "eager_us_per_call": round(eager_us, 2),
                          "graph_busbw_gbs": round(busbw, 1), "exact": ok}), flush=True)
    cl.destroy()
