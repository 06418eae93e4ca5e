"""Config-5 layer schedules on one B200 (8 virtual ranks): GEMM -> AllReduce per
row-parallel projection, sequential vs token-chunked on two streams with the
fold kernel capped to a few CTAs (so the GEMM keeps most SMs).  Few layers,
relative numbers only.  One JSON line per (chunks, fold CTAs)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_15882_b200 import comm  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

n, tokens, hidden, layers = 8, 65536, 5120, 8
k_attn, k_mlp = 640, 3456
g = torch.Generator(device="cuda").manual_seed(5)
outs = [torch.empty(tokens, hidden, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
xa = [torch.randn(tokens, k_attn, device="cuda", generator=g).bfloat16() for _ in range(n)]
xm = [torch.randn(tokens, k_mlp, device="cuda", generator=g).bfloat16() for _ in range(n)]
wa = [(torch.randn(k_attn, hidden, device="cuda", generator=g) / 32).bfloat16() for _ in range(n)]
wm = [(torch.randn(k_mlp, hidden, device="cuda", generator=g) / 64).bfloat16() for _ in range(n)]
clique = comm.Clique(n)
clique.set_autotune(False)
clique.set_shares(CollectiveOp.ALLREDUCE, (1000, 0, 0))
main = torch.cuda.current_stream()
side = torch.cuda.Stream()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / layers


def gemm(which, rows=slice(None)):
    xs, ws = (xa, wa) if which == 0 else (xm, wm)
    for r in range(n):
        torch.matmul(xs[r][rows], ws[r], out=outs[r][rows])


def sequential():
    for _ in range(layers):
        for w in (0, 1):
            gemm(w)
            clique.all_reduce(outs, outs)


def make_chunked(chunks):
    per = tokens // chunks
    views = [[o[c * per:(c + 1) * per] for o in outs] for c in range(chunks)]
    evg = [torch.cuda.Event() for _ in range(chunks)]
    evc = torch.cuda.Event()

    def run():
        for _ in range(layers):
            for w in (0, 1):
                main.wait_event(evc)
                for c in range(chunks):
                    gemm(w, slice(c * per, (c + 1) * per))
                    evg[c].record(main)
                    side.wait_event(evg[c])
                    clique.all_reduce(views[c], views[c], stream=side)
                evc.record(side)
        main.wait_event(evc)
    return run


def gemm_only():
    for _ in range(layers):
        gemm(0)
        gemm(1)


def comm_only():
    for _ in range(layers):
        clique.all_reduce(outs, outs)
        clique.all_reduce(outs, outs)


print(json.dumps({"gemm_ms_per_layer": round(timed(gemm_only), 3),
                  "comm_ms_per_layer": round(timed(comm_only), 3),
                  "sequential_ms_per_layer": round(timed(sequential), 3)}), flush=True)
for chunks in (2, 4, 8):
    for ctas in (0, 16, 32, 64, 96):
        clique.set_nvlink_ctas(ctas)
        print(json.dumps({"chunks": chunks, "fold_ctas": ctas or "auto",
                          "ms_per_layer": round(timed(make_chunked(chunks)), 3)}), flush=True)
clique.set_nvlink_ctas(0)
