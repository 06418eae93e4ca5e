"""Seeded random SEQUENCES on one long-lived communicator per executor: mixed
collectives, sizes (one-shot, two-shot, multi-round with 1 MiB slots), dtypes,
shares (PCIe on and off), in-place and timing on/off, back to back without a
sync between calls.  Every result is checked bit-for-bit against the oracle, so
the cross-call state machines (device epochs, slot regions, one-shot parity,
PCIe counter semaphores, staging reuse) are exercised the way an application
drives them rather than one fresh communicator per case."""

import os
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

from test_gpu_parity import OPS, TORCH_DT, _inputs, _np  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    flx.load_library()
    oracle.build()


def _plan(seed, calls):
    rng = random.Random(seed)
    out = []
    for _ in range(calls):
        coll = rng.choice(["allreduce"] * 3 + ["allgather", "reducescatter", "alltoall"])
        dtype = rng.choice([2, 6, 7, 9])
        op = rng.choice(["sum", "max", "min"]) if coll in ("allreduce", "reducescatter") else "sum"
        count = rng.choice([3, 1000, 16384, 65536, 300001, 1 << 19])
        g = rng.choice([1000, 1000, 950, 800])
        out.append((coll, dtype, op, count, (g, 1000 - g, 0), rng.random() < 0.3,
                    rng.random() < 0.2))
    return out


@pytest.mark.parametrize("n", [3, 8])
@pytest.mark.parametrize("loopback", [False, True])
def test_random_sequence_on_one_communicator(loopback, n):
    os.environ["FLX_SLOT_MB"] = "1"  # multi-round calls in the multi-rank engine
    try:
        c = flx.Clique(n, loopback=loopback)
    finally:
        del os.environ["FLX_SLOT_MB"]
    pending = []
    with c:
        calls = int(os.environ.get("FLX_SEQ_CALLS", "80"))  # soak runs raise it
        for i, (coll, dtype, op, count, g, inplace, untimed) in enumerate(
                _plan(7 + 2 * loopback + n + 1000 * int(os.environ.get("FLX_SEQ_SEED", "0")),
                      calls)):
            c.set_shares(CollectiveOp(coll), g)
            c.set_timing(not untimed)
            align = c.comms[0].alignment(CollectiveOp(coll))
            seed = 1000 + i
            if coll == "allreduce":
                cpu = _inputs(n, count, dtype, seed)
                s = [h.cuda() for h in cpu]
                r = s if inplace else [torch.empty_like(x) for x in s]
                c.all_reduce(s, r, op=op)
                want = lambda cpu=cpu, dtype=dtype, op=op, g=g, align=align: oracle.allreduce(
                    [_np(h, dtype) for h in cpu], dtype, OPS[op], g, align)
            elif coll == "allgather":
                cpu = _inputs(n, count, dtype, seed)
                s = [h.cuda() for h in cpu]
                r = [torch.empty(n * count, dtype=TORCH_DT[dtype], device="cuda") for _ in range(n)]
                c.all_gather(s, r)
                want = lambda cpu=cpu, dtype=dtype, g=g, align=align: oracle.allgather(
                    [_np(h, dtype) for h in cpu], dtype, g, align)
            elif coll == "alltoall":
                cpu = _inputs(n, n * count, dtype, seed)
                s = [h.cuda() for h in cpu]
                r = [torch.empty_like(x) for x in s]
                c.all_to_all(s, r)
                want = lambda cpu=cpu, dtype=dtype, g=g, align=align: oracle.alltoall(
                    [_np(h, dtype) for h in cpu], dtype, g, align)
            else:
                cpu = _inputs(n, n * count, dtype, seed)
                s = [h.cuda() for h in cpu]
                r = [torch.empty(count, dtype=TORCH_DT[dtype], device="cuda") for _ in range(n)]
                c.reduce_scatter(s, r, op=op)
                want = lambda cpu=cpu, dtype=dtype, op=op, g=g, align=align: \
                    oracle.reducescatter([_np(h, dtype) for h in cpu], dtype, OPS[op], g, align)
            pending.append((i, coll, r, dtype, want, s))  # keep s alive until checked
            if len(pending) == 6 or i == calls - 1:  # several calls in flight between checks
                torch.cuda.synchronize()
                for j, cl, rr, dt, wf, _ in pending:
                    w = wf()
                    for k in range(n):
                        np.testing.assert_array_equal(_np(rr[k], dt), w[k],
                                                      err_msg=f"call {j} ({cl}) rank {k}")
                pending.clear()


def test_two_communicators_interleaved():
    # e.g. a TP and a DP group in one process: a virtual clique and a loopback
    # world on the same GPU, calls interleaved without syncs, no cross-talk
    n = 4
    a = flx.Clique(n)
    b = flx.Clique(n, loopback=True)
    try:
        for c in (a, b):
            c.set_shares(CollectiveOp.ALLREDUCE, (900, 100, 0))
        outs = []
        for it in range(6):
            for c, count in ((a, 70001 + it), (b, 123457 - it)):
                cpu = _inputs(n, count, 7, 500 + it * 2 + (c is b))
                s = [h.cuda() for h in cpu]
                r = [torch.empty_like(x) for x in s]
                c.all_reduce(s, r)
                outs.append((c, cpu, r, s))
        torch.cuda.synchronize()
        for c, cpu, r, _ in outs:
            want = oracle.allreduce([h.numpy() for h in cpu], 7, 0, (900, 100, 0),
                                    c.comms[0].alignment(CollectiveOp.ALLREDUCE))
            for k in range(n):
                np.testing.assert_array_equal(_np(r[k], 7), want[k])
    finally:
        a.destroy()
        b.destroy()
