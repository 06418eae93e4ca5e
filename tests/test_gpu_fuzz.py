"""Seeded random sweep: collective x executor x dtype x op x shares x size x in-place,
each checked bit-for-bit against the CPU oracle (complements the hand-picked cases)."""

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

# FLX_FUZZ_CASES / FLX_FUZZ_SEED widen the sweep for soak runs (default: 48 cases)
RNG = random.Random(int(os.environ.get("FLX_FUZZ_SEED", "20261018")))
CASES = []
for i in range(int(os.environ.get("FLX_FUZZ_CASES", "48"))):
    coll = RNG.choice(["allreduce", "allgather", "reducescatter", "alltoall"])
    n = RNG.choice([2, 3, 4, 5, 8])
    dtype = RNG.choice([0, 2, 6, 7, 8, 9])
    op = RNG.choice(["sum", "max", "min", "prod"]) if coll in ("allreduce",
                                                               "reducescatter") else "sum"
    if op == "prod" and dtype in (6, 9):
        op = "sum"  # fp16/bf16 products overflow quickly; sum/max/min cover the fold
    count = RNG.choice([1, 17, 1000, 4099, 65536, 200003, 1 << 18])
    g = RNG.choice([1000, 980, 900, 700, 500])
    CASES.append((i, coll, n, dtype, op, count, (g, 1000 - g, 0), RNG.random() < 0.3,
                  RNG.random() < 0.4))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    flx.load_library()
    oracle.build()


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[1]}-n{c[2]}-t{c[3]}")
def test_fuzz_against_oracle(case):
    _, coll, n, dtype, op, count, granules, inplace, loopback = case
    seed = hash(case[:6]) & 0xFFFF
    with flx.Clique(n, loopback=loopback) as c:
        c.set_shares(CollectiveOp(coll), granules)
        align = c.comms[0].alignment(CollectiveOp(coll))
        if coll == "allreduce":
            cpu = _inputs(n, count, dtype, seed)
            s = [h.cuda() for h in cpu]
            r = s if inplace else [torch.empty_like(x) for x in s]
            c.all_reduce(s, r, op=op)
            want = oracle.allreduce([_np(h, dtype) for h in cpu], dtype, OPS[op], granules, align)
        elif coll == "allgather":
            cpu = _inputs(n, count, dtype, seed)
            r = [torch.empty(n * count, dtype=TORCH_DT[dtype], device="cuda") for _ in range(n)]
            if inplace:
                for k in range(n):
                    r[k][k * count:(k + 1) * count].copy_(cpu[k])
                s = [r[k][k * count:(k + 1) * count] for k in range(n)]
            else:
                s = [h.cuda() for h in cpu]
            c.all_gather(s, r)
            want = oracle.allgather([_np(h, dtype) for h in cpu], dtype, granules, align)
        elif coll == "alltoall":
            cpu = _inputs(n, n * count, dtype, seed)
            s = [h.cuda() for h in cpu]
            r = [torch.empty_like(x) for x in s]
            c.all_to_all(s, r)
            want = oracle.alltoall([_np(h, dtype) for h in cpu], dtype, granules, align)
        else:
            cpu = _inputs(n, n * count, dtype, seed)
            s = [h.cuda() for h in cpu]
            r = [s[k][k * count:(k + 1) * count] for k in range(n)] if inplace else \
                [torch.empty(count, dtype=TORCH_DT[dtype], device="cuda") for _ in range(n)]
            c.reduce_scatter(s, r, op=op)
            want = oracle.reducescatter([_np(h, dtype) for h in cpu], dtype, OPS[op], granules,
                                        align)
        torch.cuda.synchronize()
        for k in range(n):
            np.testing.assert_array_equal(_np(r[k].contiguous(), dtype), want[k],
                                          err_msg=f"rank {k}")
