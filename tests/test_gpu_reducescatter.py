"""GPU parity of ReduceScatter in both executors, vs the oracle."""

import ctypes
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.links import PathKind  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

from test_gpu_parity import OPS, TORCH_DT, _inputs, _np  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    flx.load_library()
    oracle.build()


def _run(n, count, dtype, op, granules, loopback, inplace=False, calls=1, seed=0):
    cpu = _inputs(n, n * count, dtype, seed)
    sends = [t.cuda() for t in cpu]
    if inplace:
        recvs = [sends[r][r * count:(r + 1) * count] for r in range(n)]
    else:
        recvs = [torch.empty(count, dtype=TORCH_DT[dtype], device="cuda") for _ in range(n)]
    with flx.Clique(n, loopback=loopback) as c:
        c.set_shares(CollectiveOp.REDUCESCATTER, granules)
        for _ in range(calls):
            if inplace:
                for s, h in zip(sends, cpu):
                    s.copy_(h)
            c.reduce_scatter(sends, recvs, op=op)
        torch.cuda.synchronize()
        got = [_np(r.contiguous(), dtype) for r in recvs]
        pb = c.path_bytes()
        align = c.comms[0].alignment(CollectiveOp.REDUCESCATTER)
    want = oracle.reducescatter([_np(h, dtype) for h in cpu], dtype, OPS[op], granules, align)
    return got, want, pb


CASES = [
    (2, 4096, 7, "sum", (1000, 0, 0)),
    (8, 1 << 16, 7, "sum", (1000, 0, 0)),
    (8, (1 << 17) + 5, 9, "sum", (900, 100, 0)),
    (4, 1 << 17, 6, "max", (800, 200, 0)),
    (3, 30001, 2, "sum", (700, 300, 0)),
    (8, 1, 7, "sum", (1000, 0, 0)),
    (5, 0, 7, "sum", (1000, 0, 0)),
]


@pytest.mark.parametrize("loopback", [False, True])
@pytest.mark.parametrize("n,count,dtype,op,granules", CASES)
def test_reduce_scatter_matches_oracle(loopback, n, count, dtype, op, granules):
    got, want, pb = _run(n, count, dtype, op, granules, loopback, seed=n + dtype, calls=2)
    for r in range(n):
        np.testing.assert_array_equal(got[r], want[r], err_msg=f"rank {r}")
    if granules[1] and count * 2 >= 8192:
        assert pb[PathKind.PCIE_STAGED] > 0


@pytest.mark.parametrize("loopback", [False, True])
def test_reduce_scatter_in_place(loopback):
    got, want, _ = _run(4, (1 << 16) + 3, 7, "sum", (850, 150, 0), loopback, inplace=True)
    for r in range(4):
        np.testing.assert_array_equal(got[r], want[r])


def test_mixed_collectives_share_flags_and_staging():
    # AllReduce, AllGather, ReduceScatter and AllToAll interleaved on one
    # loopback world (shared epochs/semaphores across protocols; an AllToAll
    # right before an AllReduce must not move the outbox guard), every result exact
    n, count = 4, (1 << 16) + 1
    g = (900, 100, 0)
    cpu = _inputs(n, n * count, 7, 21)
    with flx.Clique(n, loopback=True) as w:
        for op in CollectiveOp:
            w.set_shares(op, g)
        for _ in range(3):
            s = [h.cuda() for h in cpu]
            ar = [torch.empty_like(x) for x in s]
            w.all_reduce(s, ar)
            ag_in = [x[:count] for x in s]
            ag = [torch.empty(n * count, device="cuda") for _ in range(n)]
            w.all_gather(ag_in, ag)
            rs = [torch.empty(count, device="cuda") for _ in range(n)]
            w.reduce_scatter(s, rs)
            a2a = [torch.empty_like(x) for x in s]
            w.all_to_all(s, a2a)
            torch.cuda.synchronize()
            want_ar = oracle.allreduce([h.numpy() for h in cpu], 7, 0, g, n * 4096)
            want_ag = oracle.allgather([h.numpy()[:count] for h in cpu], 7, g, 4096)
            want_rs = oracle.reducescatter([h.numpy() for h in cpu], 7, 0, g, 4096)
            want_a2a = oracle.alltoall([h.numpy() for h in cpu], 7, g,
                                       w.comms[0].alignment(CollectiveOp.ALLTOALL))
            for r in range(n):
                np.testing.assert_array_equal(_np(ar[r], 7), want_ar[r])
                np.testing.assert_array_equal(_np(ag[r], 7), want_ag[r])
                np.testing.assert_array_equal(_np(rs[r], 7), want_rs[r])
                np.testing.assert_array_equal(_np(a2a[r], 7), want_a2a[r])


@pytest.mark.parametrize("loopback", [False, True])
@pytest.mark.parametrize("n,count,dtype,granules", [
    (2, 4096, 7, (1000, 0, 0)), (8, (1 << 15) + 3, 9, (900, 100, 0)), (3, 20001, 0, (600, 400, 0)),
])
def test_all_to_all_matches_oracle(loopback, n, count, dtype, granules):
    cpu = _inputs(n, n * count, dtype, n * 7 + dtype)
    sends = [h.cuda() for h in cpu]
    recvs = [torch.empty_like(s) for s in sends]
    with flx.Clique(n, loopback=loopback) as c:
        c.set_shares(CollectiveOp.ALLTOALL, granules)
        for _ in range(2):
            c.all_to_all(sends, recvs)
        torch.cuda.synchronize()
        align = c.comms[0].alignment(CollectiveOp.ALLTOALL)
        got = [_np(r, dtype) for r in recvs]
        with pytest.raises(ValueError):
            c.all_to_all(sends, sends)  # in place is rejected
    want = oracle.alltoall([_np(h, dtype) for h in cpu], dtype, granules, align)
    for r in range(n):
        np.testing.assert_array_equal(got[r], want[r])


def test_nccl_reduce_scatter_symbol():
    shim = flx.library_path().parent / "libflexlink_nccl.so"
    if not shim.exists():
        pytest.skip("nccl shim not built")
    S = ctypes.CDLL(str(shim))
    n, count = 4, 5000
    cpu = _inputs(n, n * count, 9, 3)
    sends = [t.cuda() for t in cpu]
    recvs = [torch.empty(count, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    comms = (ctypes.c_void_p * n)()
    assert S.ncclCommInitAll(comms, n, (ctypes.c_int * n)(*([0] * n))) == 0
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert S.ncclGroupStart() == 0
    for i in range(n):
        assert S.ncclReduceScatter(ctypes.c_void_p(sends[i].data_ptr()),
                                   ctypes.c_void_p(recvs[i].data_ptr()), ctypes.c_size_t(count),
                                   9, 0, ctypes.c_void_p(comms[i]), stream) == 0
    assert S.ncclGroupEnd() == 0
    torch.cuda.synchronize()
    want = oracle.reducescatter([_np(h, 9) for h in cpu], 9, 0)
    for r in range(n):
        np.testing.assert_array_equal(_np(recvs[r], 9), want[r])
    for i in range(n):
        S.ncclCommDestroy(ctypes.c_void_p(comms[i]))
