"""The widest world the library takes (FLX_MAX_VIRTUAL_RANKS = 16), both
executors, all four collectives, with a PCIe share, against the oracle.  At 16
ranks the rank kernels' peer signalling uses every one of warp 0's 16 lanes per
flag kind (cta_signal_peers / cta_wait_peers) and loopback fits 16 CTAs per rank."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

from test_gpu_parity import OPS, TORCH_DT, _inputs, _np  # noqa: E402

N = 16


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    flx.load_library()
    oracle.build()


@pytest.mark.parametrize("loopback", [False, True])
@pytest.mark.parametrize("dtype,op,count", [(7, "sum", 300007), (9, "sum", 1 << 17),
                                            (2, "max", 65536 + 5)])
def test_allreduce_16_ranks(loopback, dtype, op, count):
    g = (900, 100, 0)
    cpu = _inputs(N, count, dtype, 16 + dtype)
    s = [h.cuda() for h in cpu]
    r = [torch.empty_like(x) for x in s]
    with flx.Clique(N, loopback=loopback) as c:
        c.set_shares(CollectiveOp.ALLREDUCE, g)
        c.all_reduce(s, r, op=op)
        torch.cuda.synchronize()
        align = c.comms[0].alignment(CollectiveOp.ALLREDUCE)
    want = oracle.allreduce([_np(h, dtype) for h in cpu], dtype, OPS[op], g, align)
    for k in range(N):
        np.testing.assert_array_equal(_np(r[k].cpu(), dtype), want[k], err_msg=f"rank {k}")


@pytest.mark.parametrize("loopback", [False, True])
def test_gather_scatter_alltoall_16_ranks(loopback):
    g = (950, 50, 0)
    dtype, count = 7, 16 * 4099
    cpu = _inputs(N, count, dtype, 77, integer=True)
    s = [h.cuda() for h in cpu]
    with flx.Clique(N, loopback=loopback) as c:
        for op in (CollectiveOp.ALLGATHER, CollectiveOp.REDUCESCATTER, CollectiveOp.ALLTOALL):
            c.set_shares(op, g)
        ag = [torch.empty(N * count, device="cuda") for _ in range(N)]
        c.all_gather(s, ag)
        rs = [torch.empty(count // N, device="cuda") for _ in range(N)]
        c.reduce_scatter(s, rs)
        a2a = [torch.empty_like(x) for x in s]
        c.all_to_all(s, a2a)
        torch.cuda.synchronize()
    full = torch.cat(cpu)
    total = torch.stack([h.double() for h in cpu]).sum(0)
    blk = count // N
    for k in range(N):
        assert torch.equal(ag[k].cpu(), full), k
        # integer-valued inputs: the sum is exact in any order
        assert torch.equal(rs[k].cpu().double(), total[k * blk:(k + 1) * blk]), k
        want = torch.cat([cpu[q][k * blk:(k + 1) * blk] for q in range(N)])
        assert torch.equal(a2a[k].cpu(), want), k
