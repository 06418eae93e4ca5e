"""Messages past the 32-bit byte range, both executors.

Per-rank sends of 2.5 GiB (+ a ragged tail) put the PCIe slice, the rank
chunks and the AllGather's recv blocks at byte offsets above 2^31 and, for the
AllGather's 5 GiB recv buffers, above 2^32: any 32-bit offset or count in the
partition, the kernels' indexing or the staging pipeline shows up as a wrong
result.  Integer-valued inputs keep the sums exact in any order, so torch's
own sum is the check at this size (the oracle would take minutes).
"""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.links import PathKind  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

GIB = 1 << 30


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    flx.load_library()
    yield
    torch.cuda.empty_cache()


@pytest.mark.parametrize("loopback", [False, True])
def test_allreduce_past_2gib_per_rank(loopback):
    n, count = 2, (5 * GIB // 2) // 4 + 3  # 2.5 GiB + 12 B of fp32 per rank
    g = torch.Generator(device="cuda").manual_seed(77)
    sends = [torch.randint(-1024, 1024, (count,), device="cuda", generator=g).float()
             for _ in range(n)]
    recvs = [torch.empty_like(s) for s in sends]
    exact = sends[0] + sends[1]
    with flx.Clique(n, loopback=loopback) as c:
        c.set_shares(CollectiveOp.ALLREDUCE, (990, 10, 0))
        c.all_reduce(sends, recvs)
        torch.cuda.synchronize()
        assert c.path_bytes()[PathKind.PCIE_STAGED] > 0
    for r in recvs:
        assert torch.equal(r, exact)
    del sends, recvs, exact


@pytest.mark.parametrize("loopback", [False, True])
def test_allgather_past_4gib_recv(loopback):
    n, count = 2, (5 * GIB // 2) // 2 + 1  # 2.5 GiB + 2 B of bf16 per rank -> 5 GiB recv
    g = torch.Generator(device="cuda").manual_seed(78)
    sends = [torch.randint(-30000, 30000, (count,), device="cuda", generator=g,
                           dtype=torch.int16).view(torch.bfloat16) for _ in range(n)]
    recvs = [torch.empty(n * count, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    with flx.Clique(n, loopback=loopback) as c:
        c.set_shares(CollectiveOp.ALLGATHER, (990, 10, 0))
        c.all_gather(sends, recvs)
        torch.cuda.synchronize()
        assert c.path_bytes()[PathKind.PCIE_STAGED] > 0
    for r in recvs:
        for p in range(n):
            assert torch.equal(r[p * count:(p + 1) * count].view(torch.int16),
                               sends[p].view(torch.int16))
    del sends, recvs


@pytest.mark.parametrize("loopback", [False, True])
def test_reducescatter_and_alltoall_past_4gib_send(loopback):
    n, block = 2, (5 * GIB // 2) // 4 + 1  # 2 blocks of 2.5 GiB + 4 B fp32: 5 GiB sends
    g = torch.Generator(device="cuda").manual_seed(79)
    sends = [torch.randint(-1024, 1024, (n * block,), device="cuda", generator=g).float()
             for _ in range(n)]
    with flx.Clique(n, loopback=loopback) as c:
        for op in (CollectiveOp.REDUCESCATTER, CollectiveOp.ALLTOALL):
            c.set_shares(op, (990, 10, 0))
        rs = [torch.empty(block, device="cuda") for _ in range(n)]
        c.reduce_scatter(sends, rs)
        torch.cuda.synchronize()
        for r in range(n):
            want = sends[0][r * block:(r + 1) * block] + sends[1][r * block:(r + 1) * block]
            assert torch.equal(rs[r], want)
        del rs, want
        a2a = [torch.empty_like(s) for s in sends]
        c.all_to_all(sends, a2a)
        torch.cuda.synchronize()
        for r in range(n):
            for p in range(n):
                assert torch.equal(a2a[r][p * block:(p + 1) * block],
                                   sends[p][r * block:(r + 1) * block])
    del sends, a2a
