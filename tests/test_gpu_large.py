"""Messages past 32-bit sizes: more than 2^31 elements and 4 GiB per rank, both
executors, with a PCIe share — every count, offset and grid computation must be
64-bit.  Integer-valued data, so the exact result is a torch sum on the GPU
(size-independent property; the oracle would take minutes at this size)."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.links import PathKind  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    flx.load_library()


def _ints(count, dtype, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randint(-8, 9, (count,), device="cuda", generator=g, dtype=torch.int8).to(dtype)


@pytest.mark.parametrize("loopback", [False, True])
def test_allreduce_bf16_past_2g_elements(loopback):
    n, count = 2, (1 << 31) + 19  # 4 GiB + 38 B of bf16 per rank
    s = [_ints(count, torch.bfloat16, r) for r in range(n)]
    want = (s[0].float() + s[1].float()).bfloat16()  # |sum| <= 16: exact in bf16
    with flx.Clique(n, loopback=loopback) as c:
        c.set_shares(CollectiveOp.ALLREDUCE, (950, 50, 0))
        c.all_reduce(s, s)  # in place
        torch.cuda.synchronize()
        pb = c.path_bytes()
    assert pb[PathKind.PCIE_STAGED] > (1 << 27)  # a real PCIe slice (~200 MiB)
    for r in range(n):
        assert torch.equal(s[r], want), r


@pytest.mark.parametrize("loopback", [False, True])
def test_allgather_past_4gib_output(loopback):
    n, count = 2, (1 << 30) + 7  # 2 GiB + 14 B of bf16 sent per rank: > 4 GiB gathered
    s = [_ints(count, torch.bfloat16, 10 + r) for r in range(n)]
    out = [torch.empty(n * count, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
    with flx.Clique(n, loopback=loopback) as c:
        c.set_shares(CollectiveOp.ALLGATHER, (950, 50, 0))
        c.all_gather(s, out)
        torch.cuda.synchronize()
    for r in range(n):
        assert torch.equal(out[r][:count], s[0]) and torch.equal(out[r][count:], s[1]), r


@pytest.mark.parametrize("loopback", [False, True])
def test_reducescatter_and_alltoall_past_2g_elements(loopback):
    n, blk = 2, (1 << 30) + 9  # blocks of 2 GiB + 18 B of bf16: 2^31 + 18 elements sent
    s = [_ints(n * blk, torch.bfloat16, 20 + r) for r in range(n)]
    rs = [torch.empty(blk, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
    with flx.Clique(n, loopback=loopback) as c:
        c.set_shares(CollectiveOp.REDUCESCATTER, (950, 50, 0))
        c.set_shares(CollectiveOp.ALLTOALL, (950, 50, 0))
        c.reduce_scatter(s, rs)
        torch.cuda.synchronize()
        for r in range(n):
            want = (s[0][r * blk:(r + 1) * blk].float() + s[1][r * blk:(r + 1) * blk].float())
            assert torch.equal(rs[r], want.bfloat16()), r
        del rs
        a2a = [torch.empty_like(x) for x in s]
        c.all_to_all(s, a2a)
        torch.cuda.synchronize()
    for r in range(n):
        for q in range(n):
            assert torch.equal(a2a[r][q * blk:(q + 1) * blk], s[q][r * blk:(r + 1) * blk]), (r, q)
