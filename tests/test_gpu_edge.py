"""Zero-length collectives are successful no-ops (NCCL's rule) in both
executors, for every collective, and leave the communicator in step: a normal
call right after is exact (the multi-rank engine's per-CTA epochs must not
drift on an empty call)."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    flx.load_library()


@pytest.mark.parametrize("loopback", [False, True])
def test_zero_length_calls_then_a_normal_one(loopback):
    n = 4
    with flx.Clique(n, loopback=loopback) as c:
        for op in CollectiveOp:
            c.set_shares(op, (900, 100, 0))
        e = [torch.empty(0, device="cuda") for _ in range(n)]
        for _ in range(2):
            c.all_reduce(e, [torch.empty(0, device="cuda") for _ in range(n)])
            c.all_gather(e, [torch.empty(0, device="cuda") for _ in range(n)])
            c.reduce_scatter(e, [torch.empty(0, device="cuda") for _ in range(n)])
            c.all_to_all(e, [torch.empty(0, device="cuda") for _ in range(n)])
        torch.cuda.synchronize()
        count = (1 << 18) + 12
        g = torch.Generator(device="cuda").manual_seed(5)
        s = [torch.randint(-50, 50, (count,), device="cuda", generator=g).float() for _ in range(n)]
        r = [torch.empty_like(x) for x in s]
        c.all_reduce(s, r)
        out = [torch.empty(n * count, device="cuda") for _ in range(n)]
        c.all_gather(s, out)
        torch.cuda.synchronize()
    want = torch.stack(s).sum(0)
    for k in range(n):
        assert torch.equal(r[k], want), k
        assert torch.equal(out[k], torch.cat(s)), k


def test_interleaved_communicators_on_one_gpu():
    # two multi-rank worlds (loopback) and a virtual-rank clique alive at once,
    # calls interleaved: per-world scratch, flags, epochs and tuner state never
    # cross, and every result is exact
    n, count = 4, (1 << 20) + 4
    g = torch.Generator(device="cuda").manual_seed(9)
    with flx.Clique(n, loopback=True) as a, flx.Clique(n, loopback=True) as b, \
            flx.Clique(n) as v:
        for c in (a, b, v):
            c.set_shares(CollectiveOp.ALLREDUCE, (900, 100, 0))
        for it in range(4):
            data = {}
            for name, c in (("a", a), ("b", b), ("v", v)):
                s = [torch.randint(-99, 100, (count + it,), device="cuda", generator=g).float()
                     for _ in range(n)]
                r = [torch.empty_like(x) for x in s]
                c.all_reduce(s, r)
                data[name] = (s, r)
            torch.cuda.synchronize()
            for name, (s, r) in data.items():
                want = torch.stack(s).sum(0)
                assert all(torch.equal(x, want) for x in r), (it, name)
