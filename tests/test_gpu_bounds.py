"""Out-of-bounds write guard (compute-sanitizer is closed on this pool).

Every send/recv tensor is a slice in the middle of a larger allocation whose
margins hold a canary; after each collective (both executors, odd sizes,
PCIe shares, every collective) the result must be exact AND every canary byte
untouched."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

CANARY = -12345.5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    flx.load_library()
    oracle.build()


OFF = {"aligned": 4100, "misaligned": 4101}  # 16 B aligned / 4 B aligned start
_mode = {"off": 4100}


def guarded(count, fill=None):
    off = _mode["off"]
    base = torch.full((count + 2 * off,), CANARY, device="cuda")
    view = base[off:off + count]
    if fill is not None:
        view.copy_(fill)
    return base, view


def check_canary(base, count):
    off = _mode["off"]
    head = base[:off]
    tail = base[off + count:]
    assert bool((head == CANARY).all()) and bool((tail == CANARY).all()), "out-of-bounds write"


@pytest.mark.parametrize("where", list(OFF))
@pytest.mark.parametrize("loopback", [False, True])
@pytest.mark.parametrize("n,count", [(3, 70001), (4, 4099), (8, 1 << 15)])
def test_no_write_outside_buffers(where, loopback, n, count):
    _mode["off"] = OFF[where]
    g = torch.Generator().manual_seed(n * 31 + count)
    host = [torch.randn(n * count, generator=g) for _ in range(n)]
    shares = (900, 100, 0)
    with flx.Clique(n, loopback=loopback) as c:
        for op in CollectiveOp:
            c.set_shares(op, shares)
        al = {op: c.comms[0].alignment(op) for op in CollectiveOp}
        sends = [guarded(n * count, h.cuda()) for h in host]
        s = [v for _, v in sends]
        # AllReduce
        recvs = [guarded(n * count) for _ in range(n)]
        c.all_reduce(s, [v for _, v in recvs])
        want = oracle.allreduce([h.numpy() for h in host], 7, 0, shares, al[CollectiveOp.ALLREDUCE])
        for (b, v), w in zip(recvs, want):
            check_canary(b, n * count)
            np.testing.assert_array_equal(v.cpu().numpy(), w)
        # AllGather (send = first block)
        recvs = [guarded(n * count) for _ in range(n)]
        c.all_gather([v[:count] for v in s], [v for _, v in recvs])
        want = oracle.allgather([h.numpy()[:count] for h in host], 7, shares,
                                al[CollectiveOp.ALLGATHER])
        for (b, v), w in zip(recvs, want):
            check_canary(b, n * count)
            np.testing.assert_array_equal(v.cpu().numpy(), w)
        # ReduceScatter
        recvs = [guarded(count) for _ in range(n)]
        c.reduce_scatter(s, [v for _, v in recvs])
        want = oracle.reducescatter([h.numpy() for h in host], 7, 0, shares,
                                    al[CollectiveOp.REDUCESCATTER])
        for (b, v), w in zip(recvs, want):
            check_canary(b, count)
            np.testing.assert_array_equal(v.cpu().numpy(), w)
        # AllToAll
        recvs = [guarded(n * count) for _ in range(n)]
        c.all_to_all(s, [v for _, v in recvs])
        want = oracle.alltoall([h.numpy() for h in host], 7, shares, al[CollectiveOp.ALLTOALL])
        for (b, v), w in zip(recvs, want):
            check_canary(b, n * count)
            np.testing.assert_array_equal(v.cpu().numpy(), w)
        torch.cuda.synchronize()
        for b, _ in sends:  # sends are read-only for every collective
            check_canary(b, n * count)
