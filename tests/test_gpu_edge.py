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


@pytest.mark.parametrize("loopback", [False, True])
def test_entry_points_restore_the_callers_context(loopback):
    """NCCL's rule: a call leaves the caller's current CUDA context as it found
    it.  The entry points switch devices internally (cudaSetDevice); a thread
    that never touched CUDA — a framework's watchdog thread reading path times
    or async errors — must still have no context bound afterwards."""
    import threading

    import cuda.bindings.driver as drv

    def current():
        r, ctx = drv.cuCtxGetCurrent()
        assert r == drv.CUresult.CUDA_SUCCESS
        return int(ctx) if ctx is not None else 0

    n, count = 4, (1 << 16) + 5
    with flx.Clique(n, loopback=loopback) as c:
        c.set_shares(CollectiveOp.ALLREDUCE, (900, 100, 0))
        s = [torch.ones(count, device="cuda") for _ in range(n)]
        r = [torch.empty_like(x) for x in s]
        before = current()
        c.all_reduce(s, r)
        assert current() == before != 0
        torch.cuda.synchronize()
        seen = {}

        def watchdog():
            seen["start"] = current()
            seen["times"] = c.comms[0].path_times()
            seen["err"] = c.comms[0].async_error()
            seen["end"] = current()

        t = threading.Thread(target=watchdog)
        t.start()
        t.join()
        assert seen["start"] == 0 and seen["end"] == 0, seen
        assert seen["err"] == 0 and seen["times"][0] > 0
        assert all(torch.equal(x, torch.full_like(x, n)) for x in r)


@pytest.mark.parametrize("loopback", [False, True])
def test_broadcast_is_bit_exact_for_every_dtype(loopback):
    """flxBroadcast / ncclBroadcast: one striped MAX-over-uint8 AllReduce of the
    bytes with zeros from the non-roots — the root's bits everywhere, -0.0 and
    NaN payloads included, any size, in place or not."""
    n = 4
    with flx.Clique(n, loopback=loopback) as c:
        c.set_shares(CollectiveOp.ALLREDUCE, (900, 100, 0))
        for dt, count in ((torch.float32, (1 << 20) + 3), (torch.bfloat16, 777),
                          (torch.int64, 5), (torch.uint8, 4096 * 3 + 1)):
            for root in (0, n - 1):
                g = torch.Generator(device="cuda").manual_seed(root + count)
                sends = [torch.randint(-100, 100, (count,), device="cuda", generator=g).to(dt)
                         for _ in range(n)]
                if dt == torch.float32:
                    bits = sends[root].view(torch.int32)
                    bits[0] = -2147483648            # -0.0
                    bits[1] = 0x7FC00123              # a NaN with a payload
                want = sends[root].clone()
                recvs = [torch.full_like(s, 7) for s in sends]
                c.broadcast(sends, recvs, root=root)
                torch.cuda.synchronize()
                for r in recvs:
                    assert torch.equal(r.view(torch.uint8), want.view(torch.uint8)), (dt, root)
                c.broadcast(sends, root=root)  # in place
                torch.cuda.synchronize()
                for s in sends:
                    assert torch.equal(s.view(torch.uint8), want.view(torch.uint8)), (dt, root)


@pytest.mark.parametrize("loopback", [False, True])
def test_average_is_the_striped_sum_divided(loopback):
    """FLX_OP_AVG (== ncclAvg) on AllReduce and ReduceScatter: the rank-order
    fold (fp32 accumulation, one rounding for 16-bit types), then one division
    by nranks on the caller's stream — C division for integers."""
    n, count = 3, (1 << 18) + 2  # 3 equal ReduceScatter blocks
    with flx.Clique(n, loopback=loopback) as c:
        for op in (CollectiveOp.ALLREDUCE, CollectiveOp.REDUCESCATTER):
            c.set_shares(op, (900, 100, 0))
        g = torch.Generator(device="cuda").manual_seed(11)
        for dt in (torch.float32, torch.bfloat16, torch.int32):
            if dt == torch.int32:
                sends = [torch.randint(-10**6, 10**6, (count,), device="cuda", generator=g,
                                       dtype=torch.int32) for _ in range(n)]
            else:
                sends = [torch.randn(count, device="cuda", generator=g).to(dt) for _ in range(n)]
            acc = sends[0].double() if dt == torch.int32 else sends[0].float()
            for x in sends[1:]:
                acc = acc + (x.double() if dt == torch.int32 else x.float())
            if dt == torch.int32:
                want = torch.div(acc.long(), n, rounding_mode="trunc").to(dt)
            else:
                # IEEE division by a tensor (torch divides by a scalar through its
                # reciprocal, which can differ in the last bit)
                q = acc.to(dt).float()
                want = (q / torch.full_like(q, n)).to(dt)
            recvs = [torch.empty_like(x) for x in sends]
            c.all_reduce(sends, recvs, op="avg")
            blk = count // n
            rs = [torch.empty(blk, device="cuda", dtype=dt) for _ in range(n)]
            c.reduce_scatter(sends, rs, op="avg")
            torch.cuda.synchronize()
            for r in recvs:
                assert torch.equal(r, want), dt
            for i, r in enumerate(rs):
                assert torch.equal(r, want[i * blk:(i + 1) * blk]), dt


@pytest.mark.parametrize("loopback", [False, True])
def test_reduce_lands_on_the_root_only(loopback):
    """flxReduce / ncclReduce: the striped fold lands in the root's recv; the
    other ranks' recvs are untouched (their result goes to stream-ordered
    scratch); in place on the root; AVG and MAX too."""
    n, count = 4, (1 << 18) + 9
    with flx.Clique(n, loopback=loopback) as c:
        c.set_shares(CollectiveOp.ALLREDUCE, (900, 100, 0))
        g = torch.Generator(device="cuda").manual_seed(13)
        sends = [torch.randint(-500, 500, (count,), device="cuda", generator=g).float()
                 for _ in range(n)]
        for op, want in (("sum", torch.stack(sends).sum(0)), ("max", torch.stack(sends).amax(0)),
                         ("avg", torch.stack(sends).sum(0) / 4)):
            for root in (0, 2):
                recvs = [torch.full_like(x, 3.0) for x in sends]
                c.reduce(sends, recvs, op=op, root=root)
                torch.cuda.synchronize()
                for r, x in enumerate(recvs):
                    assert torch.equal(x, want if r == root else torch.full_like(x, 3.0)), (op, r)
        keep = [x.clone() for x in sends]
        c.reduce(sends, sends, root=1)  # in place
        torch.cuda.synchronize()
        assert torch.equal(sends[1], torch.stack(keep).sum(0))
        assert all(torch.equal(sends[r], keep[r]) for r in (0, 2, 3))


@pytest.mark.parametrize("loopback", [False, True])
def test_gather_and_scatter(loopback):
    """flxGather / flxScatter (NCCL 2.28's ncclGather / ncclScatter): the root's
    recv holds every rank's block in rank order; every rank receives its block
    of the root's send; non-root recvs / sends are not touched."""
    n, count = 4, (1 << 16) + 5
    with flx.Clique(n, loopback=loopback) as c:
        for op in (CollectiveOp.ALLGATHER, CollectiveOp.ALLTOALL):
            c.set_shares(op, (900, 100, 0))
        g = torch.Generator(device="cuda").manual_seed(17)
        for dt in (torch.float32, torch.bfloat16):
            sends = [torch.randn(count, device="cuda", generator=g).to(dt) for _ in range(n)]
            for root in (0, 3):
                recvs = [torch.full((n * count,), 5.0, device="cuda", dtype=dt) for _ in range(n)]
                c.gather(sends, recvs, root=root)
                torch.cuda.synchronize()
                for r, x in enumerate(recvs):
                    want = torch.cat(sends) if r == root else torch.full_like(x, 5.0)
                    assert torch.equal(x, want), ("gather", dt, root, r)
                big = [torch.randn(n * count, device="cuda", generator=g).to(dt) for _ in range(n)]
                keep = [b.clone() for b in big]
                outs = [torch.empty(count, device="cuda", dtype=dt) for _ in range(n)]
                c.scatter(big, outs, root=root)
                torch.cuda.synchronize()
                for r, x in enumerate(outs):
                    assert torch.equal(x, keep[root][r * count:(r + 1) * count]), ("scatter", dt, r)
                assert all(torch.equal(b, k) for b, k in zip(big, keep))


def test_failed_group_with_reduce_scratch_is_refused_cleanly():
    """A group whose members do not all take part fails at its end; flxReduce's
    non-root scratch in it is released (stream-ordered) and the communicator
    keeps working."""
    n, count = 4, 1 << 16
    L = flx.load_library()
    with flx.Clique(n) as c:
        s = [torch.ones(count, device="cuda") * (i + 1) for i in range(n)]
        r = [torch.zeros(count, device="cuda") for _ in range(n)]
        assert L.flxGroupStart() == 0
        c.comms[1].reduce(s[1], r[1], root=0)  # non-root: scratch allocated
        c.comms[2].reduce(s[2], r[2], root=0)
        assert L.flxGroupEnd() != 0  # ranks 0 and 3 never joined
        torch.cuda.synchronize()
        c.reduce(s, r, root=0)
        torch.cuda.synchronize()
        assert torch.equal(r[0], torch.full_like(r[0], n * (n + 1) / 2))
