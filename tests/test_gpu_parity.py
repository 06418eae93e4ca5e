"""GPU parity: the native striped collectives vs the CPU oracle, bit for bit.

Every case runs N virtual ranks on cuda:0 through the C-ABI (flxCommInitAll
with a repeated device + flxGroupStart/End) and compares each rank's result
with ``oracle.allreduce`` / ``oracle.allgather`` on the same seeded inputs and
the same shares.  Shares that put bytes on the PCIe path exercise the real
D2H -> pinned host -> H2D pipeline and its counter semaphores.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.links import PathKind  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp, partition  # noqa: E402

TORCH_DT = {0: torch.int8, 1: torch.uint8, 2: torch.int32, 3: torch.uint32, 4: torch.int64,
            5: torch.uint64, 6: torch.float16, 7: torch.float32, 8: torch.float64,
            9: torch.bfloat16}
NP_VIEW = {6: np.uint16, 9: np.uint16}
OPS = {"sum": 0, "prod": 1, "max": 2, "min": 3}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU boxes)")
    flx.load_library()
    oracle.build()
    yield


def _inputs(n, count, dtype, seed, integer=False):
    g = torch.Generator(device="cpu").manual_seed(seed)
    out = []
    for r in range(n):
        if dtype in (0, 1, 2, 3, 4, 5):
            lo, hi = (0, 7) if dtype in (1, 3, 5) else (-5, 6)
            t = torch.randint(lo, hi, (count,), generator=g, dtype=torch.int64)
            t = t.to(TORCH_DT[dtype])
        elif integer:
            t = torch.randint(-64, 65, (count,), generator=g).to(TORCH_DT[dtype])
        else:
            t = (torch.randn(count, generator=g, dtype=torch.float64) * 3).to(TORCH_DT[dtype])
        out.append(t)
    return out


def _np(t, dtype):
    a = t.cpu()
    if dtype in NP_VIEW:
        return a.view(torch.int16).numpy().view(np.uint16).copy()
    if dtype == 3:
        return a.view(torch.int32).numpy().view(np.uint32).copy()
    if dtype == 5:
        return a.view(torch.int64).numpy().view(np.uint64).copy()
    return a.numpy().copy()


def _run_allreduce(n, count, dtype, op, granules, inplace=False, offset=0, seed=0):
    cpu = _inputs(n, count + offset, dtype, seed)
    dev = [t.cuda() for t in cpu]
    sends = [d[offset:] for d in dev]
    recvs = sends if inplace else [torch.empty_like(s) for s in sends]
    with flx.Clique(n) as clique:
        clique.set_shares(CollectiveOp.ALLREDUCE, granules)
        clique.all_reduce(sends, recvs, op=op)
        torch.cuda.synchronize()
        got = [_np(r, dtype) for r in recvs]
        pbytes = clique.path_bytes()
        align = clique.comms[0].alignment(CollectiveOp.ALLREDUCE)
    want = oracle.allreduce([_np(c[offset:], dtype) for c in cpu], dtype, OPS[op],
                            granules=granules, alignment=align)
    return got, want, pbytes, align


CASES = [
    # (nranks, count, dtype, op, granules)
    (2, 4096, 7, "sum", (1000, 0, 0)),
    (8, 1 << 16, 7, "sum", (1000, 0, 0)),
    (8, 1 << 16, 9, "sum", (1000, 0, 0)),
    (8, 1 << 16, 6, "sum", (1000, 0, 0)),
    (8, (1 << 18) + 5, 7, "sum", (900, 100, 0)),
    (8, (1 << 18) + 3, 9, "sum", (850, 150, 0)),
    (4, 1 << 18, 8, "sum", (800, 200, 0)),
    (3, 100003, 7, "sum", (700, 300, 0)),
    (16, 1 << 15, 7, "sum", (900, 100, 0)),
    (5, 77777, 2, "sum", (900, 100, 0)),
    (8, 1 << 16, 4, "prod", (1000, 0, 0)),
    (8, 1 << 16, 0, "sum", (1000, 0, 0)),
    (8, 1 << 16, 1, "max", (900, 100, 0)),
    (6, 12345, 7, "max", (1000, 0, 0)),
    (6, 12345, 9, "min", (1000, 0, 0)),
    (7, 54321, 5, "sum", (1000, 0, 0)),
    (8, 1 << 16, 3, "min", (1000, 0, 0)),
    (2, 1 << 16, 7, "prod", (500, 500, 0)),
    (1, 1000, 7, "sum", (1000, 0, 0)),
    (8, 0, 7, "sum", (1000, 0, 0)),
    (8, 1, 7, "sum", (1000, 0, 0)),
    (8, 3, 9, "sum", (1000, 0, 0)),
]


@pytest.mark.parametrize("n,count,dtype,op,granules", CASES)
def test_allreduce_matches_oracle(n, count, dtype, op, granules):
    got, want, pbytes, align = _run_allreduce(n, count, dtype, op, granules, seed=n * 131 + dtype)
    for r in range(n):
        np.testing.assert_array_equal(got[r], want[r], err_msg=f"rank {r}")
    esz = torch.empty(0, dtype=TORCH_DT[dtype]).element_size()
    split = partition(count * esz, {k: g for k, g in zip(PathKind, granules)}, align)
    assert [pbytes[k] for k in PathKind] == [split.get(k, 0) for k in PathKind]


@pytest.mark.parametrize("dtype", [7, 9])
def test_allreduce_inplace(dtype):
    got, want, _, _ = _run_allreduce(8, (1 << 17) + 7, dtype, "sum", (880, 120, 0), inplace=True)
    for r in range(8):
        np.testing.assert_array_equal(got[r], want[r])


@pytest.mark.parametrize("dtype", [7, 9, 0])
def test_allreduce_misaligned_buffers(dtype):
    # 1-element offset breaks 16 B alignment -> scalar kernel path
    got, want, _, _ = _run_allreduce(4, 5000, dtype, "sum", (1000, 0, 0), offset=1)
    for r in range(4):
        np.testing.assert_array_equal(got[r], want[r])


def test_allreduce_fp32_matches_torch_fixed_order():
    # independent check: torch's own left fold in rank order gives the same bits
    cpu = _inputs(8, 1 << 16, 7, seed=7)
    dev = [t.cuda() for t in cpu]
    with flx.Clique(8) as clique:
        out = clique.all_reduce(dev, [torch.empty_like(d) for d in dev])
        torch.cuda.synchronize()
    acc = dev[0].clone()
    for d in dev[1:]:
        acc = acc + d
    for o in out:
        assert torch.equal(o, acc)


def _run_allgather(n, count, dtype, granules, inplace=False, seed=0):
    cpu = _inputs(n, count, dtype, seed)
    sends = [t.cuda() for t in cpu]
    if inplace:
        recvs = [torch.empty(n * count, dtype=TORCH_DT[dtype], device="cuda") for _ in range(n)]
        for r in range(n):
            recvs[r][r * count:(r + 1) * count].copy_(sends[r])
        sends = [recvs[r][r * count:(r + 1) * count] for r in range(n)]
    else:
        recvs = [torch.empty(n * count, dtype=TORCH_DT[dtype], device="cuda") for _ in range(n)]
    with flx.Clique(n) as clique:
        clique.set_shares(CollectiveOp.ALLGATHER, granules)
        clique.all_gather(sends, recvs)
        torch.cuda.synchronize()
        got = [_np(r, dtype) for r in recvs]
        align = clique.comms[0].alignment(CollectiveOp.ALLGATHER)
    want = oracle.allgather([_np(c, dtype) for c in cpu], dtype, granules=granules,
                            alignment=align)
    return got, want


@pytest.mark.parametrize("n,count,dtype,granules", [
    (2, 4096, 7, (1000, 0, 0)),
    (8, 1 << 16, 9, (1000, 0, 0)),
    (8, (1 << 18) + 1, 9, (900, 100, 0)),
    (3, 99999, 0, (800, 200, 0)),
    (16, 1 << 14, 7, (950, 50, 0)),
    (8, 1, 7, (1000, 0, 0)),
    (4, 0, 7, (1000, 0, 0)),
])
def test_allgather_matches_oracle(n, count, dtype, granules):
    got, want = _run_allgather(n, count, dtype, granules, seed=n + dtype)
    for r in range(n):
        np.testing.assert_array_equal(got[r], want[r])


def test_allgather_inplace():
    got, want = _run_allgather(8, (1 << 16) + 3, 9, (900, 100, 0), inplace=True)
    for r in range(8):
        np.testing.assert_array_equal(got[r], want[r])


def test_repeated_calls_reuse_staging_ring():
    # many calls through a 2-buffer ring with small chunks: counters keep advancing
    cpu = _inputs(4, 1 << 18, 7, seed=3)
    dev = [t.cuda() for t in cpu]
    want = oracle.allreduce([_np(c, 7) for c in cpu], 7, 0, granules=(600, 400, 0),
                            alignment=4 * 4096)
    with flx.Clique(4) as clique:
        clique.set_shares(CollectiveOp.ALLREDUCE, (600, 400, 0))
        clique.set_staging(64 << 10, 2)
        outs = [torch.empty_like(d) for d in dev]
        for _ in range(12):
            clique.all_reduce(dev, outs)
        torch.cuda.synchronize()
        for r in range(4):
            np.testing.assert_array_equal(_np(outs[r], 7), want[r])
        clique.set_staging(16 << 10, 1)  # single-buffer ring
        clique.all_reduce(dev, outs)
        torch.cuda.synchronize()
        for r in range(4):
            np.testing.assert_array_equal(_np(outs[r], 7), want[r])


def test_large_allreduce_exact_properties():
    # C1 shape (8 ranks x 256 MiB fp32) with integer-valued inputs: the sum is
    # exact in any order, so compare with torch's sum; all ranks identical.
    n, count = 8, 64 << 20
    g = torch.Generator(device="cuda").manual_seed(1000)
    sends = [torch.randint(-1024, 1024, (count,), device="cuda", generator=g).float()
             for _ in range(n)]
    recvs = [torch.empty_like(s) for s in sends]
    with flx.Clique(n) as clique:
        clique.set_shares(CollectiveOp.ALLREDUCE, (990, 10, 0))
        clique.all_reduce(sends, recvs)
        torch.cuda.synchronize()
        assert clique.path_bytes()[PathKind.PCIE_STAGED] > 0
    exact = torch.stack(sends).sum(0)
    for r in recvs:
        assert torch.equal(r, exact)


def test_config2_allgather_full_size_bitexact():
    # C2 shape: 8 ranks x 16,777,216 bf16 (32 MiB) -> 256 MiB gathered, with a
    # PCIe share: every rank's output must be the concatenation of all sends.
    n, count = 8, 16 << 20
    g = torch.Generator(device="cuda").manual_seed(1002)
    sends = [torch.randn(count, device="cuda", generator=g).bfloat16() for _ in range(n)]
    recvs = [torch.empty(n * count, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    with flx.Clique(n) as clique:
        clique.set_shares(CollectiveOp.ALLGATHER, (950, 50, 0))
        clique.all_gather(sends, recvs)
        torch.cuda.synchronize()
        assert clique.path_bytes()[PathKind.PCIE_STAGED] > 0
    want = torch.cat(sends).view(torch.int16)
    for r in recvs:
        assert torch.equal(r.view(torch.int16), want)


def test_config5_shape_bf16_allreduce_exact():
    # C5 shape: [65536, 5120] bf16 per rank (640 MiB), 8 ranks, PCIe share on.
    # Integer-valued inputs in [-16, 16): every partial sum is an integer of
    # magnitude <= 128, exact in bf16 and fp32, so the fold equals torch's sum
    # whatever the order -- a size-independent check at the full size.
    n, count = 8, 65536 * 5120
    g = torch.Generator(device="cuda").manual_seed(1005)
    sends = [torch.randint(-16, 16, (count,), device="cuda", generator=g).bfloat16()
             for _ in range(n)]
    with flx.Clique(n) as clique:
        clique.set_shares(CollectiveOp.ALLREDUCE, (980, 20, 0))
        exact = torch.stack(sends).float().sum(0).bfloat16()
        clique.all_reduce(sends, sends)  # in place, as the TP layer does
        torch.cuda.synchronize()
        assert clique.path_bytes()[PathKind.PCIE_STAGED] > 0
    for s in sends:
        assert torch.equal(s.view(torch.int16), exact.view(torch.int16))


def test_path_times_and_history():
    n = 8
    dev = [torch.randn(1 << 22, device="cuda") for _ in range(n)]
    outs = [torch.empty_like(d) for d in dev]
    with flx.Clique(n) as clique:
        clique.set_shares(CollectiveOp.ALLREDUCE, (980, 20, 0))
        for _ in range(5):
            clique.all_reduce(dev, outs)
        hist = clique.comms[0].path_times_history(16)
        assert len(hist) == 5
        for h in hist:
            assert h[PathKind.NVLINK] > 0 and h[PathKind.PCIE_STAGED] > 0
        rep = clique.report(CollectiveOp.ALLREDUCE, dev[0].numel() * 4)
        assert rep.total == max(rep.durations.values()) > 0


def test_stage1_on_real_path_converges_and_guards():
    from paper_2510_15882_b200.links import preset
    from paper_2510_15882_b200.stage1 import TunerConfig

    n = 8
    dev = [torch.randn(1 << 22, device="cuda") for _ in range(n)]
    outs = [torch.empty_like(d) for d in dev]
    with flx.Clique(n) as clique:
        topo = preset("B200").restricted([PathKind.NVLINK, PathKind.PCIE_STAGED])
        shares, trace, tuned, base = flx.tune_shares(
            clique, topo, CollectiveOp.ALLREDUCE, dev, outs,
            TunerConfig(max_iterations=30), warmup=1, repeats=3)
        assert trace.iterations >= 1
        assert sum(shares.as_dict().values()) == 1000
        # installed shares are what the next call uses, and results stay exact
        clique.all_reduce(dev, outs)
        torch.cuda.synchronize()
        acc = dev[0].clone()
        for d in dev[1:]:
            acc = acc + d
        for o in outs:
            assert torch.equal(o, acc)


def test_invalid_usage_is_loud():
    dev = [torch.zeros(16, device="cuda") for _ in range(2)]
    with flx.Clique(2) as clique:
        with pytest.raises(ValueError):
            clique.set_shares(CollectiveOp.ALLREDUCE, (500, 400, 0))  # sum != 1000
        with pytest.raises(ValueError):
            clique.set_shares(CollectiveOp.ALLREDUCE, (900, 0, 100))  # no NIC path
        with pytest.raises(ValueError):
            clique.comms[0].all_reduce(dev[0])  # virtual rank outside a group


def test_nccl_named_entry_points_drive_the_same_path():
    import ctypes

    shim = flx.library_path().parent / "libflexlink_nccl.so"
    if not shim.exists():
        pytest.skip("nccl shim not built")
    S = ctypes.CDLL(str(shim))
    n, count = 4, (1 << 16) + 3
    cpu = _inputs(n, count, 7, seed=5)
    sends = [t.cuda() for t in cpu]
    recvs = [torch.empty_like(s) for s in sends]
    comms = (ctypes.c_void_p * n)()
    devs = (ctypes.c_int * n)(*([0] * n))
    assert S.ncclCommInitAll(comms, n, devs) == 0
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert S.ncclGroupStart() == 0
    for i in range(n):
        assert S.ncclAllReduce(ctypes.c_void_p(sends[i].data_ptr()),
                               ctypes.c_void_p(recvs[i].data_ptr()), ctypes.c_size_t(count), 7, 0,
                               ctypes.c_void_p(comms[i]), stream) == 0
    assert S.ncclGroupEnd() == 0
    torch.cuda.synchronize()
    want = oracle.allreduce([_np(c, 7) for c in cpu], 7, 0)
    for r in range(n):
        np.testing.assert_array_equal(_np(recvs[r], 7), want[r])
    for i in range(n):
        assert S.ncclCommDestroy(ctypes.c_void_p(comms[i])) == 0


@pytest.mark.parametrize("granules", [(1000, 0, 0), (900, 100, 0)])
def test_cuda_graph_capture_and_replay(granules):
    # the striped call captured into a CUDA graph (PCIe handshake becomes graph
    # edges) and replayed on fresh inputs gives the oracle's bits every time
    n, count = 4, (1 << 18) + 5
    g = torch.Generator(device="cpu").manual_seed(11)
    sends = [torch.empty(count, device="cuda") for _ in range(n)]
    recvs = [torch.empty_like(s) for s in sends]
    with flx.Clique(n) as clique:
        clique.set_shares(CollectiveOp.ALLREDUCE, granules)
        clique.all_reduce(sends, recvs)  # eager warm-up sizes the staging ring
        torch.cuda.synchronize()
        stream = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            clique.all_reduce(sends, recvs)
        align = clique.comms[0].alignment(CollectiveOp.ALLREDUCE)
        for _ in range(3):
            host = [torch.randn(count, generator=g) for _ in range(n)]
            for s, h in zip(sends, host):
                s.copy_(h)
            graph.replay()
            torch.cuda.synchronize()
            want = oracle.allreduce([h.numpy() for h in host], 7, 0, granules, align)
            for r in range(n):
                np.testing.assert_array_equal(_np(recvs[r], 7), want[r])
        # eager calls still work (and still use the counter semaphores) afterwards
        clique.all_reduce(sends, recvs)
        torch.cuda.synchronize()
        for r in range(n):
            np.testing.assert_array_equal(_np(recvs[r], 7), want[r])


def test_validation_cache_never_reuses_stale_tensors():
    # Clique caches the checked tensor set; new tensor objects (even at recycled
    # addresses and ids, with another dtype or layout) are re-validated
    with flx.Clique(4) as c:
        for dt in (torch.float32, torch.bfloat16, torch.float32, torch.float16):
            xs = [torch.full((4096,), float(i + 1), device="cuda", dtype=dt) for i in range(4)]
            for _ in range(2):
                for i, x in enumerate(xs):
                    x.fill_(float(i + 1))
                c.all_reduce(xs, xs)
            torch.cuda.synchronize()
            assert all(bool((x == 10).all()) for x in xs), dt
            del xs
        ys = [torch.ones(64, 64, device="cuda").t() for _ in range(4)]  # non-contiguous
        with pytest.raises(ValueError):
            c.all_reduce(ys, ys)


@pytest.mark.parametrize("loopback", [False, True])
def test_group_call_with_one_stream_per_rank(loopback):
    # ncclGroupStart(); ncclAllReduce(..., stream_i) per rank; ncclGroupEnd():
    # the collective waits for every rank's stream (inputs produced there) and
    # every rank's stream waits for the collective (results consumed there)
    n, count = 4, (1 << 18) + 8  # partial sums stay below 2**24: exact in fp32
    L = flx.load_library()
    with flx.Clique(n, loopback=loopback) as c:
        c.set_shares(CollectiveOp.ALLREDUCE, (900, 100, 0))
        streams = [torch.cuda.Stream() for _ in range(n)]
        xs = [torch.empty(count, device="cuda") for _ in range(n)]
        outs = [torch.empty(count, device="cuda") for _ in range(n)]
        for it in range(3):
            for i, (st, x) in enumerate(zip(streams, xs)):
                with torch.cuda.stream(st):
                    torch.cuda._sleep(2000 * (i + 1))  # make producer timing differ
                    x.fill_(float(i + 1 + it))
            assert L.flxGroupStart() == 0
            for i, comm_i in enumerate(c.comms):
                comm_i.all_reduce(xs[i], outs[i], stream=streams[i])
            assert L.flxGroupEnd() == 0
            sums = []
            for st, o in zip(streams, outs):
                with torch.cuda.stream(st):
                    sums.append(o.sum())
            torch.cuda.synchronize()
            want = float(sum(i + 1 + it for i in range(n))) * count
            assert all(float(s) == want for s in sums), (it, [float(s) for s in sums], want)


@pytest.mark.parametrize("loopback", [False, True])
def test_group_with_several_collectives_per_rank(loopback):
    # NCCL allows several collectives between ncclGroupStart and ncclGroupEnd;
    # they run in issue order per rank (AllReduce, then an AllGather of its
    # result on the same stream, then a ReduceScatter), and a rank that issues a
    # different collective than rank 0 in the same slot is refused
    n, count = 4, (1 << 16) + 8
    L = flx.load_library()
    g = torch.Generator(device="cuda").manual_seed(3)
    xs = [torch.randint(-9, 10, (count,), device="cuda", generator=g).float() for _ in range(n)]
    red = [torch.empty(count, device="cuda") for _ in range(n)]
    gat = [torch.empty(n * count, device="cuda") for _ in range(n)]
    rs = [torch.empty(count // n, device="cuda") for _ in range(n)]
    with flx.Clique(n, loopback=loopback) as c:
        for op in (CollectiveOp.ALLREDUCE, CollectiveOp.ALLGATHER, CollectiveOp.REDUCESCATTER):
            c.set_shares(op, (900, 100, 0))
        assert L.flxGroupStart() == 0
        for i, comm_i in enumerate(c.comms):
            comm_i.all_reduce(xs[i], red[i])
            comm_i.all_gather(red[i], gat[i])
            comm_i.reduce_scatter(xs[i], rs[i])
        assert L.flxGroupEnd() == 0
        torch.cuda.synchronize()
        total = torch.stack(xs).sum(0)
        for i in range(n):
            assert torch.equal(red[i], total), i
            assert torch.equal(gat[i], total.repeat(n)), i
            assert torch.equal(rs[i], total[i * (count // n):(i + 1) * (count // n)]), i
        assert L.flxGroupStart() == 0
        for i, comm_i in enumerate(c.comms):
            if i == 1:
                comm_i.all_gather(red[i], gat[i])
            else:
                comm_i.all_reduce(xs[i], red[i])
        assert L.flxGroupEnd() == 5  # flxInvalidUsage (== ncclInvalidUsage): nothing launched
