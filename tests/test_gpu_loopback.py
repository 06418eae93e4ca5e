"""GPU parity of the multi-GPU engine, emulated on one device (flxCommInitLoopback).

Same kernels and protocols as one-process-per-GPU: push/reduce/pull over
peer-mapped scratch with release/acquire epoch flags (here the "peers" are
other ranks' buffers on the same GPU, the kernel launched cooperatively over
all ranks), and the host-hub PCIe path with cross-rank counter semaphores.
Results must equal the CPU oracle bit for bit.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.links import PathKind  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402

from test_gpu_parity import TORCH_DT, OPS, _inputs, _np  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    flx.load_library()
    oracle.build()


def _allreduce(n, count, dtype, op, granules, inplace=False, calls=1, seed=0):
    cpu = _inputs(n, count, dtype, seed)
    sends = [t.cuda() for t in cpu]
    recvs = sends if inplace else [torch.empty_like(s) for s in sends]
    with flx.Clique(n, loopback=True) as w:
        w.set_shares(CollectiveOp.ALLREDUCE, granules)
        for _ in range(calls):
            if inplace:
                for s, c in zip(sends, cpu):
                    s.copy_(c)
            w.all_reduce(sends, recvs, op=op)
        torch.cuda.synchronize()
        got = [_np(r, dtype) for r in recvs]
        align = w.comms[0].alignment(CollectiveOp.ALLREDUCE)
        pb = w.path_bytes()
    want = oracle.allreduce([_np(c, dtype) for c in cpu], dtype, OPS[op], granules, align)
    return got, want, pb


@pytest.mark.parametrize("n,count,dtype,op,granules", [
    (2, 4096, 7, "sum", (1000, 0, 0)),
    (4, (1 << 18) + 5, 7, "sum", (1000, 0, 0)),
    (8, 1 << 18, 9, "sum", (1000, 0, 0)),
    (8, (1 << 19) + 3, 7, "sum", (900, 100, 0)),
    (4, 1 << 19, 9, "sum", (800, 200, 0)),
    (3, 300007, 2, "max", (850, 150, 0)),
    (8, 1 << 17, 6, "sum", (700, 300, 0)),
    (5, 99999, 8, "min", (1000, 0, 0)),
    (2, 1 << 18, 0, "sum", (500, 500, 0)),
])
def test_loopback_allreduce_matches_oracle(n, count, dtype, op, granules):
    got, want, pb = _allreduce(n, count, dtype, op, granules, seed=n + dtype)
    for r in range(n):
        np.testing.assert_array_equal(got[r], want[r], err_msg=f"rank {r}")
    if granules[1]:
        assert pb[PathKind.PCIE_STAGED] > 0


def test_loopback_config1_full_size_exact():
    # C1 at full size through the multi-GPU engine: 8 ranks x 256 MiB fp32
    # with the default 64 MiB slots (several two-shot rounds per call) and a
    # PCIe share through the host hub.  Integer-valued inputs: exact sums in
    # any order, so torch's sum is the size-independent check.
    n, count = 8, 64 << 20
    g = torch.Generator(device="cuda").manual_seed(1000)
    sends = [torch.randint(-1024, 1024, (count,), device="cuda", generator=g).float()
             for _ in range(n)]
    recvs = [torch.empty_like(s) for s in sends]
    exact = torch.stack(sends).sum(0)
    with flx.Clique(n, loopback=True) as w:
        w.set_shares(CollectiveOp.ALLREDUCE, (990, 10, 0))
        for _ in range(2):
            w.all_reduce(sends, recvs)
        torch.cuda.synchronize()
        assert w.path_bytes()[PathKind.PCIE_STAGED] > 0
    for r in recvs:
        assert torch.equal(r, exact)


def test_loopback_repeated_calls_and_inplace():
    got, want, _ = _allreduce(8, (1 << 18) + 7, 7, "sum", (900, 100, 0), inplace=True, calls=5)
    for r in range(8):
        np.testing.assert_array_equal(got[r], want[r])
    got, want, _ = _allreduce(4, 1 << 18, 9, "sum", (850, 150, 0), calls=7)
    for r in range(4):
        np.testing.assert_array_equal(got[r], want[r])


def test_loopback_multi_round_scratch():
    os.environ["FLX_SLOT_MB"] = "1"  # 1 MiB inbox slots -> many rounds per call
    try:
        got, want, _ = _allreduce(4, 3 << 20, 7, "sum", (1000, 0, 0), calls=2)
    finally:
        del os.environ["FLX_SLOT_MB"]
    for r in range(4):
        np.testing.assert_array_equal(got[r], want[r])


@pytest.mark.parametrize("n,count,dtype,granules", [
    (2, 4096, 7, (1000, 0, 0)),
    (8, (1 << 17) + 1, 9, (1000, 0, 0)),
    (8, 1 << 18, 9, (900, 100, 0)),
    (3, 100003, 0, (700, 300, 0)),
])
def test_loopback_allgather_matches_oracle(n, count, dtype, granules):
    cpu = _inputs(n, count, dtype, n)
    sends = [t.cuda() for t in cpu]
    recvs = [torch.empty(n * count, dtype=TORCH_DT[dtype], device="cuda") for _ in range(n)]
    with flx.Clique(n, loopback=True) as w:
        w.set_shares(CollectiveOp.ALLGATHER, granules)
        for _ in range(3):
            w.all_gather(sends, recvs)
        torch.cuda.synchronize()
        align = w.comms[0].alignment(CollectiveOp.ALLGATHER)
        got = [_np(r, dtype) for r in recvs]
    want = oracle.allgather([_np(c, dtype) for c in cpu], dtype, granules, align)
    for r in range(n):
        np.testing.assert_array_equal(got[r], want[r])


def test_loopback_and_fused_virtual_ranks_agree_bitwise():
    cpu = _inputs(8, 1 << 18, 9, 77)
    a = [t.cuda() for t in cpu]
    b = [t.cuda() for t in cpu]
    oa = [torch.empty_like(x) for x in a]
    ob = [torch.empty_like(x) for x in b]
    with flx.Clique(8, loopback=True) as w, flx.Clique(8) as v:
        w.set_shares(CollectiveOp.ALLREDUCE, (880, 120, 0))
        v.set_shares(CollectiveOp.ALLREDUCE, (1000, 0, 0))
        w.all_reduce(a, oa)
        v.all_reduce(b, ob)
        torch.cuda.synchronize()
    for x, y in zip(oa, ob):
        assert torch.equal(x, y)


def test_loopback_path_times():
    n = 4
    dev = [torch.randn(1 << 22, device="cuda") for _ in range(n)]
    outs = [torch.empty_like(d) for d in dev]
    with flx.Clique(n, loopback=True) as w:
        w.set_shares(CollectiveOp.ALLREDUCE, (950, 50, 0))
        for _ in range(3):
            w.all_reduce(dev, outs)
        h = w.comms[1].path_times_history(8)
        assert len(h) == 3 and all(x[PathKind.NVLINK] > 0 and x[PathKind.PCIE_STAGED] > 0 for x in h)


def test_loopback_cuda_graph_capture_and_replay():
    # The rank kernels keep their flag epochs on the device, so the multi-rank
    # collectives (all four protocols, several slot rounds per call) can be
    # captured once and replayed on fresh inputs, interleaved with eager calls.
    n, count = 4, (3 << 18) + 4
    os.environ["FLX_SLOT_MB"] = "1"  # several rounds per call
    try:
        w = flx.Clique(n, loopback=True)
    finally:
        del os.environ["FLX_SLOT_MB"]
    g = torch.Generator(device="cpu").manual_seed(5)
    sends = [torch.empty(n * count, device="cuda") for _ in range(n)]
    ar = [torch.empty_like(s) for s in sends]
    ag = [torch.empty(n * count, device="cuda") for _ in range(n)]
    ag_in = [s[:count] for s in sends]
    rs = [torch.empty(count, device="cuda") for _ in range(n)]
    a2a = [torch.empty_like(s) for s in sends]
    with w:
        for op in CollectiveOp:
            w.set_shares(op, (1000, 0, 0))
        stream = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            w.all_reduce(sends, ar)
            w.all_gather(ag_in, ag)
            w.reduce_scatter(sends, rs)
            w.all_to_all(sends, a2a)
        a2a_align = w.comms[0].alignment(CollectiveOp.ALLTOALL)
        g1 = (1000, 0, 0)
        for it in range(4):
            host = [torch.randn(n * count, generator=g).round() for _ in range(n)]
            for s, h in zip(sends, host):
                s.copy_(h)
            if it % 2:
                graph.replay()
            else:  # eager calls advance the same device epochs
                w.all_reduce(sends, ar)
                w.all_gather(ag_in, ag)
                w.reduce_scatter(sends, rs)
                w.all_to_all(sends, a2a)
            torch.cuda.synchronize()
            hn = [h.numpy() for h in host]
            want_ar = oracle.allreduce(hn, 7, 0, g1, n * 4096)
            want_ag = oracle.allgather([x[:count] for x in hn], 7, g1, 4096)
            want_rs = oracle.reducescatter(hn, 7, 0, g1, 4096)
            want_a2a = oracle.alltoall(hn, 7, g1, a2a_align)
            for r in range(n):
                np.testing.assert_array_equal(_np(ar[r], 7), want_ar[r])
                np.testing.assert_array_equal(_np(ag[r], 7), want_ag[r])
                np.testing.assert_array_equal(_np(rs[r], 7), want_rs[r])
                np.testing.assert_array_equal(_np(a2a[r], 7), want_a2a[r])


def test_loopback_capture_with_pcie_share_replays():
    # the PCIe path's token handshake uses constant values, so a striped
    # multi-rank collective (NVLink + PCIe) is captured once and replayed,
    # interleaved with eager calls, for all four protocols
    n, count, g = 4, (1 << 18) + 64, (850, 150, 0)
    gen = torch.Generator(device="cpu").manual_seed(21)
    sends = [torch.empty(n * count, device="cuda") for _ in range(n)]
    ar = [torch.empty_like(s) for s in sends]
    ag = [torch.empty(n * count, device="cuda") for _ in range(n)]
    ag_in = [s[:count] for s in sends]
    rs = [torch.empty(count, device="cuda") for _ in range(n)]
    a2a = [torch.empty_like(s) for s in sends]
    with flx.Clique(n, loopback=True) as w:
        for op in CollectiveOp:
            w.set_shares(op, g)
        stream = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            w.all_reduce(sends, ar)
            w.all_gather(ag_in, ag)
            w.reduce_scatter(sends, rs)
            w.all_to_all(sends, a2a)
        assert w.path_bytes()[PathKind.PCIE_STAGED] > 0
        aligns = {op: w.comms[0].alignment(op) for op in CollectiveOp}
        for it in range(5):
            host = [torch.randn(n * count, generator=gen) for _ in range(n)]
            for s, h in zip(sends, host):
                s.copy_(h)
            if it % 2 == 0:
                graph.replay()
            else:
                w.all_reduce(sends, ar)
                w.all_gather(ag_in, ag)
                w.reduce_scatter(sends, rs)
                w.all_to_all(sends, a2a)
            torch.cuda.synchronize()
            hn = [h.numpy() for h in host]
            want_ar = oracle.allreduce(hn, 7, 0, g, aligns[CollectiveOp.ALLREDUCE])
            want_ag = oracle.allgather([x[:count] for x in hn], 7, g,
                                       aligns[CollectiveOp.ALLGATHER])
            want_rs = oracle.reducescatter(hn, 7, 0, g, aligns[CollectiveOp.REDUCESCATTER])
            want_a2a = oracle.alltoall(hn, 7, g, aligns[CollectiveOp.ALLTOALL])
            for r in range(n):
                np.testing.assert_array_equal(_np(ar[r], 7), want_ar[r], err_msg=f"it {it}")
                np.testing.assert_array_equal(_np(ag[r], 7), want_ag[r])
                np.testing.assert_array_equal(_np(rs[r], 7), want_rs[r])
                np.testing.assert_array_equal(_np(a2a[r], 7), want_a2a[r])


def test_loopback_varying_sizes_multi_round():
    # Back-to-back calls whose sizes (and short last rounds) differ: every CTA
    # keeps one fixed region of each slot, so a fast rank's next round never
    # lands in bytes a slower peer CTA is still reading.
    n = 4
    os.environ["FLX_SLOT_MB"] = "1"
    try:
        w = flx.Clique(n, loopback=True)
    finally:
        del os.environ["FLX_SLOT_MB"]
    g = torch.Generator(device="cpu").manual_seed(9)
    with w:
        for op in CollectiveOp:
            w.set_shares(op, (1000, 0, 0))
        for count in (3 << 18, 5000, (1 << 20) + 12, 1 << 16, 777777, 4):
            host = [torch.randn(n * count, generator=g) for _ in range(n)]
            sends = [h.cuda() for h in host]
            ar = [torch.empty_like(s) for s in sends]
            ag = [torch.empty(n * count, device="cuda") for _ in range(n)]
            rs = [torch.empty(count, device="cuda") for _ in range(n)]
            w.all_reduce(sends, ar)
            w.all_gather([s[:count] for s in sends], ag)
            w.reduce_scatter(sends, rs)
            torch.cuda.synchronize()
            hn = [h.numpy() for h in host]
            want_ar = oracle.allreduce(hn, 7, 0, (1000, 0, 0), n * 4096)
            want_ag = oracle.allgather([x[:count] for x in hn], 7, (1000, 0, 0), 4096)
            want_rs = oracle.reducescatter(hn, 7, 0, (1000, 0, 0), 4096)
            for r in range(n):
                np.testing.assert_array_equal(_np(ar[r], 7), want_ar[r])
                np.testing.assert_array_equal(_np(ag[r], 7), want_ag[r])
                np.testing.assert_array_equal(_np(rs[r], 7), want_rs[r])


@pytest.mark.parametrize("oneshot_kb", ["256", "0"])
def test_loopback_oneshot_and_twoshot_interleaved(oneshot_kb):
    # AllReduce slices up to FLX_ONESHOT_KB run the one-shot protocol (its own
    # double-buffered inbox), larger ones the two-shot; interleaved with
    # AllGather on the main slots, in place and out of place, all exact.
    n = 8
    os.environ["FLX_ONESHOT_KB"] = oneshot_kb
    try:
        w = flx.Clique(n, loopback=True)
    finally:
        del os.environ["FLX_ONESHOT_KB"]
    g = torch.Generator(device="cpu").manual_seed(3)
    with w:
        for op in CollectiveOp:
            w.set_shares(op, (1000, 0, 0))
        for it, (count, dtype, op) in enumerate([
                (1024, 7, "sum"), (1 << 20, 7, "sum"), (5, 9, "sum"), (4096, 6, "max"),
                (65536, 7, "sum"), (65536, 7, "sum"), (3 << 18, 9, "sum"), (100, 2, "min"),
                (16384, 8, "prod"), (1, 7, "sum")]):
            cpu = _inputs(n, count, dtype, 100 + it)
            sends = [c.cuda() for c in cpu]
            inplace = it % 3 == 1
            recvs = sends if inplace else [torch.empty_like(s) for s in sends]
            w.all_reduce(sends, recvs, op=op)
            ag = [torch.empty(n * 64, dtype=TORCH_DT[dtype], device="cuda") for _ in range(n)]
            ag_in = [c[:64].cuda() for c in cpu] if count >= 64 else None
            if ag_in is not None:
                w.all_gather(ag_in, ag)
            torch.cuda.synchronize()
            want = oracle.allreduce([_np(c, dtype) for c in cpu], dtype, OPS[op], (1000, 0, 0),
                                    n * 4096)
            for r in range(n):
                np.testing.assert_array_equal(_np(recvs[r], dtype), want[r], err_msg=f"it {it}")
            if ag_in is not None:
                want_ag = oracle.allgather([_np(c, dtype)[:64] for c in cpu], dtype, (1000, 0, 0),
                                           4096)
                for r in range(n):
                    np.testing.assert_array_equal(_np(ag[r], dtype), want_ag[r])


@pytest.mark.parametrize("loopback", [False, True])
def test_timing_off_keeps_results_and_zeroes_path_times(loopback):
    n, count, g = 4, (1 << 18) + 8, (850, 150, 0)
    cpu = _inputs(n, count, 7, 55)
    sends = [c.cuda() for c in cpu]
    recvs = [torch.empty_like(s) for s in sends]
    with flx.Clique(n, loopback=loopback) as w:
        w.set_shares(CollectiveOp.ALLREDUCE, g)
        w.set_timing(False)
        for _ in range(3):
            w.all_reduce(sends, recvs)
        torch.cuda.synchronize()
        assert all(v == 0 for v in w.comms[0].path_times().values())
        align = w.comms[0].alignment(CollectiveOp.ALLREDUCE)
        want = oracle.allreduce([c.numpy() for c in cpu], 7, 0, g, align)
        for r in range(n):
            np.testing.assert_array_equal(_np(recvs[r], 7), want[r])
        w.set_timing(True)
        w.all_reduce(sends, recvs)
        torch.cuda.synchronize()
        t = w.comms[0].path_times()
        assert t[PathKind.NVLINK] > 0 and t[PathKind.PCIE_STAGED] > 0


@pytest.mark.parametrize("count", [1000, (1 << 18) + 4])  # one-shot and two-shot
def test_loopback_sixteen_ranks(count):
    # the widest world (kMaxRanks): 15 peers per flag wait / signal warp
    n, g = 16, (950, 50, 0)
    cpu = _inputs(n, count, 7, 16)
    sends = [c.cuda() for c in cpu]
    recvs = [torch.empty_like(s) for s in sends]
    ag = [torch.empty(n * count, device="cuda") for _ in range(n)]
    with flx.Clique(n, loopback=True) as w:
        w.set_shares(CollectiveOp.ALLREDUCE, g)
        w.set_shares(CollectiveOp.ALLGATHER, g)
        w.all_reduce(sends, recvs)
        w.all_gather(sends, ag)
        torch.cuda.synchronize()
        want = oracle.allreduce([c.numpy() for c in cpu], 7, 0, g,
                                w.comms[0].alignment(CollectiveOp.ALLREDUCE))
        want_ag = oracle.allgather([c.numpy() for c in cpu], 7, g,
                                   w.comms[0].alignment(CollectiveOp.ALLGATHER))
    for r in range(n):
        np.testing.assert_array_equal(_np(recvs[r], 7), want[r])
        np.testing.assert_array_equal(_np(ag[r], 7), want_ag[r])


@pytest.mark.parametrize("ll", ["1", "0"])
def test_loopback_ll_and_flagged_oneshot_interleaved(ll):
    # Small slices run the LL one-shot (epoch inside every 64-bit word, no
    # fence), mid-size ones the flagged one-shot, large ones the slot
    # protocols; the three share the per-CTA epochs and the one-shot parities.
    # Every collective, ragged sizes (some CTAs get empty parts), buffers at
    # 4-byte offsets (the LL path's unaligned user loads/stores), in place.
    n = 8
    os.environ["FLX_LL"] = ll
    try:
        w = flx.Clique(n, loopback=True)
    finally:
        del os.environ["FLX_LL"]
    with w:
        for op in CollectiveOp:
            w.set_shares(op, (1000, 0, 0))
        al = {op: w.comms[0].alignment(op) for op in CollectiveOp}
        g1 = (1000, 0, 0)
        sizes = [3, 1000, 4097, 25600, 18 * 1024, 200000, 1, 9000, 25601, 7]
        for it, count in enumerate(sizes):
            dtype = (7, 9, 6, 2)[it % 4]
            off = it % 2  # one element in: 4 B (fp32/int32) or 2 B (16-bit) aligned
            cpu = _inputs(n, n * count, dtype, 500 + it)
            base = [torch.zeros(n * count + 1, dtype=TORCH_DT[dtype], device="cuda")
                    for _ in range(n)]
            sends = [b[off:off + n * count] for b in base]
            for s, c in zip(sends, cpu):
                s.copy_(c)
            ar = sends if it % 3 == 2 else [torch.empty_like(s) for s in sends]
            hn = [_np(c, dtype) for c in cpu]
            w.all_reduce(sends, ar)
            torch.cuda.synchronize()
            want = oracle.allreduce(hn, dtype, 0, g1, al[CollectiveOp.ALLREDUCE])
            for r in range(n):
                np.testing.assert_array_equal(_np(ar[r], dtype), want[r], err_msg=f"ar {it}")
            for s, c in zip(sends, cpu):  # restore after an in-place call
                s.copy_(c)
            ag = [torch.empty(n * count, dtype=TORCH_DT[dtype], device="cuda") for _ in range(n)]
            w.all_gather([s[:count] for s in sends], ag)
            rs = [torch.empty(count, dtype=TORCH_DT[dtype], device="cuda") for _ in range(n)]
            w.reduce_scatter(sends, rs)
            a2a = [torch.empty_like(s) for s in sends]
            w.all_to_all(sends, a2a)
            torch.cuda.synchronize()
            want_ag = oracle.allgather([x[:count] for x in hn], dtype, g1,
                                       al[CollectiveOp.ALLGATHER])
            want_rs = oracle.reducescatter(hn, dtype, 0, g1, al[CollectiveOp.REDUCESCATTER])
            want_a2a = oracle.alltoall(hn, dtype, g1, al[CollectiveOp.ALLTOALL])
            for r in range(n):
                np.testing.assert_array_equal(_np(ag[r], dtype), want_ag[r], err_msg=f"ag {it}")
                np.testing.assert_array_equal(_np(rs[r], dtype), want_rs[r], err_msg=f"rs {it}")
                np.testing.assert_array_equal(_np(a2a[r], dtype), want_a2a[r],
                                              err_msg=f"a2a {it}")
