"""PCIe-leg watchdog behind flxCommGetAsyncError / ncclCommGetAsyncError
(csrc/world.cu ``world_aborted``).

Copy-engine waits on a dead peer's token words never time out by themselves,
so the watchdog reports a PCIe leg that stays unfinished FLX_TIMEOUT_S after it
was seen RUNNING.  The h2d stream writes "leg started" / "leg finished" counters
into pinned memory, so a leg still queued behind the caller's own long kernels
is not a stall (the old rule timed from the host-side issue and aborted a
healthy communicator whose stream was merely busy)."""

import os
import socket
import time

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.multiprocessing as mp  # noqa: E402

from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402


def _sleep_cycles(seconds: float) -> int:
    khz = torch.cuda.get_device_properties(0).clock_rate  # kHz (max SM clock)
    return int(seconds * khz * 1e3)


def test_pcie_leg_queued_behind_user_work_is_not_a_stall(monkeypatch):
    monkeypatch.setenv("FLX_TIMEOUT_S", "1")  # read when the world is created
    n, count = 4, 1 << 20
    g = torch.Generator(device="cuda").manual_seed(3)
    sends = [torch.randint(-99, 99, (count,), device="cuda", generator=g).float()
             for _ in range(n)]
    recvs = [torch.empty_like(s) for s in sends]
    exact = torch.stack(sends).sum(0)
    with flx.Clique(n, loopback=True) as w:
        w.set_shares(CollectiveOp.ALLREDUCE, (900, 100, 0))  # pinned: no tuning reads
        w.all_reduce(sends, recvs)
        torch.cuda.synchronize()
        assert w.path_bytes()[1] > 0
        assert w.comms[0].async_error() == 0
        # 3 s of the caller's own work ahead of the next striped call, polled
        # the way a framework's watchdog thread polls ncclCommGetAsyncError
        torch.cuda._sleep(_sleep_cycles(3.0))
        for r in recvs:
            r.zero_()
        w.all_reduce(sends, recvs)
        seen, t0 = set(), time.monotonic()
        while time.monotonic() - t0 < 2.5:
            seen.add(w.comms[0].async_error())
            time.sleep(0.05)
        torch.cuda.synchronize()
        assert seen == {0}, seen
        assert w.comms[0].async_error() == 0
        assert all(torch.equal(r, exact) for r in recvs)
        w.all_reduce(sends, recvs)  # the communicator is still usable
        torch.cuda.synchronize()
        assert all(torch.equal(r, exact) for r in recvs)


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stall_worker(rank, world, port, q):
    import faulthandler
    import sys

    import torch.distributed as dist

    faulthandler.dump_traceback_later(90, exit=True, file=sys.stderr)  # a hang prints where
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), FLX_ALLOW_SHARED_GPU="1",
                      FLX_SLOT_MB="1", FLX_PCIE_STAGE_MB="8", FLX_BOOT_TIMEOUT="60",
                      FLX_TIMEOUT_S="1")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_15882_b200 import comm

        c = comm.Communicator.from_process_group()
        c.set_shares(CollectiveOp.ALLREDUCE, (0, 1000, 0))  # PCIe only: no waiting kernel
        if rank == 0:
            # rank 1 never calls: this rank's PCIe leg parks on its token words
            t = torch.ones(1 << 18, device="cuda")
            c.all_reduce(t)
            t0, err = time.monotonic(), 0
            while time.monotonic() - t0 < 30 and err == 0:
                err = c.async_error()
                time.sleep(0.05)
            q.put((err, time.monotonic() - t0))
        dist.barrier()
        if rank == 0:
            c.abort()  # releases the parked waits; no destroy barrier
        else:
            c.destroy()
    finally:
        dist.destroy_process_group()


def test_pcie_leg_waiting_on_a_dead_peer_is_reported_and_aborts():
    from paper_2510_15882_b200.build import build

    build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_stall_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        err, waited = q.get(timeout=120)
        for p in procs:
            p.join(timeout=60)
        assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
    assert err == 3, err  # flxInternalError == ncclInternalError
    assert 0.9 < waited < 10, waited


def _park(stream, word_ptr):
    """Enqueue a wait on `stream` for a pinned host word to become 1."""
    import cuda.bindings.driver as drv

    (r,) = drv.cuStreamWaitValue32(drv.CUstream(stream.cuda_stream), drv.CUdeviceptr(word_ptr), 1,
                                   drv.CUstreamWaitValue_flags.CU_STREAM_WAIT_VALUE_EQ)
    assert r == drv.CUresult.CUDA_SUCCESS, r


@pytest.mark.parametrize("loopback", [False, True])
def test_first_launches_do_not_block_behind_a_parked_stream(loopback):
    """With another stream of the device parked on a host word (as a PCIe leg
    parks on a late peer's token), the first launch of every kernel a
    collective uses — fold / fan-out kernels, the rank kernels with their
    dynamic-shared-memory opt-in — returns to the host at once: communicator
    init preloaded every module, so no lazy load waits behind the parked work."""
    import threading

    n, count = 4, (1 << 16) + 3
    with flx.Clique(n, loopback=loopback) as c:
        for op in CollectiveOp:
            c.set_shares(op, (1000, 0, 0))
        g = torch.Generator(device="cuda").manual_seed(9)
        outs = {}
        for dt in (torch.float64, torch.bfloat16, torch.int32):  # first use of each
            s = [torch.randint(-9, 9, (count,), device="cuda", generator=g).to(dt)
                 for _ in range(n)]
            outs[dt] = (s, [torch.empty_like(x) for x in s],
                        [torch.empty(n * count, device="cuda", dtype=dt) for _ in range(n)])
        torch.cuda.synchronize()  # inputs ready; only FlexLink launches from here on
        word = torch.zeros(1, dtype=torch.int32).pin_memory()
        parked = torch.cuda.Stream()
        _park(parked, word.data_ptr())
        done = threading.Event()

        def issue():
            for s, r, gat in outs.values():
                c.all_reduce(s, r)
                c.all_gather(s, gat)
            done.set()

        t = threading.Thread(target=issue, daemon=True)
        t.start()
        returned = done.wait(timeout=20)
        word.fill_(1)  # release the parked stream (the host word is pinned)
        t.join(timeout=60)
        torch.cuda.synchronize()
        assert returned, "a first launch blocked behind the parked stream"
        for dt, (s, r, gat) in outs.items():
            want = torch.stack([x.double() for x in s]).sum(0).to(dt)
            assert all(torch.equal(x, want) for x in r), dt
            assert all(torch.equal(x, torch.cat(s)) for x in gat), dt
