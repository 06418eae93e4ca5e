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
