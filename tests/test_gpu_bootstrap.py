"""Multi-process bootstrap on one GPU: flxCommInitRank across 2 real processes.

Exercises what the loopback world cannot: the shm rendezvous named by the
unique id, the exchange and opening of CUDA-IPC handles, and the shared,
cudaHostRegister'ed staging segment.  Both processes sit on the same GPU
(FLX_ALLOW_SHARED_GPU), so NO collective runs (the per-GPU rank kernels of two
processes would wait on each other); data crosses only through plain copies
(flxCommDebugPeer) with gloo barriers in between.
"""

import ctypes
import os
import socket
import time

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), FLX_ALLOW_SHARED_GPU="1",
                      FLX_SLOT_MB="1", FLX_PCIE_STAGE_MB="1", FLX_BOOT_TIMEOUT="60")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_15882_b200 import comm

        c = comm.Communicator.from_process_group()
        L = comm.load_library()
        n = 4096
        mine = (ctypes.c_ubyte * n)(*([(rank * 37 + i) % 251 for i in range(n)]))
        for region in (0, 1):
            assert L.flxCommDebugPeer(c.handle, rank, region, 1, mine, n) == 0
        torch.cuda.synchronize()
        dist.barrier()
        got = {}
        for region in (0, 1):
            for peer in range(world):
                buf = (ctypes.c_ubyte * n)()
                assert L.flxCommDebugPeer(c.handle, peer, region, 0, buf, n) == 0
                got[(region, peer)] = bytes(buf)
        dist.barrier()
        out[rank] = {"nranks": c.nranks, "rank": c.rank, "got": got}
        c.destroy()
    finally:
        dist.destroy_process_group()


def test_two_process_bootstrap_ipc_and_shared_staging():
    from paper_2510_15882_b200.build import build

    build()
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _port(), out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        assert res[rank]["nranks"] == world and res[rank]["rank"] == rank
        for region in (0, 1):
            for peer in range(world):
                want = bytes((peer * 37 + i) % 251 for i in range(4096))
                assert res[rank]["got"][(region, peer)] == want, (rank, region, peer)


def _abort_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), FLX_ALLOW_SHARED_GPU="1",
                      FLX_SLOT_MB="1", FLX_PCIE_STAGE_MB="1", FLX_BOOT_TIMEOUT="60",
                      FLX_TIMEOUT_S="1", FLX_SHARED_GPU_KERNELS="1")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_15882_b200 import comm

        c = comm.Communicator.from_process_group()
        if rank == 0:
            # rank 1 never joins: rank 0's kernel (the only one spinning on this
            # GPU) gives up after FLX_TIMEOUT_S and the communicator is aborted
            t = torch.ones(1024, device="cuda")
            t0 = time.perf_counter()
            c.all_reduce(t)
            torch.cuda.synchronize()
            waited = time.perf_counter() - t0
            async_err = c.async_error()  # ncclCommGetAsyncError
            try:
                c.all_reduce(t)
                out[0] = ("no error", waited, async_err)
            except comm.FlexLinkError as e:
                out[0] = (e.code, waited, async_err)
        dist.barrier()
        if rank == 0:
            c.abort()  # ncclCommAbort: the rank that saw the error does not wait for peers
        else:
            c.destroy()
    finally:
        dist.destroy_process_group()


def test_peer_timeout_aborts_instead_of_hanging():
    # SURVEY 8(b) error conventions: a peer that never arrives ends in
    # flxInternalError (== ncclInternalError, 3) after FLX_TIMEOUT_S, not a hang.
    from paper_2510_15882_b200.build import build

    build()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_abort_worker, args=(2, _port(), out), nprocs=2, join=True)
        code, waited, async_err = out[0]
    assert code == 3 and async_err == 3, (code, async_err)
    assert 0.5 < waited < 30, waited


def _pcie_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), FLX_ALLOW_SHARED_GPU="1",
                      FLX_SLOT_MB="1", FLX_PCIE_STAGE_MB="8", FLX_BOOT_TIMEOUT="60")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_15882_b200 import comm
        from paper_2510_15882_b200.striping import CollectiveOp

        c = comm.Communicator.from_process_group()
        for op in CollectiveOp:  # PCIe only: no NVLink-path kernel, so nothing on
            c.set_shares(op, (0, 1000, 0))  # this shared GPU spins on a peer
        count = 1 << 18  # a multiple of the alignment: the whole message is on PCIe

        def data(r, n_elems):
            return (torch.arange(n_elems, dtype=torch.float32) * (r + 1)) % 251 - 100

        res = {}
        for it in range(3):  # repeated calls reuse the host regions (token handshake)
            x = data(rank + it, count).cuda()
            ar = torch.empty_like(x)
            c.all_reduce(x, ar)
            ag = torch.empty(world * count, device="cuda")
            c.all_gather(x, ag)
            big = data(rank + it, world * count).cuda()
            rs = torch.empty(count, device="cuda")
            c.reduce_scatter(big, rs)
            a2a = torch.empty_like(big)
            c.all_to_all(big, a2a)
            torch.cuda.synchronize()
            xs = [data(r + it, count) for r in range(world)]
            bigs = [data(r + it, world * count) for r in range(world)]
            ok = torch.equal(ar.cpu(), sum(xs)) and torch.equal(ag.cpu(), torch.cat(xs))
            ok = ok and torch.equal(rs.cpu(), sum(b[rank * count:(rank + 1) * count] for b in bigs))
            ok = ok and torch.equal(a2a.cpu(), torch.cat(
                [bigs[p][rank * count:(rank + 1) * count] for p in range(world)]))
            res[it] = bool(ok)
        res["pcie_bytes"] = c.path_bytes()[1]
        out[rank] = res
        dist.barrier()
        c.destroy()
    finally:
        dist.destroy_process_group()


def test_two_process_pcie_only_collectives():
    # The host-hub PCIe path across two real processes (shared cudaHostRegister'ed
    # segment, token words written and awaited by different processes).  Only
    # copy engines, stream memory ops and non-waiting fold kernels run, so the
    # two processes may share this GPU.
    from paper_2510_15882_b200.build import build

    build()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_pcie_worker, args=(2, _port(), out), nprocs=2, join=True)
        res = dict(out)
    for rank in range(2):
        assert all(res[rank][it] for it in range(3)), res[rank]
        assert res[rank]["pcie_bytes"] > 0
