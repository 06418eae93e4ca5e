"""flxCommSplit / ncclCommSplit across two real processes (csrc/flexlink.cu).

Ranks exchange (color, key) through the parent's agreement board, each color
bootstraps a child communicator under an id derived from the parent's, ordered
by key.  Both processes share the one GPU, so every byte runs on the host-staged
PCIe path (FLX_SHARES=0,1000 at every communicator's creation; sizes a multiple
of the alignment) — no kernel waits on the other process."""

import os
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(r, n):
    return ((torch.arange(n, dtype=torch.float32) * (r + 2)) % 97 - 40).cuda()


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), FLX_ALLOW_SHARED_GPU="1",
                      FLX_SLOT_MB="1", FLX_PCIE_STAGE_MB="8", FLX_BOOT_TIMEOUT="60",
                      FLX_SHARES="0,1000")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_15882_b200 import comm

        count = 1 << 18
        res = {}
        c = comm.Communicator.from_process_group()
        x = _data(rank, count)
        # one color, keys reversing the order
        a = c.split(0, key=-rank)
        res["a"] = (a.nranks, a.rank)
        s = torch.empty_like(x)
        a.all_reduce(x, s)
        g = torch.empty(2 * count, device="cuda")
        a.all_gather(x, g)
        torch.cuda.synchronize()
        want_g = torch.cat([_data(1 - j, count) for j in range(2)])  # new rank j = parent 1-j
        res["a_ok"] = bool(torch.equal(s, _data(0, count) + _data(1, count)) and
                           torch.equal(g, want_g))
        # one color per rank: two single-rank communicators
        b = c.split(rank, 0)
        res["b"] = (b.nranks, b.rank)
        sb = torch.empty_like(x)
        b.all_reduce(x, sb)
        torch.cuda.synchronize()
        res["b_ok"] = bool(torch.equal(sb, x))
        # rank 1 joins none
        d = c.split(7 if rank == 0 else -1, 0)
        res["d"] = None if d is None else (d.nranks, d.rank)
        # the parent keeps working after three splits
        sp = torch.empty_like(x)
        c.all_reduce(x, sp)
        torch.cuda.synchronize()
        res["parent_ok"] = bool(torch.equal(sp, _data(0, count) + _data(1, count)))
        res["pcie"] = a.path_bytes()[1]
        dist.barrier()
        for child in (a, b, d):
            if child is not None:
                child.destroy()
        c.destroy()
        out[rank] = res
    finally:
        dist.destroy_process_group()


def test_split_across_two_processes():
    from paper_2510_15882_b200.build import build

    build()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, _port(), out), nprocs=2, join=True)
        res = dict(out)
    for rank in range(2):
        r = res[rank]
        assert r["a"] == (2, 1 - rank), r
        assert r["a_ok"] and r["b_ok"] and r["parent_ok"], r
        assert r["b"] == (1, 0), r
        assert r["d"] == ((1, 0) if rank == 0 else None), r
        assert r["pcie"] > 0, r
