"""Host logic of the 'flexlink' c10d backend at world size 2, on CPU (gloo).

FlexLinkBackend's composed operations — broadcast on the bytes of any dtype
(flxBroadcast's zeros-then-MAX-over-uint8 rule), ReduceOp.AVG passed to the
library as FLX_OP_AVG (floats and integers) — run here with a stand-in communicator whose broadcast / all_reduce /
reduce_scatter are gloo's, so byte views, the root's placement and ragged
lengths are checked across two real processes without a GPU.  The GPU
test (tests/test_gpu_c10d.py) runs the same methods over the real kernels.
"""
import os
import socket
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _worker(rank: int, world: int, port: int, q) -> None:
    import torch
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT))
    from paper_2510_15882_b200 import c10d

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    class GlooComm:  # FlexLink Communicator's tensor API, served by gloo
        def broadcast(self, send, recv=None, root=0, stream=None):
            # flxBroadcast's rule: the root's bytes, zeros elsewhere, MAX over uint8
            recv = send if recv is None else recv
            if rank == root:
                recv.copy_(send)
            else:
                recv.zero_()
            dist.all_reduce(recv, op=dist.ReduceOp.MAX)

        def all_to_all(self, send, recv, stream=None):
            dist.all_to_all_single(recv, send)

        def all_gather(self, send, recv, stream=None):
            dist.all_gather_into_tensor(recv, send)

        @staticmethod
        def _avg(t):  # FLX_OP_AVG's finish: IEEE division for floats, C division for ints
            if t.is_floating_point():
                t.copy_(t / torch.full_like(t, world))
            else:
                t.copy_(torch.div(t, world, rounding_mode="trunc"))

        def all_reduce(self, send, recv, op="sum", stream=None):
            assert op in ("sum", "avg"), op
            recv.copy_(send)
            dist.all_reduce(recv)
            if op == "avg":
                self._avg(recv)

        def reduce_scatter(self, send, recv, op="sum", stream=None):
            assert op in ("sum", "avg"), op
            full = send.clone()
            dist.all_reduce(full)
            n = recv.numel()
            recv.copy_(full[rank * n:(rank + 1) * n])
            if op == "avg":
                self._avg(recv)

    class Host(c10d.FlexLinkBackend):
        def __init__(self):
            dist.ProcessGroup.__init__(self, rank, world)
            self.comm = GlooComm()

        @property
        def _stream(self):
            return None

    be = Host()
    bad = []
    # broadcast: every dtype's bytes, ragged lengths (not multiples of N or 16 B)
    for root in range(world):
        for dt, cnt in ((torch.float32, 1), (torch.float32, 37), (torch.bfloat16, 1001),
                        (torch.int64, 5), (torch.uint8, 16 * world + 3)):
            src = (torch.arange(cnt, dtype=torch.float64) * (root + 1.5) - 7).to(dt)
            if dt.is_floating_point:
                src[0] = -0.0
            t = src.clone() if rank == root else torch.full_like(src, 3)
            opts = dist.BroadcastOptions()
            opts.rootRank = root
            be.broadcast([t], opts).wait()
            if not torch.equal(t.view(-1).view(torch.uint8), src.view(-1).view(torch.uint8)):
                bad.append(f"broadcast root {root} {dt} {cnt}")
    # AVG: floating sum then / world; integer tensors refused
    x = torch.arange(10, dtype=torch.float32) + rank * 3
    o = dist.AllreduceOptions()
    o.reduceOp = dist.ReduceOp.AVG
    be.allreduce([x], o)
    want = (sum(torch.arange(10, dtype=torch.float32) + r * 3 for r in range(world))) / world
    if not torch.equal(x, want):
        bad.append("allreduce avg")
    big = torch.arange(4 * world, dtype=torch.float32) * (rank + 1)
    out = torch.empty(4)
    ro = dist.ReduceScatterOptions()
    ro.reduceOp = dist.ReduceOp.AVG
    be._reduce_scatter_base(out, big, ro)
    full = sum(torch.arange(4 * world, dtype=torch.float32) * (r + 1) for r in range(world))
    if not torch.equal(out, full[rank * 4:(rank + 1) * 4] / world):
        bad.append("reduce_scatter avg")
    xi = torch.tensor([7, -7, 3], dtype=torch.int32) * (rank + 1)
    be.allreduce([xi], o)  # integers: C division of the sum (truncation), as NCCL
    si = sum(torch.tensor([7, -7, 3], dtype=torch.int64) * (r + 1) for r in range(world))
    if not torch.equal(xi, torch.div(si, world, rounding_mode="trunc").to(torch.int32)):
        bad.append("integer avg")
    dist.destroy_process_group()
    q.put((rank, bad))


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_broadcast_and_avg_composition_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: [], 1: []}, results
    assert all(p.exitcode == 0 for p in procs)


if __name__ == "__main__":
    pytest.main([__file__, "-q"])
