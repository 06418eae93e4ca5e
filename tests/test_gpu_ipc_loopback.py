"""The multi-GPU engine's rank kernels on CUDA-IPC-mapped peer memory.

A helper process allocates ranks 1..N-1's scratch and flag blocks and exports
them over CUDA IPC (flxDebugHostRemoteRanks); this process builds a loopback
world whose ranks 1..N-1 live in those mappings (flxCommInitLoopbackIpc) and
runs every collective through the rank kernels — two-shot, slot protocols,
flagged one-shot and LL packets, release/acquire flags all landing in another
process's allocations — bit-exact against the CPU oracle.  Only this process
launches kernels: the helper runs none, so no kernel waits on another
process's kernel on the one GPU (B200_PROFILING.md, Xid 109)."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle
from paper_2510_15882_b200 import comm
from paper_2510_15882_b200.striping import CollectiveOp

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("n", [2, 4])
def test_rank_kernels_on_ipc_mapped_peer_memory(n):
    uid = comm.Communicator.unique_id()
    env = dict(os.environ, PYTHONPATH=str(ROOT), FLX_SLOT_MB="8")
    helper = subprocess.Popen(
        [sys.executable, "-c",
         "import sys; from paper_2510_15882_b200 import comm; "
         f"comm.host_remote_ranks({n}, bytes.fromhex('{uid.hex()}'), 0, 120.0)"],
        env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    os.environ["FLX_SLOT_MB"] = "8"  # both processes must agree on the scratch layout
    try:
        g = torch.Generator().manual_seed(n)
        with comm.Clique(n, device=0, loopback=True, ipc_id=uid) as w:
            for op, shares in ((CollectiveOp.ALLREDUCE, (1000, 0, 0)),
                               (CollectiveOp.ALLREDUCE, (900, 100, 0))):
                w.set_shares(op, shares)
                # 300 KiB+: two-shot (several rounds at 8 MiB slots); 40 KiB: LL one-shot
                for count in ((1 << 21) + 5, 10_000 + 3):
                    host = [torch.randint(-99, 99, (count,), generator=g).float() for _ in range(n)]
                    sends = [h.cuda() for h in host]
                    recvs = [torch.empty_like(s) for s in sends]
                    for _ in range(3):
                        w.all_reduce(sends, recvs)
                    torch.cuda.synchronize()
                    align = w.comms[0].alignment(op)
                    want = oracle.allreduce([h.numpy() for h in host], 7, oracle.SUM, shares, align)
                    for r in range(n):
                        np.testing.assert_array_equal(recvs[r].cpu().numpy(), want[r])
            w.set_shares(CollectiveOp.ALLGATHER, (1000, 0, 0))
            w.set_shares(CollectiveOp.REDUCESCATTER, (1000, 0, 0))
            w.set_shares(CollectiveOp.ALLTOALL, (1000, 0, 0))
            for count in (1 << 20, 1000):
                host = [torch.randint(-99, 99, (count * n,), generator=g).float() for _ in range(n)]
                sends = [h.cuda() for h in host]
                ag = [torch.empty(count * n * n, device="cuda") for _ in range(n)]
                rs = [torch.empty(count, device="cuda") for _ in range(n)]
                a2a = [torch.empty_like(s) for s in sends]
                w.all_gather(sends, ag)
                w.reduce_scatter(sends, rs)
                w.all_to_all(sends, a2a)
                torch.cuda.synchronize()
                full = torch.stack(host).sum(0)
                for r in range(n):
                    assert torch.equal(ag[r].cpu(), torch.cat(host))
                    assert torch.equal(rs[r].cpu(), full[r * count:(r + 1) * count])
                    want = torch.cat([host[q][r * count:(r + 1) * count] for q in range(n)])
                    assert torch.equal(a2a[r].cpu(), want)
    finally:
        del os.environ["FLX_SLOT_MB"]
        out, err = helper.communicate(timeout=120)
    assert helper.returncode == 0, err[-2000:]
