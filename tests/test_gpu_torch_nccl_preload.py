"""PyTorch's own, unmodified NCCL process group on FlexLink through
LD_PRELOAD=libflexlink_nccl.so (tools/torch_nccl_preload.py): ProcessGroupNCCL
creates its communicators with ncclCommInitRankConfig and issues ncclAllReduce /
ncclAllGather / ncclReduceScatter, which resolve to FlexLink — exact, with
FlexLink kernels counted.  World 1, and world 2 as two processes on this GPU with
every byte pinned to the host-staged PCIe path (FLX_SHARES=0,1000)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
SHIM = ROOT / "paper_2510_15882_b200" / "libflexlink_nccl.so"


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _launch(world, extra):
    from paper_2510_15882_b200.build import build, build_nccl_shim

    build()
    if build_nccl_shim() is None:
        pytest.skip("/usr/include/nccl.h absent: shim not built")
    port = _port()
    procs = []
    for r in range(world):
        env = dict(os.environ, LD_PRELOAD=str(SHIM), RANK=str(r), WORLD_SIZE=str(world),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), **extra)
        procs.append(subprocess.Popen([sys.executable, str(ROOT / "tools" / "torch_nccl_preload.py")],
                                      cwd=ROOT, env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=300) for p in procs]
    lines = []
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, (o, e[-3000:])
        lines.append(json.loads(o.strip().splitlines()[-1]))
    return lines


def test_torch_nccl_backend_world1_runs_on_flexlink():
    (line,) = _launch(1, {})
    assert all(line["exact"].values()), line
    assert line["flexlink_kernels"] >= 3, line  # AllReduce, AllGather, ReduceScatter


def test_torch_nccl_backend_two_processes_pcie_path():
    lines = _launch(2, {"FLX_ALLOW_SHARED_GPU": "1", "FLX_SHARES": "0,1000", "FLX_SLOT_MB": "1",
                        "FLX_PCIE_STAGE_MB": "8", "FLX_BOOT_TIMEOUT": "120"})
    for line in lines:
        assert all(line["exact"].values()), lines
