"""torch.distributed backend "flexlink" (paper_2510_15882_b200/c10d.py): the
torch API names (dist.all_reduce, all_gather_into_tensor, all_gather,
reduce_scatter_tensor, all_to_all_single, barrier) run FlexLink's collectives,
exact against the expected integer-valued results.

* world 2, two processes sharing this GPU: every byte on the host-staged PCIe
  path (copy engines + stream memory ops only, so no kernel spins on the other
  process), through the real flxCommInitRank bootstrap over the c10d store;
* world 1: the NVLink-path kernels on the same API."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
WORKER = ROOT / "tests" / "c10d_worker.py"


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, extra_env):
    port = _port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), LOCAL_RANK=str(r), **extra_env)
        procs.append(subprocess.Popen([sys.executable, str(WORKER)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=300) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, (o, e[-3000:])
        assert " bad 0" in o


def test_c10d_backend_two_processes_pcie_path():
    _run(2, {"FLX_ALLOW_SHARED_GPU": "1", "FLX_SLOT_MB": "1", "FLX_PCIE_STAGE_MB": "8",
             "FLX_C10D_PCIE_ONLY": "1", "FLX_BOOT_TIMEOUT": "60"})


def test_c10d_backend_world_one_nvlink_path():
    _run(1, {})
