"""Both copy paths of the multi-GPU engine stay exact.

The rank kernels' copy phases run as TMA bulk copies through a shared-memory
ring by default (RankArgs::bulk, rank_kernels.cuh cta_copy_bulk); FLX_BULK=0
selects the 16 B register copies.  The rest of the GPU suite runs the default,
so this re-runs the loopback and IPC-loopback parity tests (oracle-checked, all
four collectives, ragged and misaligned cases) in a child process with
FLX_BULK=0.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_register_copy_path_matches_oracle():
    env = dict(os.environ, FLX_BULK="0")
    out = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
         "tests/test_gpu_loopback.py", "tests/test_gpu_ipc_loopback.py",
         "tests/test_gpu_reducescatter.py"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert " passed" in out.stdout
