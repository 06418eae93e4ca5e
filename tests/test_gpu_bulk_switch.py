"""The opt-in copy paths stay exact: register copies in the multi-GPU engine
(FLX_BULK=0) and the bulk-copy virtual-rank kernels (FLX_TMA=1).

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


def test_tma_fold_and_fanout_variants_match_oracle():
    # FLX_TMA=1: the virtual-rank fold / fan-out as cp.async.bulk + mbarrier
    # kernels (kernels.cuh fold_tma_kernel / fanout_tma_kernel; opt-in, slower
    # than the single-pass kernels on B200) — the oracle-checked AllReduce /
    # AllGather cases of test_gpu_parity.py through them
    env = dict(os.environ, FLX_TMA="1")
    out = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
         "tests/test_gpu_parity.py", "-k",
         "matches_oracle or inplace or misaligned or config2 or large_allreduce"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert " passed" in out.stdout
