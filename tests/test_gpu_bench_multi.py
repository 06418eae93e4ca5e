"""The one-process-per-GPU bench path (run_multi_gpu) under torchrun, smoke-run
at WORLD_SIZE 1 on a 1-GPU box (FLX_BENCH_MULTI=1): every leg executes and the
result checks hold.  The N>1 control logic is covered on CPU (gloo, world 2)."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_run_multi_gpu_path_smoke():
    env = dict(os.environ, FLX_BENCH_MULTI="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--steps", "2", "--warmup", "3"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    # rank 0's stdout is exactly the JSON line (NCCL's banner is routed to stderr)
    assert len(out.stdout.strip().splitlines()) == 1, out.stdout
    line = json.loads(out.stdout)
    assert line["n_gpus"] == 1 and line["result_matches_exact_sum"] is True
    assert line["e2e"]["result_exact"] is True and line["allgather"]["matches_nccl_bitwise"]
    assert line["gpu_launches"] > 0 and "clocks" in line
    for name in ("reducescatter", "alltoall"):
        assert line[name]["matches_nccl_bitwise"] is True, line[name]
