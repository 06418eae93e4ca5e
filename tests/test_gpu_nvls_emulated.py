"""The NVLS AllReduce / AllGather kernels executed with every multimem
operation emulated over unicast buffers, all ranks on this GPU in one
cooperative grid (tools/nvls_emulate.cu, FLX_NVLS_EMULATE).  The pool's GPUs
are in no multicast fabric (tests/test_gpu_nvls.py skips the switch path with
the driver's reason); this checks everything around the multimem instructions —
per-CTA partition (it caught a floor-then-round partition that skipped the last
16 B of some lengths, profiles/r2/nvls_emulated_old_partition_failures.jsonl),
per-CTA epochs over repeated calls, both arrive barriers, staging / landing
offsets and the AllGather stride — bit-exact against a rank-order CPU fold."""
import json
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_nvls_kernels_emulated_exact(tmp_path):
    exe = tmp_path / "nvls_emulate"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "-o", str(exe), str(ROOT / "tools" / "nvls_emulate.cu")], check=True,
                   capture_output=True, timeout=600)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    rows = [json.loads(line) for line in out.stdout.splitlines() if line.startswith("{")]
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert len(rows) == 3 * (8 + 6) and all(r.get("exact") for r in rows), rows
