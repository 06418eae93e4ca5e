"""bench.py contract pieces that run without a GPU: the reference arm's JSON
line, the busbw formulas and the ncu-traffic readers used in the roofline."""

import json
import subprocess
import sys
from pathlib import Path

import bench

ROOT = Path(__file__).resolve().parents[1]


def test_busbw_formulas():
    # nccl-tests conventions: AllReduce (S/t)*2(N-1)/N, AllGather (S_out/t)*(N-1)/N
    assert bench.busbw_allreduce(8e9, 1.0, 8) == 8 * 2 * 7 / 8
    assert bench.busbw_allgather(8e9, 1.0, 8) == 8 * 7 / 8


def test_ncu_traffic_reads_the_committed_captures():
    fold = bench.ncu_traffic("profiles/r1/fold_once_ncu_summary.txt")
    fan = bench.ncu_traffic("profiles/r1/fanout_once_ncu_summary.txt")
    assert fold and abs(fold - 2 * 8 * 256 * 2**20) / (2 * 8 * 256 * 2**20) < 0.05
    assert fan and abs(fan - 9 * 256 * 2**20) / (9 * 256 * 2**20) < 0.05
    assert bench.ncu_traffic("profiles/r1/does_not_exist.txt") is None


def test_both_arms_name_the_same_workload():
    one = bench.workload_config(1)
    assert one["bytes_per_rank"] == bench.AR_BYTES and one["sim_ranks"] == 8
    assert bench.workload_config(4)["workload"].endswith("over 4 GPUs")


def test_reference_arm_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "3"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert len(out.stdout.strip().splitlines()) == 1, out.stdout  # exactly one JSON line
    line = json.loads(out.stdout)
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["unit"] == "GB/s" and line["higher_is_better"] is True and line["value"] > 0
    assert line["config"] == bench.workload_config(1)
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_gpus_n_without_n_gpus_fails_loudly():
    # `python bench.py --gpus 2` launches 2 ranks itself; on a box with fewer
    # GPUs it refuses (non-zero exit, a reason on stderr) and never prints a
    # 1-GPU line in place of the N-GPU one
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    import torch

    if torch.cuda.device_count() >= 2:
        import pytest

        pytest.skip("this box has >= 2 GPUs: the N-rank run is the real thing")
    assert out.returncode != 0
    assert "n_gpus" not in out.stdout and out.stdout.strip() == ""
    assert "needs 2 visible GPUs" in out.stderr
