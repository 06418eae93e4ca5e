"""A plain C program, written against nccl.h, runs FlexLink through the NCCL
names across two real processes (tools/nccl_two_process.c): ncclGetUniqueId,
fork, ncclCommInitRank, ncclAllReduce / ncclAllGather / ncclReduceScatter,
three calls each, exact on both ranks — with the communicators from
ncclCommInitRank, and from ncclCommInitRankConfig (non-blocking flag,
maxCTAs).  PCIe-only shares, so the two processes can share this GPU without
either one's kernels spinning on the other."""

import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("mode", ["init_rank", "config"])
def test_nccl_names_across_two_processes(tmp_path, mode):
    from paper_2510_15882_b200.build import build, build_nccl_shim

    build()
    if build_nccl_shim() is None:
        pytest.skip("/usr/include/nccl.h absent: shim not built")
    lib = ROOT / "paper_2510_15882_b200"
    exe = tmp_path / "nccl_two_process"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I/usr/local/cuda/include",
                    f"-I{ROOT / 'include'}", str(ROOT / "tools" / "nccl_two_process.c"),
                    f"-L{lib}", "-lflexlink_nccl", "-lflexlink", "-L/usr/local/cuda/lib64",
                    "-lcudart", f"-Wl,-rpath,{lib}", "-Wl,-rpath,/usr/local/cuda/lib64",
                    "-o", str(exe)], check=True)
    args = [str(exe)] + (["config"] if mode == "config" else [])
    out = subprocess.run(args, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), (out.returncode,
                                                                        out.stdout, out.stderr)
