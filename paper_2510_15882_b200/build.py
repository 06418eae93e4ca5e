"""Build libflexlink.so (sm_100a) in-tree with nvcc.

``python -m paper_2510_15882_b200.build`` or ``build()`` from
``__graft_entry__``.  Objects compile in parallel; the shared library lands
next to this file so it travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
CSRC = HERE / "csrc"
LIB = HERE / "libflexlink.so"
SOURCES = ["flexlink.cu", "launch.cu", "world.cu", "nvls.cu", "tuner.cpp", "autotune.cpp",
           "rank_launch_i8.cu", "rank_launch_i32.cu", "rank_launch_i64.cu", "rank_launch_f16.cu",
           "rank_launch_f32.cu", "rank_launch_f64.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-ffp-contract=off",
         "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}"]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libflexlink")
    return cand


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    nvcc = _nvcc()
    objdir = HERE / "build"
    objdir.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    srcs = [CSRC / s for s in SOURCES if (CSRC / s).exists()]
    objs = [objdir / (s.stem + ".o") for s in srcs]

    def compile_one(pair):
        src, obj = pair
        if not force and not _stale(obj, [src] + headers):
            return None
        cmd = [nvcc, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr[-4000:]}")
        return res.stderr if verbose else None

    with ThreadPoolExecutor(max_workers=len(srcs)) as pool:
        for log in pool.map(compile_one, zip(srcs, objs)):
            if log:
                sys.stderr.write(log)
    if force or _stale(LIB, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lpthread", "-lrt"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    build_nccl_shim(force)
    return LIB


SHIM = HERE / "libflexlink_nccl.so"


def build_nccl_shim(force: bool = False) -> Path | None:
    """NCCL-named entry points over libflexlink (checked against /usr/include/nccl.h)."""
    src = CSRC / "nccl_shim.c"
    hdr = Path("/usr/include/nccl.h")
    if not hdr.exists():
        return None
    if not force and not _stale(SHIM, [src, LIB, ROOT / "include" / "flexlink.h"]):
        return SHIM
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-Wall", "-Werror", "-o", str(SHIM),
           str(src), f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include", f"-L{HERE}",
           "-lflexlink", "-Wl,-rpath,$ORIGIN"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nccl shim build failed:\n{res.stderr[-4000:]}")
    return SHIM


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
