"""Build libflexlink.so with extra -D flags into another directory (A/B runs of
compile-time schedule switches, e.g. -DFLX_ROUNDS_PER_CALL=1 -DFLX_STAGGER=0).
Point the Python binding at it with FLEXLINK_LIBRARY=<dir>/libflexlink.so.
Usage: python tools/build_variant.py <out_dir> -DNAME=VALUE ..."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_15882_b200 import build as B  # noqa: E402

out = Path(sys.argv[1])
defs = sys.argv[2:]
out.mkdir(parents=True, exist_ok=True)
srcs = [B.CSRC / s for s in B.SOURCES]


def one(src):
    obj = out / (src.stem + ".o")
    subprocess.run([B._nvcc(), *B.ARCH, *B.FLAGS, *defs, "-c", str(src), "-o", str(obj)],
                   check=True)
    return str(obj)


with ThreadPoolExecutor(len(srcs)) as pool:
    objs = list(pool.map(one, srcs))
subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(out / "libflexlink.so"), *objs,
                "-lpthread", "-lrt"], check=True)
print(out / "libflexlink.so")
