"""The 'flexlink' torch.distributed backend registers on any host and refuses
to run without its native library / a GPU (no CPU fallback)."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_backend_registers_and_fails_loudly_without_gpu():
    code = """
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, %r)
from paper_2510_15882_b200 import c10d
c10d.register(); c10d.register()  # idempotent
assert dist.Backend.FLEXLINK == "flexlink"
if torch.cuda.is_available():
    print("gpu box: skip"); sys.exit(0)
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29517")
try:
    dist.init_process_group("flexlink", rank=0, world_size=1)
except Exception as e:
    print("refused:", type(e).__name__); sys.exit(0)
sys.exit(3)
""" % str(ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "refused" in out.stdout or "skip" in out.stdout
