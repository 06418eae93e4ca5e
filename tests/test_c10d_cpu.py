"""The 'flexlink' torch.distributed backend registers on any host and refuses
to run without its native library / a GPU (no CPU fallback)."""
import subprocess
import sys
from pathlib import Path

import pytest

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


def test_functional_collectives_resolve_the_python_group_by_name():
    # host logic only: a subclass whose allreduce doubles on the CPU stands in
    # for the communicator, so group_name / work plumbing run without a GPU
    code = """
import os, sys, torch, torch.distributed as dist
import torch.distributed._functional_collectives as funcol
sys.path.insert(0, %r)
from paper_2510_15882_b200 import c10d
class Stub(c10d.FlexLinkBackend):
    def __init__(self, store, rank, size, timeout):
        dist.ProcessGroup.__init__(self, rank, size)
        self.comm = None
    def allreduce(self, tensors, opts=None):
        c10d._op_name(opts.reduceOp)
        for t in tensors:
            t.mul_(2)
        return c10d._DoneWork(tensors)
dist.Backend.register_backend("flxstub", lambda s, r, n, t: Stub(s, r, n, t), devices=["cpu"])
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29519")
dist.init_process_group("flxstub", rank=0, world_size=1)
assert dist.group.WORLD.group_name == dist.distributed_c10d._world.pg_names[dist.group.WORLD]
y = funcol.wait_tensor(funcol.all_reduce(torch.ones(8), "sum", dist.group.WORLD))
assert torch.equal(y, torch.full((8,), 2.0)), y
try:
    funcol.wait_tensor(funcol.all_reduce(torch.ones(8), "bxor", dist.group.WORLD))
    sys.exit(4)
except Exception as e:
    assert "sum/prod/max/min/avg" in str(e), e
dist.destroy_process_group()
print("ok")
""" % str(ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stdout[-1000:] + out.stderr[-2000:]
    assert "ok" in out.stdout


def test_avg_goes_to_the_library_for_every_dtype():
    """ReduceOp.AVG is passed through as the library's FLX_OP_AVG (== ncclAvg):
    the striped sum and its division happen in libflexlink, for floating and
    integer tensors alike; nothing is left for the Python backend to finish."""
    import torch

    from paper_2510_15882_b200 import c10d
    from paper_2510_15882_b200.comm import _OPS

    assert _OPS["avg"] == 4  # FLX_OP_AVG == ncclAvg
    for dt in (torch.float32, torch.bfloat16, torch.int32):
        assert c10d._flx_op("avg", torch.ones(2, dtype=dt)) == "avg"
    assert c10d._flx_op("max", torch.ones(2, dtype=torch.int32)) == "max"
    t = torch.tensor([3.0, -6.0, 1.0])
    c10d._finish("avg", t, 3)  # a no-op now
    assert torch.equal(t, torch.tensor([3.0, -6.0, 1.0]))
