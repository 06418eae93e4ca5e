"""In-library two-stage balancer on the real path (csrc/autotune.cpp).

No flxSetShares anywhere: the communicator itself runs Stage 1 (baseline,
rate probe, Algorithm 1, guard) on the first calls of a size bucket and
Stage 2 afterwards, from CUDA-event times — the paper's drop-in behaviour
(PAPER.md:5,46,172,203).  Results stay exact whatever split the balancer
picks (every path applies the same fixed-order fold)."""

import os
import subprocess
from pathlib import Path

import pytest
import torch

from paper_2510_15882_b200 import comm
from paper_2510_15882_b200.links import PathKind
from paper_2510_15882_b200.striping import CollectiveOp

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
MIB = 1 << 20


def _inputs(n, count, seed=7):
    g = torch.Generator(device="cuda").manual_seed(seed)
    sends = [torch.randint(-1024, 1024, (count,), device="cuda", generator=g).float()
             for _ in range(n)]
    return sends, [torch.empty_like(s) for s in sends], torch.stack(sends).sum(0)


def test_capped_clique_tunes_onto_pcie_without_set_shares():
    n, count = 8, 16 * MIB  # 64 MiB fp32 per rank
    sends, recvs, exact = _inputs(n, count)
    with comm.Clique(n, device=0) as c:
        c.set_nvlink_ctas(2)  # config 4: NVLink path slow enough to need help
        phases = set()
        for _ in range(120):
            c.all_reduce(sends, recvs)
            phases.add(c.tune_info(CollectiveOp.ALLREDUCE, count * 4)["phase"])
        torch.cuda.synchronize()
        info = c.tune_info(CollectiveOp.ALLREDUCE, count * 4)
        assert {"baseline", "probe", "stage1", "stage2"} <= phases, phases
        assert info["phase"] == "stage2" and info["kept_tuned"], info
        assert info["tuned_ms"] < info["nvlink_only_ms"], info
        assert c.path_bytes()[PathKind.PCIE_STAGED] > 0
        trace = c.tune_trace(CollectiveOp.ALLREDUCE, count * 4)
        assert trace and trace[-1]["action"] in ("stable", "early_exit"), trace
        assert info["stage2_calls"] > 0
        for r in recvs:
            assert torch.equal(r, exact)


def test_uncapped_guard_and_exactness():
    n, count = 8, 8 * MIB
    sends, recvs, exact = _inputs(n, count, seed=3)
    with comm.Clique(n, device=0) as c:
        for _ in range(80):
            c.all_reduce(sends, recvs)
        torch.cuda.synchronize()
        info = c.tune_info(CollectiveOp.ALLREDUCE, count * 4)
        assert info["phase"] == "stage2", info
        # the guard keeps a split only if it beat NVLink-only on the same run
        if info["kept_tuned"]:
            assert info["tuned_ms"] < info["nvlink_only_ms"]
        else:
            assert info["shares"] == [1000, 0, 0]
        for r in recvs:
            assert torch.equal(r, exact)


def test_pinned_small_and_disabled_buckets_are_left_alone():
    n = 4
    with comm.Clique(n, device=0) as c:
        big, small = 8 * MIB, 64 * 1024
        sends, recvs, exact = _inputs(n, big)
        c.set_shares(CollectiveOp.ALLREDUCE, (1000, 0, 0), big * 4)  # pinned bucket
        for _ in range(12):
            c.all_reduce(sends, recvs)
        assert c.tune_info(CollectiveOp.ALLREDUCE, big * 4)["phase"] == "idle"
        s2, r2, e2 = _inputs(n, small)
        for _ in range(12):
            c.all_reduce(s2, r2)
        assert c.tune_info(CollectiveOp.ALLREDUCE, small * 4)["phase"] == "idle"  # < min bytes
        torch.cuda.synchronize()
        assert all(torch.equal(r, exact) for r in recvs)
        assert all(torch.equal(r, e2) for r in r2)
    with comm.Clique(n, device=0) as c:
        c.set_autotune(False)
        sends, recvs, exact = _inputs(n, 8 * MIB)
        for _ in range(12):
            c.all_reduce(sends, recvs)
        assert c.tune_info(CollectiveOp.ALLREDUCE, 32 * MIB)["phase"] == "idle"
        assert c.path_bytes()[PathKind.PCIE_STAGED] == 0


def test_allgather_and_world_engine_autotune_exact():
    """AllGather on virtual ranks and AllReduce on the loopback world (the
    flxCommInitRank engine) both tune and stay exact."""
    n = 4
    with comm.Clique(n, device=0) as c:
        c.set_nvlink_ctas(1)
        cnt = 8 * MIB  # bf16: 16 MiB per rank
        g = torch.Generator(device="cuda").manual_seed(5)
        ag_s = [torch.randn(cnt, device="cuda", generator=g).bfloat16() for _ in range(n)]
        ag_r = [torch.empty(n * cnt, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
        for _ in range(90):
            c.all_gather(ag_s, ag_r)
        torch.cuda.synchronize()
        assert c.tune_info(CollectiveOp.ALLGATHER, cnt * 2)["phase"] == "stage2"
        want = torch.cat(ag_s)
        assert all(torch.equal(r, want) for r in ag_r)
    with comm.Clique(n, device=0, loopback=True) as w:
        w.set_nvlink_ctas(1)
        sends, recvs, exact = _inputs(n, 8 * MIB, seed=11)
        for _ in range(90):
            w.all_reduce(sends, recvs)
        torch.cuda.synchronize()
        info = w.tune_info(CollectiveOp.ALLREDUCE, 32 * MIB)
        assert info["phase"] == "stage2", info
        assert all(torch.equal(r, exact) for r in recvs)


def test_share_cache_skips_stage1(tmp_path, monkeypatch):
    cache = tmp_path / "shares.txt"
    script = f"""
import os, torch
os.environ["FLX_SHARE_CACHE"] = {str(cache)!r}
from paper_2510_15882_b200 import comm
from paper_2510_15882_b200.striping import CollectiveOp
n, count = 4, 8 << 20
x = [torch.ones(count, device="cuda") * (i + 1) for i in range(n)]
y = [torch.empty_like(t) for t in x]
with comm.Clique(n, device=0) as c:
    c.set_nvlink_ctas(1)
    for _ in range(80):
        c.all_reduce(x, y)
    torch.cuda.synchronize()
    info = c.tune_info(CollectiveOp.ALLREDUCE, count * 4)
    assert all(torch.equal(t, torch.full_like(t, n * (n + 1) / 2)) for t in y)
    print(info["from_cache"], info["stage1_iterations"], info["shares"])
"""
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    first = subprocess.run(["python", "-c", script], capture_output=True, text=True, env=env,
                           timeout=300)
    assert first.returncode == 0, first.stderr
    assert first.stdout.split()[0] == "False"
    assert cache.exists() and cache.read_text().strip()
    second = subprocess.run(["python", "-c", script], capture_output=True, text=True, env=env,
                            timeout=300)
    assert second.returncode == 0, second.stderr
    assert second.stdout.split()[:2] == ["True", "0"], second.stdout


def test_nccl_only_program_gets_striped(tmp_path):
    from paper_2510_15882_b200.build import build, build_nccl_shim

    build()
    if build_nccl_shim() is None:
        pytest.skip("/usr/include/nccl.h absent: shim not built")
    lib = ROOT / "paper_2510_15882_b200"
    exe = tmp_path / "nccl_autotune"
    subprocess.run(["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I/usr/local/cuda/include",
                    f"-I{ROOT / 'include'}", str(ROOT / "tools" / "nccl_autotune.c"),
                    f"-L{lib}", "-lflexlink_nccl", "-lflexlink", "-L/usr/local/cuda/lib64",
                    "-lcudart", f"-Wl,-rpath,{lib}", "-Wl,-rpath,/usr/local/cuda/lib64",
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), (out.returncode,
                                                                        out.stdout, out.stderr)


def test_tuned_split_is_captured_into_cuda_graphs_and_survives_timing_off():
    """A CUDA graph captured after Stage 1 replays the tuned split (captures take no
    tuning step), and switching per-path timing off keeps the split."""
    n, count = 8, 8 * MIB
    sends, recvs, exact = _inputs(n, count, seed=21)
    with comm.Clique(n, device=0) as c:
        c.set_nvlink_ctas(2)
        for _ in range(120):
            c.all_reduce(sends, recvs)
        torch.cuda.synchronize()
        info = c.tune_info(CollectiveOp.ALLREDUCE, count * 4)
        assert info["phase"] == "stage2" and info["kept_tuned"], info
        calls = info["calls"]
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        for r in recvs:
            r.zero_()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            c.all_reduce(sends, recvs)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert all(torch.equal(r, exact) for r in recvs)
        assert c.path_bytes()[PathKind.PCIE_STAGED] > 0
        assert c.tune_info(CollectiveOp.ALLREDUCE, count * 4)["calls"] == calls  # no step
        c.set_timing(False)
        for _ in range(5):
            c.all_reduce(sends, recvs)
        torch.cuda.synchronize()
        assert c.path_bytes()[PathKind.PCIE_STAGED] > 0  # still the tuned split
        assert all(torch.equal(r, exact) for r in recvs)


def test_interleaved_buckets_tune_independently_past_the_event_ring():
    """Two AllReduce buckets and an AllGather bucket issued round-robin for more than
    the 64-slot timing ring: measured calls are harvested before their events are
    reused, every bucket reaches Stage 2, results stay exact."""
    n = 4
    a_s, a_r, a_x = _inputs(n, 8 * MIB, seed=31)       # bucket 25
    b_s, b_r, b_x = _inputs(n, 16 * MIB + 4096, seed=32)  # bucket 26
    g = torch.Generator(device="cuda").manual_seed(33)
    ag_s = [torch.randn(4 * MIB, device="cuda", generator=g) for _ in range(n)]  # 16 MiB sent
    ag_r = [torch.empty(n * 4 * MIB, device="cuda") for _ in range(n)]
    with comm.Clique(n, device=0) as c:
        c.set_nvlink_ctas(1)
        for _ in range(90):
            c.all_reduce(a_s, a_r)
            c.all_reduce(b_s, b_r)
            c.all_gather(ag_s, ag_r)
        torch.cuda.synchronize()
        for op, nbytes in ((CollectiveOp.ALLREDUCE, 32 * MIB),
                           (CollectiveOp.ALLREDUCE, 64 * MIB + 16384),
                           (CollectiveOp.ALLGATHER, 16 * MIB)):
            assert c.tune_info(op, nbytes)["phase"] == "stage2", (op, nbytes)
        assert all(torch.equal(r, a_x) for r in a_r)
        assert all(torch.equal(r, b_x) for r in b_r)
        want = torch.cat(ag_s)
        assert all(torch.equal(r, want) for r in ag_r)
