"""World-size-2 gloo tests of the multi-rank host logic (no GPU).

What the N>1 path needs from the host side, exercised across real processes:
the flxUniqueId is minted once and every rank receives the same bytes; per-path
timings are agreed (max over ranks) so Stage 1 and Stage 2 take identical
decisions on every rank even when each rank measures different noise; and
the byte split each rank computes from those shares is identical.
"""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

MIB = 1 << 20


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_15882_b200 as fl
        from paper_2510_15882_b200 import comm
        from paper_2510_15882_b200.links import PathKind

        uid = comm.broadcast_unique_id()
        uids = [None] * world
        dist.all_gather_object(uids, uid)

        rep = fl.PathTimingReport.build(fl.CollectiveOp.ALLREDUCE, world, MIB,
                                        {PathKind.NVLINK: 1.0 + rank, PathKind.PCIE_STAGED: 3.0 - rank})
        agreed = comm.agree_report(rep)

        topo = fl.preset("H800")
        spec = fl.CollectiveSpec(fl.CollectiveOp.ALLREDUCE, 8, 256 * MIB)
        noise = fl.NoiseModel(0.08, seed=100 + rank)  # every rank sees different jitter
        rng = noise.stream()

        def local_measure(state):
            return fl.simulate_collective(topo, spec, state.shares, noise=noise, rng=rng,
                                          paths=tuple(sorted(state.active)))

        def agreed_measure(state):
            return comm.agree_report(local_measure(state))

        shares_local, _ = fl.initial_tune(topo, spec, measure=local_measure)
        rng = noise.stream()
        shares_agreed, trace = fl.initial_tune(topo, spec, measure=agreed_measure)

        hook = fl.RuntimeBalancer(shares_agreed)
        for call in range(100):
            eff = topo.with_scaled_bandwidth(PathKind.PCIE_STAGED, 0.6) if call > 30 else topo
            r = fl.simulate_collective(eff, spec, hook.shares, noise=noise, rng=rng,
                                       paths=hook.active)
            hook.observe(comm.agree_report(r))
        split = fl.partition(256 * MIB, hook.shares, 8 * 4096)
        out[rank] = {
            "uids": uids, "agreed": {int(k): v for k, v in agreed.durations.items()},
            "local": shares_local.as_array(), "agreed_shares": shares_agreed.as_array(),
            "trace": [x.action for x in trace.records], "stage2": hook.shares.as_array(),
            "moves": sum(1 for e in hook.evaluations if e.moved),
            "split": [split.get(k, 0) for k in PathKind],
        }
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    from paper_2510_15882_b200.build import build

    build()  # flxGetUniqueId comes from the native library (no GPU needed)
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        return dict(out)


def test_unique_id_is_broadcast(results):
    a, b = results[0]["uids"], results[1]["uids"]
    assert a == b and a[0] == a[1] and len(a[0]) == 128 and a[0][:4] == b"FLX1"


def test_agreed_report_is_max_over_ranks(results):
    assert results[0]["agreed"] == results[1]["agreed"] == {0: 2.0, 1: 3.0}


def test_stage1_and_stage2_decisions_identical_across_ranks(results):
    r0, r1 = results[0], results[1]
    assert r0["agreed_shares"] == r1["agreed_shares"] and r0["trace"] == r1["trace"]
    assert r0["stage2"] == r1["stage2"] and r0["moves"] == r1["moves"] >= 1
    assert r0["split"] == r1["split"] and sum(r0["split"]) == 256 * MIB
