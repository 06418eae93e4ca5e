"""GPU tests of the integration surface: torch custom ops, CUDA-graph replay of the
custom op, and the link-profile probe feeding Stage 1."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2510_15882_b200 import comm as flx  # noqa: E402
from paper_2510_15882_b200 import torch_ops  # noqa: E402
from paper_2510_15882_b200.links import PathKind  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    flx.load_library()


def test_clique_custom_op_matches_oracle():
    n, count = 8, (1 << 18) + 3
    g = torch.Generator().manual_seed(4)
    host = [torch.randn(count, generator=g) for _ in range(n)]
    xs = [h.cuda() for h in host]
    with flx.Clique(n) as clique:
        clique.set_shares(CollectiveOp.ALLREDUCE, (900, 100, 0))
        cid = torch_ops.register(clique)
        torch.ops.flexlink.clique_all_reduce_(xs, cid, "sum")
        torch.cuda.synchronize()
        torch_ops.unregister(cid)
        align = clique.comms[0].alignment(CollectiveOp.ALLREDUCE)
    want = oracle.allreduce([h.numpy() for h in host], 7, 0, (900, 100, 0), align)
    for x, w in zip(xs, want):
        np.testing.assert_array_equal(x.cpu().numpy(), w)


def test_single_rank_group_ops():
    # a 1-rank communicator: all_reduce is the identity, all_gather a copy
    c = flx.Communicator.init_rank(1, flx.Communicator.unique_id(), 0)
    grp = torch_ops.FlexLinkGroup(c)
    x = torch.randn(1000, device="cuda")
    y = x.clone()
    grp.all_reduce(y)
    out = torch.ops.flexlink.all_gather(x, grp.handle)
    rs = torch.ops.flexlink.reduce_scatter(x, grp.handle, "sum")
    a2a = torch.ops.flexlink.all_to_all(x, grp.handle)
    rs2 = torch.empty_like(x)
    grp.reduce_scatter_tensor(rs2, x)
    a2a2 = torch.empty_like(x)
    grp.all_to_all_single(a2a2, x)
    torch.cuda.synchronize()
    assert torch.equal(y, x) and torch.equal(out, x)
    for t in (rs, a2a, rs2, a2a2):
        assert torch.equal(t, x)
    grp.close()
    c.destroy()


def test_probe_builds_a_loadable_profile(tmp_path):
    from paper_2510_15882_b200 import load_topology, initialize_shares
    from paper_2510_15882_b200.probe import probe_topology, topology_to_yaml

    topo, raw = probe_topology(nranks=4)
    assert raw["pcie"]["h2d"] > 10e9 and raw["pcie"]["d2h"] > 10e9
    p = tmp_path / "box.yaml"
    p.write_text(topology_to_yaml(topo))
    back = load_topology(str(p))
    assert back.link(PathKind.PCIE_STAGED).bandwidth_uni > 10e9
    assert back.link(PathKind.NVLINK).bandwidth_uni > back.link(PathKind.PCIE_STAGED).bandwidth_uni
    shares = initialize_shares(back)
    assert shares.get(PathKind.NVLINK) > shares.get(PathKind.PCIE_STAGED) > 0
