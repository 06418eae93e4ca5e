"""Worker for tests/test_gpu_c10d.py: one rank of a 'flexlink' torch.distributed
process group, exercising the torch API names against exact expectations."""
import os
import sys

import torch
import torch.distributed as dist
import torch.distributed._functional_collectives as funcol

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_15882_b200 import c10d  # noqa: E402
from paper_2510_15882_b200.striping import CollectiveOp  # noqa: E402


def vals(rank, n, shift=0):
    i = torch.arange(n, dtype=torch.float64)
    return (((i * (rank + 3) + shift) % 251) - 100).float()


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    c10d.register()
    dist.init_process_group("flexlink", rank=rank, world_size=world)
    comm = c10d.backend_of().comm
    assert c10d.backend_of(dist.group.WORLD) is c10d.backend_of()  # the group's own backend
    if os.environ.get("FLX_C10D_PCIE_ONLY"):
        # two processes share this GPU: every byte on the host-staged PCIe path
        # (copy engines only), so no NVLink-path kernel waits on the other process
        for op in CollectiveOp:
            comm.set_shares(op, (0, 1000, 0))
    n = 1 << 18  # a multiple of every alignment: no NVLink remainder
    dev = torch.device("cuda", 0)
    bad = 0
    for it in range(2):
        x = vals(rank, n, it).to(dev)
        want = sum(vals(r, n, it) for r in range(world)).to(dev)
        dist.all_reduce(x)
        bad += int(not torch.equal(x, want))
        mx = vals(rank, n, it).to(dev)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        bad += int(not torch.equal(mx, torch.stack([vals(r, n, it) for r in range(world)]).max(0)
                                   .values.to(dev)))
        av = vals(rank, n, it).to(dev)
        dist.all_reduce(av, op=dist.ReduceOp.AVG)  # integer-valued: exact sum, then / world
        bad += int(not torch.equal(av, (sum(vals(r, n, it) for r in range(world)) / world)
                                   .to(dev)))
        src = vals(rank, n, it).to(dev)
        out = torch.empty(world * n, device=dev)
        dist.all_gather_into_tensor(out, src)
        bad += int(not torch.equal(out, torch.cat([vals(r, n, it) for r in range(world)]).to(dev)))
        outs = [torch.empty(n, device=dev) for _ in range(world)]
        dist.all_gather(outs, src)
        bad += int(not all(torch.equal(o, vals(r, n, it).to(dev)) for r, o in enumerate(outs)))
        big = vals(rank, world * n, it).to(dev)
        rs = torch.empty(n, device=dev)
        dist.reduce_scatter_tensor(rs, big)
        full = sum(vals(r, world * n, it) for r in range(world))
        bad += int(not torch.equal(rs, full[rank * n:(rank + 1) * n].to(dev)))
        rsa = torch.empty(n, device=dev)
        dist.reduce_scatter_tensor(rsa, big, op=dist.ReduceOp.AVG)
        bad += int(not torch.equal(rsa, (full[rank * n:(rank + 1) * n] / world).to(dev)))
        a2a = torch.empty(world * n, device=dev)
        dist.all_to_all_single(a2a, big)
        want_a2a = torch.cat([vals(r, world * n, it)[rank * n:(rank + 1) * n]
                              for r in range(world)]).to(dev)
        bad += int(not torch.equal(a2a, want_a2a))
    # functional collectives (DTensor's path) resolve the group by name
    x = vals(rank, n).to(dev)
    y = funcol.wait_tensor(funcol.all_reduce(x, "sum", dist.group.WORLD))
    bad += int(not torch.equal(y, sum(vals(r, n) for r in range(world)).to(dev)))
    g = funcol.wait_tensor(funcol.all_gather_tensor(x, 0, dist.group.WORLD))
    bad += int(not torch.equal(g, torch.cat([vals(r, n) for r in range(world)]).to(dev)))
    big = vals(rank, world * n).to(dev)
    rs = funcol.wait_tensor(funcol.reduce_scatter_tensor(big, "sum", 0, dist.group.WORLD))
    full = sum(vals(r, world * n) for r in range(world))
    bad += int(not torch.equal(rs, full[rank * n:(rank + 1) * n].to(dev)))
    a2a = funcol.wait_tensor(funcol.all_to_all_single(big, None, None, dist.group.WORLD))
    bad += int(not torch.equal(a2a, torch.cat([vals(r, world * n)[rank * n:(rank + 1) * n]
                                               for r in range(world)]).to(dev)))
    pair = funcol.all_reduce_coalesced([vals(rank, n).to(dev), vals(rank, n, 7).to(dev)], "max",
                                       dist.group.WORLD)
    for shift, t in zip((0, 7), pair):
        want = torch.stack([vals(r, n, shift) for r in range(world)]).max(0).values.to(dev)
        bad += int(not torch.equal(funcol.wait_tensor(t), want))
    if bad:
        print(f"rank {rank} functional collectives mismatch", flush=True)
    # broadcast (flxBroadcast on the bytes): exact, any dtype.  Two processes on
    # one GPU (PCIE_ONLY) keep every collective a multiple of the alignment, so no
    # NVLink-path kernel spins on the other process (the library refuses one);
    # ragged lengths are covered at world 1 here and by tests/test_c10d_compose_cpu.py
    root = world - 1
    shared = bool(os.environ.get("FLX_C10D_PCIE_ONLY"))
    cases = (((torch.float32, 4096), (torch.bfloat16, 8192), (torch.int64, 2048)) if shared else
             ((torch.float32, n + 5), (torch.bfloat16, 1001), (torch.int64, 3)))
    for dt, cnt in cases:
        src = (vals(root, cnt) * 1.5).to(dt)
        if dt.is_floating_point:
            src[0] = -0.0  # a sum with zeros would lose the sign: copies keep it
        t = (src if rank == root else torch.full_like(src, 7)).to(dev)
        dist.broadcast(t, root)
        bad += int(not torch.equal(t.cpu().view(-1).view(torch.uint8),
                                   src.view(-1).view(torch.uint8)))
    # DDP: construction broadcasts rank 0's module state, backward averages gradients
    # (its shape checks and small buckets are ragged: world 1 only on one GPU)
    if not shared:
        bad += ddp_check(rank, world, dev)
    if bad:
        print(f"rank {rank} broadcast / DDP mismatch", flush=True)
    dist.barrier()
    # reduce to rank 0 (flxReduce): the sum there, the other ranks untouched
    rx = vals(rank, n).to(dev)
    dist.reduce(rx, 0)
    bad += int(not torch.equal(rx, sum(vals(r, n) for r in range(world)).to(dev) if rank == 0
                               else vals(rank, n).to(dev)))
    # gather / scatter to and from the last rank (flxGather / flxScatter)
    last = world - 1
    gl = [torch.empty(n, device=dev) for _ in range(world)] if rank == last else None
    dist.gather(vals(rank, n).to(dev), gl, dst=last)
    if rank == last:
        bad += int(not all(torch.equal(g, vals(r, n).to(dev)) for r, g in enumerate(gl)))
    sc = torch.empty(n, device=dev)
    dist.scatter(sc, [vals(r, n, 5).to(dev) for r in range(world)] if rank == last else None,
                 src=last)
    bad += int(not torch.equal(sc, vals(rank, n, 5).to(dev)))
    try:  # a collective FlexLink does not implement is refused, never a fallback
        dist.all_to_all_single(torch.empty(n, device=dev), x,
                               output_split_sizes=[n - world + 1] + [1] * (world - 1),
                               input_split_sizes=[n - world + 1] + [1] * (world - 1))
        if world > 1:
            bad += 1
    except Exception as e:
        if "FlexLink" not in str(e):
            bad += 1
    torch.cuda.synchronize()
    print(f"rank {rank} bad {bad}", flush=True)
    c10d.backend_of().shutdown()
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)


def ddp_check(rank, world, dev):
    bad = 0
    torch.manual_seed(100 + rank)
    model = torch.nn.Linear(64, 32).to(dev)
    ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[0])
    p0 = [p.detach().clone() for p in ddp.parameters()]
    gathered = [torch.empty_like(p0[0]) for _ in range(world)]
    dist.all_gather(gathered, p0[0])
    bad += int(not all(torch.equal(g, gathered[0]) for g in gathered))
    torch.manual_seed(7 + rank)
    ddp(torch.randn(16, 64, device=dev)).square().sum().backward()
    grads = [torch.empty_like(model.weight.grad) for _ in range(world)]
    dist.all_gather(grads, model.weight.grad)
    bad += int(not all(torch.equal(g, grads[0]) for g in grads))
    return bad


if __name__ == "__main__":
    main()
