"""PyTorch's own, unmodified NCCL process group running on FlexLink through
LD_PRELOAD=libflexlink_nccl.so: ProcessGroupNCCL creates its communicator with
ncclCommInitRankConfig and issues ncclAllReduce / ncclAllGather /
ncclReduceScatter, ncclReduce, ncclBroadcast, ncclAlltoAll (and ncclCommSplit for dist.new_group), which the shim
resolves to FlexLink.  Prints one JSON line:
the results' exactness and how many FlexLink kernels ran (flxGetLaunchCount).
Run:  LD_PRELOAD=$PWD/paper_2510_15882_b200/libflexlink_nccl.so python tools/torch_nccl_preload.py
(two ranks on one GPU: RANK / WORLD_SIZE, FLX_ALLOW_SHARED_GPU=1, FLX_SHARES=0,1000 — every
byte on the host-staged PCIe path, so no kernel spins on the other process's)."""
import ctypes
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    # one GPU per rank where the box has them (LOCAL_RANK); the one-GPU tests share cuda:0
    dev = int(os.environ.get("LOCAL_RANK", rank)) if torch.cuda.device_count() > 1 else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", dev))
    flx = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "paper_2510_15882_b200", "libflexlink.so"))
    count = ctypes.c_ulonglong()
    flx.flxGetLaunchCount.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    flx.flxGetLaunchCount(ctypes.byref(count))
    before = count.value
    n = 1 << 20  # 4 MiB of fp32: a multiple of every alignment (all bytes on one path)

    def data(r):
        g = torch.Generator(device="cuda").manual_seed(r)
        return torch.randint(-100, 100, (n,), device="cuda", generator=g).float()

    mine = data(rank)
    every = [data(r) for r in range(world)]
    x = mine.clone()
    dist.all_reduce(x)
    ok = {"all_reduce": bool(torch.equal(x, torch.stack(every).sum(0)))}
    out = torch.empty(world * n, device="cuda")
    dist.all_gather_into_tensor(out, mine)
    ok["all_gather"] = bool(torch.equal(out, torch.cat(every)))
    rs = torch.empty(n // world, device="cuda")
    dist.reduce_scatter_tensor(rs, mine)
    blk = n // world
    ok["reduce_scatter"] = bool(torch.equal(rs, torch.stack(every).sum(0)[rank * blk:(rank + 1) * blk]))
    # ReduceOp.AVG (ncclAvg, e.g. FSDP's gradient reduce-scatter): the sum, divided
    avg = mine.clone()
    dist.all_reduce(avg, op=dist.ReduceOp.AVG)
    ok["all_reduce_avg"] = bool(torch.equal(avg, torch.stack(every).sum(0) / world))
    # reduce to the last rank (ncclReduce): the sum there, other ranks untouched
    red = mine.clone()
    dist.reduce(red, dst=world - 1)
    ok["reduce"] = bool(torch.equal(red, torch.stack(every).sum(0) if rank == world - 1 else mine))
    # all_to_all_single, equal splits: PyTorch built against NCCL 2.28 calls
    # ncclAlltoAll, which the shim maps to flxAllToAll
    a2a = torch.empty_like(mine)
    dist.all_to_all_single(a2a, mine)
    blk = n // world
    ok["all_to_all"] = bool(torch.equal(a2a, torch.cat([e[rank * blk:(rank + 1) * blk]
                                                         for e in every])))
    # broadcast (DDP's state sync): bit-exact from every root, -0.0 / NaN kept
    bc_ok = True
    for root in range(world):
        for dt, cnt in ((torch.float32, 1 << 18), (torch.bfloat16, 1 << 19)):  # 1 MiB each
            src = data(root)[:cnt].to(dt)
            if dt == torch.float32:
                src.view(torch.int32)[:2] = torch.tensor([-2147483648, 0x7FC00123], device="cuda",
                                                         dtype=torch.int32)
            t = src.clone() if rank == root else torch.zeros_like(src)
            dist.broadcast(t, src=root)
            bc_ok = bc_ok and bool(torch.equal(t.view(torch.uint8), src.view(torch.uint8)))
    ok["broadcast"] = bc_ok
    # subgroups: with device_id bound, ProcessGroupNCCL makes them with
    # ncclCommSplit on the default communicator (non-members split with
    # NCCL_SPLIT_NOCOLOR) — FlexLink's split, collective over the parent
    from torch.distributed import distributed_c10d as c10d_impl

    default = c10d_impl._get_default_group()
    ok["split_path"] = bool(default.bound_device_id is not None and
                            c10d_impl._get_split_source(default) is not None)
    singles = [dist.new_group([r]) for r in range(world)]
    whole = dist.new_group(list(range(world)))
    y = mine.clone()
    dist.all_reduce(y, group=singles[rank])
    ok["new_group_single"] = bool(torch.equal(y, mine))
    z = mine.clone()
    dist.all_reduce(z, group=whole)
    ok["new_group_whole"] = bool(torch.equal(z, torch.stack(every).sum(0)))
    if world == 1:
        dist.barrier()  # a 1-element AllReduce: on a shared GPU it would be an NVLink kernel
    torch.cuda.synchronize()
    flx.flxGetLaunchCount(ctypes.byref(count))
    print(json.dumps({"rank": rank, "world": world, "exact": ok,
                      "flexlink_kernels": count.value - before,
                      "nccl_version_seen_by_torch": torch.cuda.nccl.version()}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
