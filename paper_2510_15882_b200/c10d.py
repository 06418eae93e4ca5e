"""``torch.distributed`` backend "flexlink".

After :func:`register`, ``dist.init_process_group("flexlink")`` (or
``backend="cuda:flexlink"``) routes ``dist.all_reduce`` /
``dist.all_gather_into_tensor`` / ``dist.reduce_scatter_tensor`` /
``dist.all_to_all_single`` (and their list forms) to FlexLink's striped
collectives, so tensor-parallel code that calls the torch.distributed API names
picks up the NVLink + PCIe split — and the in-library two-stage balancer —
without code changes (the motivating workload is TP AllReduce in
a Qwen-32B prefill).  The functional collectives
(`torch.distributed._functional_collectives`, which DTensor uses) resolve the
group by name; torch keeps that name in its own registry rather than in a
Python-implemented group, so :attr:`FlexLinkBackend.group_name` reads it from
there and ``funcol.all_reduce`` / ``all_gather_tensor`` /
``reduce_scatter_tensor`` / ``all_to_all_single`` reach the same kernels.

One process per GPU.  The communicator is bootstrapped through the process
group's own store (rank 0 publishes the flxUniqueId).  Collectives are
enqueued on the caller's current CUDA stream (stream-ordered like NCCL's
``async_op=False`` path), so the returned work objects are complete from the
stream's point of view.  Broadcast is FlexLink's bit-exact flxBroadcast (DDP's
construction-time state sync).  Operations FlexLink does
not implement (send/recv, uneven all_to_all splits) raise
``NotImplementedError`` instead of silently falling back to another library.
ReduceOp.AVG is the library's FLX_OP_AVG (the striped sum, then one division by
the group size: fl(fl(sum) / n) for floats, C division for integers).
"""

from __future__ import annotations

import torch
import torch.distributed as dist
from torch.futures import Future

from .comm import Communicator

__all__ = ["BACKEND", "register", "FlexLinkBackend", "backend_of"]

BACKEND = "flexlink"
_instances: list["FlexLinkBackend"] = []


class _DoneWork(dist._Work):
    """Work handle of a stream-ordered collective, enqueued on the caller's
    stream at call time.  ``wait()`` makes the CURRENT stream wait for it (as
    ProcessGroupNCCL's work does), so a caller that switched streams between
    issuing the collective and waiting still orders its use of the result."""

    def __init__(self, result, stream=None):
        super().__init__()
        self._fut = Future()
        self._fut.set_result(result)
        self._event = None
        if stream is not None:
            self._event = torch.cuda.Event()
            self._event.record(stream)

    def wait(self, timeout=None) -> bool:
        if self._event is not None:
            torch.cuda.current_stream().wait_event(self._event)
        return True

    def is_completed(self) -> bool:
        return True

    def get_future(self) -> Future:
        return self._fut


def _op_name(op) -> str:
    table = {dist.ReduceOp.SUM: "sum", dist.ReduceOp.PRODUCT: "prod", dist.ReduceOp.MAX: "max",
             dist.ReduceOp.MIN: "min", dist.ReduceOp.AVG: "avg"}
    for k, v in table.items():
        if op == k:
            return v
    raise NotImplementedError(f"FlexLink reduces with sum/prod/max/min/avg only, not {op}")


def _reduce_op(opts) -> str:
    return _op_name(opts.reduceOp if opts is not None else dist.ReduceOp.SUM)


def _flx_op(op: str, t: torch.Tensor) -> str:
    """The FlexLink reduction that runs for `op` on `t`.  AVG is the library's
    FLX_OP_AVG (== ncclAvg): the striped sum, then one division by the group
    size on the caller's stream — IEEE division for floating types
    (fl(fl(sum) / n)), C division for integers, as NCCL divides integer sums."""
    return op


def _finish(op: str, t: torch.Tensor, size: int) -> None:
    """Nothing left to do after a FlexLink reduction (AVG divides in the library)."""


class FlexLinkBackend(dist.ProcessGroup):
    """A c10d process-group backend over :class:`~paper_2510_15882_b200.comm.Communicator`."""

    def __init__(self, store, rank: int, size: int, timeout):
        super().__init__(rank, size)
        key = "flexlink/unique_id"
        if rank == 0:
            uid = Communicator.unique_id()
            store.set(key, uid)
        else:
            uid = bytes(store.get(key))
        self.comm = Communicator.init_rank(size, uid, rank)
        self._store = store
        self._barriers = 0
        try:  # the process group's timeout (a timedelta) bounds barrier waits
            self._timeout_s = float(timeout.total_seconds())
        except AttributeError:
            self._timeout_s = 1800.0
        _instances.append(self)

    # -- names
    def getBackendName(self) -> str:
        return BACKEND

    @property
    def group_name(self) -> str:
        # init_process_group / new_group record the name in torch's registry
        # (and register the group under it for the functional collectives)
        # but only push it into C++-implemented backends
        name = dist.distributed_c10d._world.pg_names.get(self)
        if name is None:
            raise RuntimeError("ProcessGroup name not set")
        return name

    @property
    def _stream(self):
        return torch.cuda.current_stream()

    # -- collectives
    def allreduce(self, tensors, opts=None):
        op = _reduce_op(opts)
        for t in tensors:
            self.comm.all_reduce(t, t, op=_flx_op(op, t), stream=self._stream)
            _finish(op, t, self.size())
        return _DoneWork(tensors, self._stream)

    def allreduce_coalesced(self, tensors, opts=None):
        return self.allreduce(tensors, opts)

    def _allgather_base(self, output, input, opts=None):
        self.comm.all_gather(input, output, stream=self._stream)
        return _DoneWork([output], self._stream)

    def allgather(self, output_lists, input_list, opts=None):
        for outs, inp in zip(output_lists, input_list):
            flat = torch.empty(inp.numel() * self.size(), dtype=inp.dtype, device=inp.device)
            self.comm.all_gather(inp.contiguous(), flat, stream=self._stream)
            for r, o in enumerate(outs):
                o.copy_(flat[r * inp.numel():(r + 1) * inp.numel()].view_as(o))
        return _DoneWork(output_lists, self._stream)

    def allgather_into_tensor_coalesced(self, outputs, inputs, opts=None):
        for o, i in zip(outputs, inputs):
            self.comm.all_gather(i, o, stream=self._stream)
        return _DoneWork(outputs, self._stream)

    def _reduce_scatter_base(self, output, input, opts=None):
        return self.reduce_scatter_tensor_coalesced([output], [input], opts)

    def reduce_scatter_tensor_coalesced(self, outputs, inputs, opts=None):
        op = _reduce_op(opts)
        for o, i in zip(outputs, inputs):
            self.comm.reduce_scatter(i, o, op=_flx_op(op, i), stream=self._stream)
            _finish(op, o, self.size())
        return _DoneWork(outputs, self._stream)

    def reduce_scatter(self, output_tensors, input_lists, opts=None):
        op = _reduce_op(opts)
        for out, ins in zip(output_tensors, input_lists):
            flat = torch.cat([i.reshape(-1) for i in ins])
            res = torch.empty(out.numel(), dtype=out.dtype, device=out.device)
            self.comm.reduce_scatter(flat, res, op=_flx_op(op, flat), stream=self._stream)
            _finish(op, res, self.size())
            out.copy_(res.view_as(out))
        return _DoneWork(output_tensors, self._stream)

    def alltoall_base(self, output, input, output_split_sizes, input_split_sizes, opts=None):
        n = self.size()
        even = input.numel() // n if input.shape[0] % n == 0 else -1
        for splits in (output_split_sizes, input_split_sizes):
            if splits and len(set(splits)) != 1:
                raise NotImplementedError("FlexLink all_to_all needs equal splits")
        if even < 0:
            raise NotImplementedError("FlexLink all_to_all needs dim 0 divisible by world size")
        self.comm.all_to_all(input.contiguous(), output, stream=self._stream)
        return _DoneWork([output], self._stream)

    def barrier(self, opts=None):
        # every rank's queued work done, then a rendezvous on the group's store
        # (no device collective: a 4-byte AllReduce would be a latency-bound
        # NVLink-path kernel for nothing)
        import time

        torch.cuda.current_stream().synchronize()
        self._barriers += 1
        key = f"flexlink/barrier/{self._barriers}"
        self._store.add(key, 1)
        t0 = time.monotonic()
        while int(self._store.add(key, 0)) < self.size():
            if time.monotonic() - t0 > self._timeout_s:
                raise RuntimeError(f"flexlink barrier {self._barriers}: not every rank arrived "
                                   f"within {self._timeout_s:.0f} s")
            time.sleep(0.001)
        return _DoneWork([])

    def shutdown(self) -> None:
        """Destroy the FlexLink communicator (its destroy barrier waits for the peers)."""
        if self.comm is not None:
            self.comm.destroy()
            self.comm = None

    # -- not implemented by FlexLink: refuse, never fall back
    def _refuse(self, name):
        raise NotImplementedError(f"{name} is not a FlexLink collective (AllReduce, AllGather, "
                                  f"ReduceScatter, AllToAll, Reduce, Broadcast, Gather, Scatter are)")

    def broadcast(self, tensors, opts=None):
        """Bit-exact broadcast (DDP's module-state sync at construction):
        FlexLink's flxBroadcast on the tensor's bytes — one striped MAX-over-uint8
        AllReduce with zeros from the non-roots, so any dtype, -0.0 and NaN
        payloads included; in place, no scratch buffers."""
        root = opts.rootRank if opts is not None else 0
        for t in tensors:
            if not t.is_contiguous():
                raise NotImplementedError("FlexLink broadcast needs a contiguous tensor")
            if self.size() == 1 or t.numel() == 0:
                continue
            self.comm.broadcast(t.view(-1).view(torch.uint8), root=root, stream=self._stream)
        return _DoneWork(tensors, self._stream)

    def reduce(self, tensors, opts=None):
        """``dist.reduce``: FlexLink's flxReduce (a striped AllReduce whose
        non-root result goes to scratch), in place on the root."""
        root = opts.rootRank if opts is not None else 0
        op = _reduce_op(opts)
        for t in tensors:
            self.comm.reduce(t, t, op=_flx_op(op, t), root=root, stream=self._stream)
            if self.rank() == root:
                _finish(op, t, self.size())
        return _DoneWork(tensors, self._stream)

    def send(self, *a, **k):
        self._refuse("send")

    def recv(self, *a, **k):
        self._refuse("recv")

    def gather(self, output_tensors, input_tensors, opts=None):
        """``dist.gather``: flxGather into one flat buffer on the root, then the
        root's output list is filled from it."""
        root = opts.rootRank if opts is not None else 0
        n, me = self.size(), self.rank()
        for i, inp in enumerate(input_tensors):
            inp = inp.contiguous()
            flat = torch.empty(n * inp.numel(), dtype=inp.dtype, device=inp.device) \
                if me == root else None
            self.comm.gather(inp, flat, root=root, stream=self._stream)
            if me == root:
                for r, o in enumerate(output_tensors[i]):
                    o.copy_(flat[r * inp.numel():(r + 1) * inp.numel()].view_as(o))
        return _DoneWork(output_tensors, self._stream)

    def scatter(self, output_tensors, input_tensors, opts=None):
        """``dist.scatter``: the root's list flattened, flxScatter into each
        rank's output."""
        root = opts.rootRank if opts is not None else 0
        me = self.rank()
        for i, out in enumerate(output_tensors):
            flat = torch.cat([t.reshape(-1) for t in input_tensors[i]]) if me == root else None
            res = out if out.is_contiguous() else torch.empty_like(out)
            self.comm.scatter(flat, res.view(-1), root=root, stream=self._stream)
            if res is not out:
                out.copy_(res)
        return _DoneWork(output_tensors, self._stream)


def _create(store, rank, size, timeout):
    return FlexLinkBackend(store, rank, size, timeout)


def register() -> None:
    """Make ``"flexlink"`` a torch.distributed backend name (idempotent)."""
    if hasattr(dist.Backend, BACKEND.upper()):
        return
    dist.Backend.register_backend(BACKEND, _create, devices=["cuda"])


def backend_of(group=None) -> FlexLinkBackend:
    """The FlexLink backend object behind ``group`` (default: the last created)."""
    if not _instances:
        raise RuntimeError("no FlexLink process group has been created")
    if group is None:
        return _instances[-1]
    try:  # the group's own CUDA backend object, when torch exposes it
        b = group._get_backend(torch.device("cuda"))
        if isinstance(b, FlexLinkBackend):
            return b
    except Exception:
        pass
    for inst in reversed(_instances):
        if inst.rank() == dist.get_rank(group) and inst.size() == dist.get_world_size(group):
            return inst
    raise RuntimeError("group is not a FlexLink process group")
