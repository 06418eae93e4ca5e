"""PyTorch integration: ``torch.ops.flexlink.*`` custom ops and a process-group-style wrapper.

SURVEY §8(f) row 1: the paper's motivating workload is TP AllReduce inside a
model (Qwen-32B prefill).  Registering the striped
collectives as ``torch.library`` custom ops makes them visible to the
dispatcher (and to ``torch.compile`` / CUDA-graph capture as opaque mutating
ops) instead of hiding them behind Python calls:

* ``torch.ops.flexlink.all_reduce_(x, comm_id, op)``        — in-place, one rank
* ``torch.ops.flexlink.all_gather(x, comm_id) -> Tensor``   — one rank
* ``torch.ops.flexlink.reduce_scatter(x, comm_id, op) -> Tensor`` — one rank
* ``torch.ops.flexlink.all_to_all(x, comm_id) -> Tensor``   — one rank
* ``torch.ops.flexlink.clique_all_reduce_(xs, clique_id, op)`` — all virtual ranks

Communicators are referenced by an integer handle from :func:`register`.
:class:`FlexLinkGroup` offers the ``torch.distributed``-style method names
(``all_reduce``, ``all_gather_into_tensor``, ``reduce_scatter_tensor``,
``all_to_all_single``) over one communicator.
"""

from __future__ import annotations

import itertools

import torch

from .comm import Clique, Communicator

__all__ = ["register", "unregister", "FlexLinkGroup"]

_REGISTRY: dict[int, object] = {}
_IDS = itertools.count(1)


def register(obj: Communicator | Clique) -> int:
    handle = next(_IDS)
    _REGISTRY[handle] = obj
    return handle


def unregister(handle: int) -> None:
    _REGISTRY.pop(handle, None)


def _get(handle: int):
    try:
        return _REGISTRY[handle]
    except KeyError:
        raise ValueError(f"no FlexLink communicator registered under {handle}") from None


@torch.library.custom_op("flexlink::all_reduce_", mutates_args=("x",))
def all_reduce_(x: torch.Tensor, comm_id: int, op: str = "sum") -> None:
    _get(comm_id).all_reduce(x, x, op=op)


@all_reduce_.register_fake
def _all_reduce_fake(x, comm_id, op="sum"):
    return None


@torch.library.custom_op("flexlink::clique_all_reduce_", mutates_args=("xs",))
def clique_all_reduce_(xs: list[torch.Tensor], clique_id: int, op: str = "sum") -> None:
    _get(clique_id).all_reduce(list(xs), list(xs), op=op)


@clique_all_reduce_.register_fake
def _clique_all_reduce_fake(xs, clique_id, op="sum"):
    return None


@torch.library.custom_op("flexlink::all_gather", mutates_args=())
def all_gather(x: torch.Tensor, comm_id: int) -> torch.Tensor:
    comm = _get(comm_id)
    out = x.new_empty((comm.nranks * x.numel(),))
    comm.all_gather(x.contiguous().view(-1), out)
    return out


@all_gather.register_fake
def _all_gather_fake(x, comm_id):
    return x.new_empty((_get(comm_id).nranks * x.numel(),))


@torch.library.custom_op("flexlink::reduce_scatter", mutates_args=())
def reduce_scatter(x: torch.Tensor, comm_id: int, op: str = "sum") -> torch.Tensor:
    comm = _get(comm_id)
    out = x.new_empty((x.numel() // comm.nranks,))
    comm.reduce_scatter(x.contiguous().view(-1), out, op=op)
    return out


@reduce_scatter.register_fake
def _reduce_scatter_fake(x, comm_id, op="sum"):
    return x.new_empty((x.numel() // _get(comm_id).nranks,))


@torch.library.custom_op("flexlink::all_to_all", mutates_args=())
def all_to_all(x: torch.Tensor, comm_id: int) -> torch.Tensor:
    out = torch.empty_like(x).view(-1)
    _get(comm_id).all_to_all(x.contiguous().view(-1), out)
    return out


@all_to_all.register_fake
def _all_to_all_fake(x, comm_id):
    return x.new_empty((x.numel(),))


class FlexLinkGroup:
    """``torch.distributed``-style calls over one FlexLink communicator."""

    def __init__(self, comm: Communicator):
        self.comm = comm
        self.handle = register(comm)

    def size(self) -> int:
        return self.comm.nranks

    def rank(self) -> int:
        return self.comm.rank

    def all_reduce(self, tensor: torch.Tensor, op: str = "sum") -> torch.Tensor:
        torch.ops.flexlink.all_reduce_(tensor, self.handle, op)
        return tensor

    def all_gather_into_tensor(self, output: torch.Tensor, inp: torch.Tensor) -> torch.Tensor:
        self.comm.all_gather(inp.contiguous().view(-1), output.view(-1))
        return output

    def reduce_scatter_tensor(self, output: torch.Tensor, inp: torch.Tensor,
                              op: str = "sum") -> torch.Tensor:
        self.comm.reduce_scatter(inp.contiguous().view(-1), output.view(-1), op=op)
        return output

    def all_to_all_single(self, output: torch.Tensor, inp: torch.Tensor) -> torch.Tensor:
        """Equal splits only (block j of ``inp`` goes to rank j)."""
        self.comm.all_to_all(inp.contiguous().view(-1), output.view(-1))
        return output

    def close(self) -> None:
        unregister(self.handle)
