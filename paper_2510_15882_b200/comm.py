"""Python face of the native data plane: communicators over ``libflexlink.so``.

This is the drop-in seam SURVEY §8(b) names: the reference's collective
executor is ``simulate_collective(topo, spec, shares)``
(`pkg/src/linkstripe/collectives.py:136-186`), injected into Stage 1 through
``initial_tune(measure=...)`` (`tuner.py:178-209`) and called per call by Stage 2
(`balancer.py:190`).  Here the same roles are played by *real* striped
collectives on B200:

* :class:`Communicator` — one rank (``flxCommInitRank``) or one virtual rank of
  a single-GPU clique (``flxCommInitAll`` with a repeated device);
* :class:`Clique` — all virtual ranks of one device, driven together inside
  ``flxGroupStart/End`` (one fused launch);
* :meth:`Clique.measure_fn` — a Stage-1 ``MeasureFn`` returning a
  :class:`~paper_2510_15882_b200.striping.PathTimingReport` built from CUDA-event
  per-path times;
* :func:`tune_shares` — Stage 1 against the real path plus the "never worse
  than NVLink-only" guard, installed into the native share table.

PyTorch tensors are the host-side currency; the library is loaded with ctypes
and fails loudly when it is missing — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import statistics
from pathlib import Path
from typing import Sequence

from .links import PathKind
from .striping import (GRANULE_TOTAL, CollectiveOp, PathTimingReport, ShareDistribution,
                       size_bucket)

__all__ = ["FlexLinkError", "load_library", "Communicator", "Clique", "dtype_code",
           "FLX_BUCKET_ALL", "tune_shares", "library_path"]

FLX_BUCKET_ALL = -2
_LIB_NAME = "libflexlink.so"
_lib = None

_RESULTS = {0: "success", 1: "unhandled cuda error", 2: "system error", 3: "internal error",
            4: "invalid argument", 5: "invalid usage", 6: "remote error", 7: "in progress"}
_OPS = {"sum": 0, "prod": 1, "max": 2, "min": 3, "avg": 4}  # avg: AllReduce / ReduceScatter
_COLL = {CollectiveOp.ALLREDUCE: 0, CollectiveOp.ALLGATHER: 1, CollectiveOp.REDUCESCATTER: 2,
         CollectiveOp.ALLTOALL: 3}


class FlexLinkError(RuntimeError):
    """A non-success ``flxResult_t``; ``code`` is the ncclResult_t-compatible value."""

    def __init__(self, code: int, where: str, detail: str):
        super().__init__(f"{where}: {_RESULTS.get(code, code)} ({detail})")
        self.code = code


class FlexLinkArgumentError(FlexLinkError, ValueError):
    """flxInvalidArgument / flxInvalidUsage — maps to the reference's ValueError."""


def library_path() -> Path:
    override = os.environ.get("FLEXLINK_LIBRARY")
    return Path(override) if override else Path(__file__).resolve().parent / _LIB_NAME


class _UniqueId(ctypes.Structure):
    _fields_ = [("internal", ctypes.c_char * 128)]


def load_library() -> ctypes.CDLL:
    """Load the in-tree ``libflexlink.so``; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not path.exists():
        raise FlexLinkError(5, "load_library",
                            f"{path} is missing; run `python -m paper_2510_15882_b200.build`")
    L = ctypes.CDLL(str(path))
    P, vp, sz, ci = ctypes.POINTER, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    sig = {
        "flxGetVersion": [P(ci)],
        "flxGetUniqueId": [P(_UniqueId)],
        "flxCommInitRank": [P(vp), ci, _UniqueId, ci],
        "flxCommInitAll": [P(vp), ci, P(ci)],
        "flxCommInitLoopback": [P(vp), ci, ci],
        "flxCommDestroy": [vp],
        "flxCommAbort": [vp],
        "flxCommSplit": [vp, ci, ci, P(vp)],
        "flxBroadcast": [vp, vp, ctypes.c_size_t, ci, ci, vp, vp],
        "flxReduce": [vp, vp, ctypes.c_size_t, ci, ci, ci, vp, vp],
        "flxGather": [vp, vp, ctypes.c_size_t, ci, ci, vp, vp],
        "flxScatter": [vp, vp, ctypes.c_size_t, ci, ci, vp, vp],
        "flxCommFinalize": [vp],
        "flxCommCount": [vp, P(ci)],
        "flxCommUserRank": [vp, P(ci)],
        "flxCommCuDevice": [vp, P(ci)],
        "flxCommGetAsyncError": [vp, P(ci)],
        "flxAllReduce": [vp, vp, sz, ci, ci, vp, vp],
        "flxAllGather": [vp, vp, sz, ci, vp, vp],
        "flxReduceScatter": [vp, vp, sz, ci, ci, vp, vp],
        "flxAllToAll": [vp, vp, sz, ci, vp, vp],
        "flxGroupStart": [],
        "flxGroupCollective": [ci, P(vp), ci, P(vp), P(vp), sz, ci, ci, vp],
        "flxGroupEnd": [],
        "flxSetShares": [vp, ci, ci, P(ci)],
        "flxGetShares": [vp, ci, ci, P(ci)],
        "flxGetPathTimes": [vp, P(ctypes.c_float)],
        "flxGetPathTimesHistory": [vp, ci, P(ctypes.c_float), P(ci)],
        "flxGetPathBytes": [vp, P(sz)],
        "flxGetAlignment": [vp, ci, P(sz)],
        "flxSetNvlinkCtas": [vp, ci],
        "flxSetTiming": [vp, ci],
        "flxSetStaging": [vp, sz, ci],
        "flxGetPathMask": [vp, P(ci)],
        "flxGetLaunchCount": [P(ctypes.c_ulonglong)],
        "flxCommDebugPeer": [vp, ci, ci, ci, vp, sz],
        "flxNvlsProbe": [ci, P(ci), ctypes.c_char_p, sz],
        "flxDebugHostRemoteRanks": [ci, ci, _UniqueId, ctypes.c_double],
        "flxCommInitLoopbackIpc": [P(vp), ci, ci, _UniqueId],
        "flxCommGetNvls": [vp, P(ci), ctypes.c_char_p, sz],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ci
    L.flxGetErrorString.argtypes = [ci]
    L.flxGetErrorString.restype = ctypes.c_char_p
    L.flxGetLastError.argtypes = []
    L.flxGetLastError.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(code: int, where: str) -> None:
    if code != 0:
        detail = load_library().flxGetLastError().decode(errors="replace")
        cls = FlexLinkArgumentError if code in (4, 5) else FlexLinkError
        raise cls(code, where, detail)


def dtype_code(dtype) -> int:
    """torch dtype -> flxDataType_t (== ncclDataType_t)."""
    import torch

    table = {torch.int8: 0, torch.uint8: 1, torch.int32: 2, torch.uint32: 3, torch.int64: 4,
             torch.uint64: 5, torch.float16: 6, torch.float32: 7, torch.float64: 8,
             torch.bfloat16: 9}
    if dtype not in table:
        raise ValueError(f"unsupported dtype {dtype}")
    return table[dtype]


def _stream_handle(stream, device: int | None = None) -> ctypes.c_void_p:
    import torch

    if stream is None:
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        if device is not None and raw is not None:  # no Stream object per call
            return ctypes.c_void_p(raw(device))
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _contiguous_cuda(t, what: str):
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    return t


def _granule_array(shares) -> ctypes.Array:
    if isinstance(shares, ShareDistribution):
        g = shares.as_array()
    elif isinstance(shares, dict):
        g = [int(shares.get(k, 0)) for k in PathKind]
    else:
        g = list(shares)
    return (ctypes.c_int * 3)(*g)


class Communicator:
    """One rank of a FlexLink communicator (owns an ``flxComm_t``)."""

    def __init__(self, handle: int, clique: "Clique | None" = None):
        self._h = ctypes.c_void_p(handle)
        self.clique = clique
        L = load_library()
        v = ctypes.c_int()
        _check(L.flxCommCount(self._h, ctypes.byref(v)), "flxCommCount")
        self.nranks = v.value
        _check(L.flxCommUserRank(self._h, ctypes.byref(v)), "flxCommUserRank")
        self.rank = v.value
        _check(L.flxCommCuDevice(self._h, ctypes.byref(v)), "flxCommCuDevice")
        self.device = v.value

    def async_error(self) -> int:
        """``ncclCommGetAsyncError``: 3 (internal error) once a peer wait timed out."""
        v = ctypes.c_int()
        _check(load_library().flxCommGetAsyncError(self._h, ctypes.byref(v)),
               "flxCommGetAsyncError")
        return v.value

    # ---- construction
    @staticmethod
    def unique_id() -> bytes:
        uid = _UniqueId()
        _check(load_library().flxGetUniqueId(ctypes.byref(uid)), "flxGetUniqueId")
        return ctypes.string_at(ctypes.addressof(uid), 128)  # .internal stops at NUL

    @classmethod
    def init_rank(cls, nranks: int, unique_id: bytes, rank: int) -> "Communicator":
        uid = _UniqueId()
        if len(unique_id) != 128:
            raise ValueError("a flxUniqueId is 128 bytes")
        ctypes.memmove(ctypes.addressof(uid), unique_id, 128)
        h = ctypes.c_void_p()
        _check(load_library().flxCommInitRank(ctypes.byref(h), nranks, uid, rank),
               "flxCommInitRank")
        return cls(h.value)

    @classmethod
    def from_process_group(cls, group=None) -> "Communicator":
        """Bootstrap over torch.distributed (one process per GPU)."""
        import torch.distributed as dist

        uid = broadcast_unique_id(group)
        return cls.init_rank(dist.get_world_size(group), uid, dist.get_rank(group))

    def split(self, color: int, key: int = 0) -> "Communicator | None":
        """``ncclCommSplit``: collective over every rank of this communicator;
        ranks with the same ``color`` form a new one ordered by ``key`` (ties:
        this rank); ``color=-1`` (NCCL_SPLIT_NOCOLOR) joins none -> None."""
        h = ctypes.c_void_p()
        _check(load_library().flxCommSplit(self._h, color, key, ctypes.byref(h)), "flxCommSplit")
        return type(self)(h.value) if h.value else None

    def destroy(self) -> None:
        if self._h:
            _check(load_library().flxCommDestroy(self._h), "flxCommDestroy")
            self._h = ctypes.c_void_p()

    def finalize(self) -> None:
        """``ncclCommFinalize``: wait for the comm's side streams to go idle."""
        _check(load_library().flxCommFinalize(self._h), "flxCommFinalize")

    def abort(self) -> None:
        """``ncclCommAbort``: give up on peers (no destroy barrier), then free."""
        if self._h:
            _check(load_library().flxCommAbort(self._h), "flxCommAbort")
            self._h = ctypes.c_void_p()

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    # ---- collectives (ncclAllReduce / ncclAllGather shapes)
    def all_reduce(self, send, recv=None, op: str = "sum", stream=None):
        """Striped AllReduce; in place when ``recv`` is None or ``recv is send``."""
        _contiguous_cuda(send, "send")
        recv = send if recv is None else _contiguous_cuda(recv, "recv")
        if recv.numel() != send.numel() or recv.dtype != send.dtype:
            raise ValueError("recv must match send in size and dtype")
        _check(load_library().flxAllReduce(
            ctypes.c_void_p(send.data_ptr()), ctypes.c_void_p(recv.data_ptr()), send.numel(),
            dtype_code(send.dtype), _OPS[op], self._h, _stream_handle(stream, send.get_device())), "flxAllReduce")
        return recv

    def gather(self, send, recv=None, root: int = 0, stream=None):
        """``ncclGather``: every rank's ``send`` into ``root``'s ``recv`` (rank i's
        elements at i*send.numel()); ``recv`` is unused elsewhere."""
        _contiguous_cuda(send, "send")
        if self.rank == root:
            _contiguous_cuda(recv, "recv")
            if recv.numel() != send.numel() * self.nranks or recv.dtype != send.dtype:
                raise ValueError("the root's recv holds nranks blocks of send's size and dtype")
        _check(load_library().flxGather(
            ctypes.c_void_p(send.data_ptr()),
            ctypes.c_void_p(recv.data_ptr() if recv is not None else 0), send.numel(),
            dtype_code(send.dtype), root, self._h, _stream_handle(stream, send.get_device())),
            "flxGather")
        return recv

    def scatter(self, send, recv, root: int = 0, stream=None):
        """``ncclScatter``: block i of ``root``'s ``send`` (nranks blocks of
        recv.numel()) into rank i's ``recv``; ``send`` is unused elsewhere."""
        _contiguous_cuda(recv, "recv")
        if self.rank == root:
            _contiguous_cuda(send, "send")
            if send.numel() != recv.numel() * self.nranks or recv.dtype != send.dtype:
                raise ValueError("the root's send holds nranks blocks of recv's size and dtype")
        _check(load_library().flxScatter(
            ctypes.c_void_p(send.data_ptr() if send is not None else 0),
            ctypes.c_void_p(recv.data_ptr()), recv.numel(), dtype_code(recv.dtype), root,
            self._h, _stream_handle(stream, recv.get_device())), "flxScatter")
        return recv

    def reduce(self, send, recv=None, op: str = "sum", root: int = 0, stream=None):
        """``ncclReduce``: the fold of every rank's ``send`` into ``root``'s
        ``recv`` (``recv`` is not touched on the other ranks and may be None)."""
        _contiguous_cuda(send, "send")
        if recv is not None:
            _contiguous_cuda(recv, "recv")
            if recv.numel() != send.numel() or recv.dtype != send.dtype:
                raise ValueError("recv must match send in size and dtype")
        elif self.rank == root:
            raise ValueError("the root needs a recv tensor")
        _check(load_library().flxReduce(
            ctypes.c_void_p(send.data_ptr()),
            ctypes.c_void_p(recv.data_ptr() if recv is not None else 0), send.numel(),
            dtype_code(send.dtype), _OPS[op], root, self._h,
            _stream_handle(stream, send.get_device())), "flxReduce")
        return recv

    def broadcast(self, send, recv=None, root: int = 0, stream=None):
        """``ncclBroadcast``: ``root``'s ``send`` into every rank's ``recv`` (in
        place when ``recv`` is None); bit-exact for any dtype."""
        recv = send if recv is None else _contiguous_cuda(recv, "recv")
        _contiguous_cuda(send, "send")
        if recv.numel() != send.numel() or recv.dtype != send.dtype:
            raise ValueError("recv must match send in size and dtype")
        _check(load_library().flxBroadcast(
            ctypes.c_void_p(send.data_ptr()), ctypes.c_void_p(recv.data_ptr()), send.numel(),
            dtype_code(send.dtype), root, self._h, _stream_handle(stream, send.get_device())),
            "flxBroadcast")
        return recv

    def all_gather(self, send, recv, stream=None):
        _contiguous_cuda(send, "send")
        _contiguous_cuda(recv, "recv")
        if recv.numel() != send.numel() * self.nranks or recv.dtype != send.dtype:
            raise ValueError("recv must hold nranks * send.numel() elements of send.dtype")
        _check(load_library().flxAllGather(
            ctypes.c_void_p(send.data_ptr()), ctypes.c_void_p(recv.data_ptr()), send.numel(),
            dtype_code(send.dtype), self._h, _stream_handle(stream, send.get_device())), "flxAllGather")
        return recv

    def reduce_scatter(self, send, recv, op: str = "sum", stream=None):
        """ncclReduceScatter: ``send`` holds nranks blocks of ``recv.numel()``."""
        _contiguous_cuda(send, "send")
        _contiguous_cuda(recv, "recv")
        if send.numel() != recv.numel() * self.nranks or recv.dtype != send.dtype:
            raise ValueError("send must hold nranks * recv.numel() elements of recv.dtype")
        _check(load_library().flxReduceScatter(
            ctypes.c_void_p(send.data_ptr()), ctypes.c_void_p(recv.data_ptr()), recv.numel(),
            dtype_code(send.dtype), _OPS[op], self._h, _stream_handle(stream, send.get_device())),
            "flxReduceScatter")
        return recv

    def all_to_all(self, send, recv, stream=None):
        """Block j of ``send`` goes to rank j; block i of ``recv`` comes from rank i."""
        _contiguous_cuda(send, "send")
        _contiguous_cuda(recv, "recv")
        if send.numel() != recv.numel() or send.numel() % self.nranks or recv.dtype != send.dtype:
            raise ValueError("send and recv must hold nranks equal blocks of one dtype")
        _check(load_library().flxAllToAll(
            ctypes.c_void_p(send.data_ptr()), ctypes.c_void_p(recv.data_ptr()),
            send.numel() // self.nranks, dtype_code(send.dtype), self._h,
            _stream_handle(stream, send.get_device())), "flxAllToAll")
        return recv

    # ---- balancer plumbing
    def set_shares(self, op: CollectiveOp, shares, nbytes: int | None = None) -> None:
        """Pin the split of one size bucket (or every bucket when ``nbytes`` is None);
        ``shares=None`` unpins it, handing it back to the in-library balancer."""
        bucket = FLX_BUCKET_ALL if nbytes is None else size_bucket(nbytes)
        g = None if shares is None else _granule_array(shares)
        _check(load_library().flxSetShares(self._h, _COLL[CollectiveOp(op)], bucket, g),
               "flxSetShares")

    def get_shares(self, op: CollectiveOp, nbytes: int | None = None) -> ShareDistribution:
        bucket = FLX_BUCKET_ALL if nbytes is None else size_bucket(nbytes)
        g = (ctypes.c_int * 3)()
        _check(load_library().flxGetShares(self._h, _COLL[CollectiveOp(op)], bucket, g),
               "flxGetShares")
        return ShareDistribution({k: g[int(k)] for k in PathKind if g[int(k)] or k == 0})

    def path_times(self) -> dict[PathKind, float]:
        """Seconds from collective start to each path's completion (last call)."""
        ms = (ctypes.c_float * 3)()
        _check(load_library().flxGetPathTimes(self._h, ms), "flxGetPathTimes")
        return {k: ms[int(k)] * 1e-3 for k in PathKind}

    def path_times_history(self, max_calls: int = 64) -> list[dict[PathKind, float]]:
        """Per-path seconds of the last ``max_calls`` calls (oldest first)."""
        ms = (ctypes.c_float * (3 * max_calls))()
        n = ctypes.c_int()
        _check(load_library().flxGetPathTimesHistory(self._h, max_calls, ms, ctypes.byref(n)),
               "flxGetPathTimesHistory")
        return [{k: ms[3 * i + int(k)] * 1e-3 for k in PathKind} for i in range(n.value)]

    def path_bytes(self) -> dict[PathKind, int]:
        b = (ctypes.c_size_t * 3)()
        _check(load_library().flxGetPathBytes(self._h, b), "flxGetPathBytes")
        return {k: int(b[int(k)]) for k in PathKind}

    def alignment(self, op: CollectiveOp) -> int:
        a = ctypes.c_size_t()
        _check(load_library().flxGetAlignment(self._h, _COLL[CollectiveOp(op)],
                                              ctypes.byref(a)), "flxGetAlignment")
        return a.value

    def set_nvlink_ctas(self, n: int) -> None:
        _check(load_library().flxSetNvlinkCtas(self._h, n), "flxSetNvlinkCtas")

    def set_staging(self, chunk_bytes: int = 0, buffers: int = 2) -> None:
        _check(load_library().flxSetStaging(self._h, chunk_bytes, buffers), "flxSetStaging")

    def set_timing(self, enabled: bool) -> None:
        """``flxSetTiming``: per-path CUDA-event timing on (default) or off."""
        _check(load_library().flxSetTiming(self._h, int(bool(enabled))), "flxSetTiming")

    def path_mask(self) -> int:
        m = ctypes.c_int()
        _check(load_library().flxGetPathMask(self._h, ctypes.byref(m)), "flxGetPathMask")
        return m.value

    def nvls(self) -> tuple[bool, str]:
        """Whether this communicator's AllReduce sums run on NVLink-SHARP, and why (not)."""
        on = ctypes.c_int()
        why = ctypes.create_string_buffer(256)
        _check(load_library().flxCommGetNvls(self._h, ctypes.byref(on), why, 256),
               "flxCommGetNvls")
        return bool(on.value), why.value.decode(errors="replace")

    def available_paths(self) -> tuple[PathKind, ...]:
        m = self.path_mask()
        return tuple(k for k in PathKind if m & (1 << int(k)))

    # ---- in-library balancer (include/flexlink_tuner.h)
    def set_autotune(self, enabled: bool) -> None:
        """``flxSetAutoTune``: Stage 1 + Stage 2 inside the library for every
        (collective, size bucket) the user did not pin with :meth:`set_shares`."""
        from . import tuner_native as tn

        _check(tn.lib().flxSetAutoTune(self._h, int(bool(enabled))), "flxSetAutoTune")

    def set_tuner_config(self, stage1=None, stage2=None, min_bytes: int = 0) -> None:
        """TunerConfig / BalancerConfig of the in-library balancer, and the smallest
        per-rank message it tunes."""
        from . import tuner_native as tn

        s1 = ctypes.byref(tn.config_c(stage1)) if stage1 is not None else None
        s2 = ctypes.byref(tn.balancer_config_c(stage2)) if stage2 is not None else None
        _check(tn.lib().flxSetTunerConfig(self._h, s1, s2, int(min_bytes)), "flxSetTunerConfig")

    def set_link_profile(self, topo) -> None:
        """Seed Stage 1 from a (probed) TopologySpec instead of the in-call probe
        round; ``None`` restores the probe."""
        from . import tuner_native as tn

        prof = ctypes.byref(tn.profile_from_topology(topo)) if topo is not None else None
        _check(tn.lib().flxSetLinkProfile(self._h, prof), "flxSetLinkProfile")

    def tune_info(self, op: CollectiveOp, nbytes: int) -> dict:
        """The autotuner's state for the size bucket of ``nbytes`` (per rank)."""
        from . import tuner_native as tn

        info = tn.TuneInfoC()
        _check(tn.lib().flxGetTuneInfo(self._h, _COLL[CollectiveOp(op)], size_bucket(nbytes),
                                       ctypes.byref(info)), "flxGetTuneInfo")
        return info.as_dict()

    def tune_trace(self, op: CollectiveOp, nbytes: int, max_records: int = 128) -> list[dict]:
        """The in-library Stage-1 trace in the reference's record shape."""
        from . import tuner_native as tn

        recs = (tn.TuneRecordC * max_records)()
        n = ctypes.c_int()
        _check(tn.lib().flxGetTuneTrace(self._h, _COLL[CollectiveOp(op)], size_bucket(nbytes),
                                        recs, max_records, ctypes.byref(n)), "flxGetTuneTrace")
        out = []
        for r in recs[:n.value]:
            out.append({"iteration": r.iteration, "action": r.action_string(),
                        "imbalance": r.imbalance, "shares": list(r.shares),
                        "durations_ms": [r.durations[p] if r.timed_mask >> p & 1 else None
                                         for p in range(3)]})
        return out

    def tune_evaluations(self, op: CollectiveOp, nbytes: int, max_records: int = 256) -> list:
        """The in-library Stage-2 evaluations (oldest first)."""
        from . import tuner_native as tn

        recs = (tn.EvalRecordC * max_records)()
        n = ctypes.c_int()
        _check(tn.lib().flxGetTuneEvaluations(self._h, _COLL[CollectiveOp(op)],
                                              size_bucket(nbytes), recs, max_records,
                                              ctypes.byref(n)), "flxGetTuneEvaluations")
        return [{"call": r.call, "gap": r.gap if r.has_gap else None, "moved": r.moved,
                 "source": r.source if r.adjusted else None,
                 "target": r.target if r.adjusted else None, "shares": list(r.shares)}
                for r in recs[:n.value]]


def share_key_bytes(op: CollectiveOp, send, recv, nranks: int) -> int:
    """The per-rank byte count the C executor partitions (and keys shares on):
    AllReduce message, AllGather send, ReduceScatter recv block, AllToAll block."""
    op = CollectiveOp(op)
    if op == CollectiveOp.REDUCESCATTER:
        return recv.numel() * recv.element_size()
    if op == CollectiveOp.ALLTOALL:
        return send.numel() // nranks * send.element_size()
    return send.numel() * send.element_size()


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 mints a flxUniqueId; every rank of ``group`` receives the same bytes."""
    import torch.distributed as dist

    box = [Communicator.unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return box[0]


def agree_report(report: PathTimingReport, group=None) -> PathTimingReport:
    """Max-over-ranks of every path's duration, so all ranks see ONE report.

    Stage 1/2 are deterministic given their inputs (ties break by PathKind,
    `tuner.py:110-118`, `balancer.py:78-79`), so feeding every rank the agreed
    report keeps the share tables identical across ranks — required, since a
    rank whose byte split differed would exchange mismatched slices.
    """
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    vals = torch.tensor([report.durations.get(k, -1.0) for k in PathKind], dtype=torch.float64,
                        device=dev)
    dist.all_reduce(vals, op=dist.ReduceOp.MAX, group=group)
    out = {k: float(vals[int(k)]) for k in PathKind if float(vals[int(k)]) >= 0.0}
    return PathTimingReport.build(report.op, report.n_gpus, report.size, out)


def rank_measure_fn(comm: Communicator, op: CollectiveOp, send, recv, group=None,
                    warmup: int = 2, repeats: int = 5, reduce_op: str = "sum"):
    """Stage-1 ``MeasureFn`` for one rank of a multi-process communicator:
    run the real collective with ``state.shares``, take per-path medians of
    the CUDA-event times, then agree them across ranks (:func:`agree_report`)."""
    import torch

    op = CollectiveOp(op)
    nbytes = share_key_bytes(op, send, recv, comm.nranks)

    def run():
        if op == CollectiveOp.ALLREDUCE:
            comm.all_reduce(send, recv, op=reduce_op)
        elif op == CollectiveOp.ALLTOALL:
            comm.all_to_all(send, recv)
        elif op == CollectiveOp.REDUCESCATTER:
            comm.reduce_scatter(send, recv, op=reduce_op)
        else:
            comm.all_gather(send, recv)

    def measure(state) -> PathTimingReport:
        comm.set_shares(op, state.shares, nbytes)
        for _ in range(warmup):
            run()
        for _ in range(repeats):
            run()
        hist = comm.path_times_history(repeats)
        b = comm.path_bytes()
        torch.cuda.synchronize()
        durations = {k: statistics.median(h[k] for h in hist) for k in state.active if b[k] > 0}
        local = PathTimingReport.build(op, comm.nranks, nbytes, durations)
        return agree_report(local, group)

    return measure


def host_remote_ranks(nranks: int, unique_id: bytes, device: int = 0,
                      seconds: float = 120.0) -> None:
    """``flxDebugHostRemoteRanks``: allocate ranks 1..nranks-1's scratch / flags
    here, export them over CUDA IPC under ``unique_id`` and block until the
    loopback world built on them (``Clique(..., loopback=True, ipc_id=...)`` in
    another process) is destroyed.  Launches no kernels."""
    uid = _UniqueId()
    ctypes.memmove(ctypes.addressof(uid), unique_id, 128)
    _check(load_library().flxDebugHostRemoteRanks(nranks, device, uid, seconds),
           "flxDebugHostRemoteRanks")


def nvls_probe(device: int = 0) -> tuple[bool, str]:
    """``flxNvlsProbe``: can this GPU run the NVLink-SHARP (multimem) AllReduce?
    Checked end to end on a one-device multicast object; returns (ok, reason)."""
    ok = ctypes.c_int()
    why = ctypes.create_string_buffer(256)
    _check(load_library().flxNvlsProbe(device, ctypes.byref(ok), why, 256), "flxNvlsProbe")
    return bool(ok.value), why.value.decode(errors="replace")


def launch_count() -> int:
    c = ctypes.c_ulonglong()
    _check(load_library().flxGetLaunchCount(ctypes.byref(c)), "flxGetLaunchCount")
    return c.value


class Clique:
    """``nranks`` virtual ranks on one GPU (``flxCommInitAll`` with a repeated device).

    Every collective takes one tensor per rank and is issued inside
    ``flxGroupStart/End``, so the library runs it as a single fused launch —
    the 1-GPU stand-in for an N-GPU NVSwitch collective.
    """

    def __init__(self, nranks: int, device: int = 0, loopback: bool = False,
                 ipc_id: bytes | None = None):
        """``loopback=False``: fused virtual ranks (flxCommInitAll, repeated device).
        ``loopback=True``: the multi-GPU engine emulated on one device
        (flxCommInitLoopback) — same kernels/protocols as one-process-per-GPU;
        with ``ipc_id``, ranks 1.. live in another process's memory exported by
        :func:`host_remote_ranks` (flxCommInitLoopbackIpc, a bootstrap self-test)."""
        L = load_library()
        handles = (ctypes.c_void_p * nranks)()
        if loopback and ipc_id is not None:
            uid = _UniqueId()
            ctypes.memmove(ctypes.addressof(uid), ipc_id, 128)
            _check(L.flxCommInitLoopbackIpc(handles, nranks, device, uid),
                   "flxCommInitLoopbackIpc")
        elif loopback:
            _check(L.flxCommInitLoopback(handles, nranks, device), "flxCommInitLoopback")
        else:
            devs = (ctypes.c_int * nranks)(*([device] * nranks))
            _check(L.flxCommInitAll(handles, nranks, devs), "flxCommInitAll")
        self.loopback = loopback
        self._handles = handles
        self.comms = [Communicator(h, self) for h in handles]
        self.nranks = nranks
        self.device = device

    def destroy(self) -> None:
        self._checked = None  # drop the cached tensor references
        for c in self.comms:
            c.destroy()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()

    def _group(self, issue) -> None:
        L = load_library()
        _check(L.flxGroupStart(), "flxGroupStart")
        try:
            for i, c in enumerate(self.comms):
                issue(i, c)
        finally:
            _check(L.flxGroupEnd(), "flxGroupEnd")

    def _validate(self, sends, recvs, gather: bool = False, scatter: bool = False):
        if len(sends) != self.nranks or len(recvs) != self.nranks:
            raise ValueError(f"need one send and one recv tensor per rank ({self.nranks})")
        # the same tensor objects at the same addresses and sizes as the last
        # call in this mode were already checked: skip the per-tensor property
        # reads.  The cache keeps that tensor set referenced (entry [2]), so a
        # freed tensor's id can never alias a new tensor while it is cached.
        key = (gather, scatter, tuple((id(t), t.data_ptr(), t.numel()) for t in sends),
               tuple((id(t), t.data_ptr(), t.numel()) for t in recvs))
        checked = getattr(self, "_checked", None)
        if checked is not None and key == checked[0]:
            return checked[1]
        self._checked = None
        s0 = sends[0]
        if scatter and s0.numel() % self.nranks:
            raise ValueError("reduce_scatter send must hold nranks equal blocks")
        want = s0.numel() * self.nranks if gather else \
            (s0.numel() // self.nranks if scatter else s0.numel())
        for s, r in zip(sends, recvs):
            _contiguous_cuda(s, "send")
            _contiguous_cuda(r, "recv")
            if s.numel() != s0.numel() or s.dtype != s0.dtype or r.numel() != want \
                    or r.dtype != s0.dtype:
                raise ValueError("all ranks need same-shaped send/recv tensors of one dtype")
        ptrs = ctypes.c_void_p * self.nranks
        # the pointer arrays and dtype ride along with the key: a repeated call
        # re-uses them instead of rebuilding 2*nranks ctypes values
        args = (ptrs(*[t.data_ptr() for t in sends]), ptrs(*[t.data_ptr() for t in recvs]),
                dtype_code(s0.dtype))
        self._checked = (key, args, (tuple(sends), tuple(recvs)))
        return args

    def _issue(self, coll: int, args, op: int, stream, count: int) -> None:
        """All ranks' calls in one ``flxGroupCollective`` (== flxGroupStart, one
        call per rank, flxGroupEnd): small messages are host-issue bound."""
        sp, rp, dt = args
        rc = load_library().flxGroupCollective(coll, self._handles, self.nranks, sp, rp, count,
                                               dt, op, _stream_handle(stream, self.device))
        _check(rc, "flxGroupCollective")

    def all_reduce(self, sends: Sequence, recvs: Sequence | None = None, op: str = "sum",
                   stream=None):
        recvs = list(sends) if recvs is None else list(recvs)
        args = self._validate(sends, recvs, gather=False)
        self._issue(0, args, _OPS[op], stream, sends[0].numel())
        return recvs

    def all_gather(self, sends: Sequence, recvs: Sequence, stream=None):
        args = self._validate(sends, recvs, gather=True)
        self._issue(1, args, 0, stream, sends[0].numel())
        return recvs

    def reduce_scatter(self, sends: Sequence, recvs: Sequence, op: str = "sum", stream=None):
        args = self._validate(sends, recvs, scatter=True)
        self._issue(2, args, _OPS[op], stream, recvs[0].numel())
        return recvs

    def all_to_all(self, sends: Sequence, recvs: Sequence, stream=None):
        args = self._validate(sends, recvs)
        if sends[0].numel() % self.nranks:
            raise ValueError("all_to_all buffers must hold nranks equal blocks")
        self._issue(3, args, 0, stream, sends[0].numel() // self.nranks)
        return recvs

    def gather(self, sends: Sequence, recvs: Sequence, root: int = 0, stream=None):
        """``recvs[root]`` gets every virtual rank's send in rank order (one group)."""
        self._group(lambda i, c: c.gather(sends[i], recvs[i], root, stream))
        return recvs

    def scatter(self, sends: Sequence, recvs: Sequence, root: int = 0, stream=None):
        """``recvs[i]`` gets block i of ``sends[root]`` (one group)."""
        self._group(lambda i, c: c.scatter(sends[i], recvs[i], root, stream))
        return recvs

    def reduce(self, sends: Sequence, recvs: Sequence, op: str = "sum", root: int = 0,
               stream=None):
        """``recvs[root]`` gets the fold of every virtual rank's send (one group);
        the other recvs are left as they were."""
        self._validate(sends, recvs)
        self._group(lambda i, c: c.reduce(sends[i], recvs[i], op, root, stream))
        return recvs

    def broadcast(self, sends: Sequence, recvs: Sequence | None = None, root: int = 0,
                  stream=None):
        """Every virtual rank's ``recvs[r]`` gets ``sends[root]`` (one group)."""
        recvs = list(sends) if recvs is None else list(recvs)
        self._validate(sends, recvs)
        self._group(lambda i, c: c.broadcast(sends[i], recvs[i], root, stream))
        return recvs

    def set_shares(self, op: CollectiveOp, shares, nbytes: int | None = None) -> None:
        for c in self.comms:
            c.set_shares(op, shares, nbytes)

    def set_nvlink_ctas(self, n: int) -> None:
        for c in self.comms:
            c.set_nvlink_ctas(n)

    def set_staging(self, chunk_bytes: int = 0, buffers: int = 2) -> None:
        for c in self.comms:
            c.set_staging(chunk_bytes, buffers)

    def set_timing(self, enabled: bool) -> None:
        for c in self.comms:
            c.set_timing(enabled)

    def set_autotune(self, enabled: bool) -> None:
        for c in self.comms:
            c.set_autotune(enabled)

    def set_tuner_config(self, stage1=None, stage2=None, min_bytes: int = 0) -> None:
        for c in self.comms:
            c.set_tuner_config(stage1, stage2, min_bytes)

    def set_link_profile(self, topo) -> None:
        for c in self.comms:
            c.set_link_profile(topo)

    def tune_info(self, op: CollectiveOp, nbytes: int) -> dict:
        return self.comms[0].tune_info(op, nbytes)

    def tune_trace(self, op: CollectiveOp, nbytes: int) -> list[dict]:
        return self.comms[0].tune_trace(op, nbytes)

    def tune_evaluations(self, op: CollectiveOp, nbytes: int) -> list[dict]:
        return self.comms[0].tune_evaluations(op, nbytes)

    def path_times(self) -> dict[PathKind, float]:
        return self.comms[0].path_times()

    def path_bytes(self) -> dict[PathKind, int]:
        return self.comms[0].path_bytes()

    def report(self, op: CollectiveOp, nbytes: int, paths=None) -> PathTimingReport:
        """PathTimingReport of the last call: paths that carried bytes (or ``paths``)."""
        t, b = self.path_times(), self.path_bytes()
        keep = [k for k in PathKind if b[k] > 0] if paths is None else sorted(paths)
        return PathTimingReport.build(CollectiveOp(op), self.nranks, nbytes,
                                      {k: t[k] for k in keep if b[k] > 0})

    def measure_fn(self, op: CollectiveOp, sends, recvs, warmup: int = 2, repeats: int = 5,
                   reduce_op: str = "sum"):
        """A Stage-1 ``MeasureFn``: run the real collective with ``state.shares``.

        Per-path durations are medians over ``repeats`` calls; paths that
        carried no bytes (alignment floor) are left out of the report so the
        tuner treats them as idle.
        """
        import torch

        op = CollectiveOp(op)
        # the byte count the share table is keyed on (per-rank message / send /
        # recv block, as the C executor partitions it)
        nbytes = share_key_bytes(op, sends[0], recvs[0], self.nranks)

        def run():
            if op == CollectiveOp.ALLREDUCE:
                self.all_reduce(sends, recvs, op=reduce_op)
            elif op == CollectiveOp.ALLTOALL:
                self.all_to_all(sends, recvs)
            elif op == CollectiveOp.REDUCESCATTER:
                self.reduce_scatter(sends, recvs, op=reduce_op)
            else:
                self.all_gather(sends, recvs)

        def measure(state) -> PathTimingReport:
            self.set_shares(op, state.shares, nbytes)
            for _ in range(warmup):
                run()
            samples: dict[PathKind, list[float]] = {}
            for _ in range(repeats):
                run()
                t, b = self.path_times(), self.path_bytes()
                for k in state.active:
                    if b[k] > 0:
                        samples.setdefault(k, []).append(t[k])
            torch.cuda.synchronize()
            durations = {k: statistics.median(v) for k, v in samples.items()}
            return PathTimingReport.build(op, self.nranks, nbytes, durations)

        return measure


def tune_shares(clique: Clique, topo, op: CollectiveOp, sends, recvs, config=None,
                warmup: int = 2, repeats: int = 5, reduce_op: str = "sum"):
    """Stage 1 on the real path, guarded, installed for this size bucket.

    Runs ``initial_tune(topo, spec, measure=clique.measure_fn(...))`` restricted
    to the paths the box has, then compares the tuned split with NVLink-only on
    the same measurement; keeps NVLink-only if the striped split is not faster
    (Stage 1 converges on imbalance, not on total time).
    Returns ``(shares, trace, tuned_total_s, nvlink_only_total_s)``.
    """
    from .stage1 import TunerConfig, TunerState, initial_tune
    from .striping import CollectiveSpec

    op = CollectiveOp(op)
    nbytes = share_key_bytes(op, sends[0], recvs[0], clique.nranks)
    avail = set(clique.comms[0].available_paths())
    paths = tuple(k for k in topo.present_paths if k in avail)
    spec = CollectiveSpec(op, max(2, clique.nranks), nbytes)
    measure = clique.measure_fn(op, sends, recvs, warmup, repeats, reduce_op)
    shares, trace = initial_tune(topo, spec, config or TunerConfig(), measure=measure,
                                 paths=paths)
    only_nv = ShareDistribution({PathKind.NVLINK: GRANULE_TOTAL})
    base = measure(TunerState(shares=only_nv, active=frozenset({PathKind.NVLINK}), step=1)).total
    tuned = measure(TunerState(shares=shares, active=frozenset(shares.loaded_paths),
                               step=1)).total
    if tuned >= base:
        shares = only_nv
    clique.set_shares(op, shares, nbytes)
    return shares, trace, tuned, base
