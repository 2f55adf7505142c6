"""Seam-sharded fold of one panorama over several GPUs (SURVEY.md §8(e),
BASELINE.json configs[3]: "overlap pairs sharded one per GPU ... with P2P
canvas gather").

One process per GPU, each holding the same ``Plan``.  ``fs_shard_schedule``
(include/fs_b200.h) assigns folds (overlap pairs) to ranks and splits the
execution into segments; after each segment the ranks exchange fold
"strips" — a fold's blended Area3 box (float4) — point to point: to rank 0,
the canvas GPU, which composes every strip in fold order into the RGBA8
panorama, and to a rank whose fold's L crop overlaps an earlier fold's box
(the C2 top/bottom bands read the seams' blended rows).  Transfers go over
``torch.distributed`` P2P (NCCL over NVLink on the B200 box) on the stream the
segments run on, so no host synchronisation sits between segments.

Exactness: every rank composes the first-cover copies of every view and the
strips its folds depend on, so a fold's crop is identical to the sequential
fold's; its blend taps are checked on the device against the canvas region
the rank holds final (``ReachCheck``, fs_device.cuh).  A tap outside it makes
``fs_plan_check`` return FS_ERR_SHARD_REACH on that rank, and
``ShardedPlan.run`` repeats the panorama unsharded on rank 0 — the result is
always the sequential fold's (proj/src/pipeline.cpp:150-204).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _native as N
from .plan import Plan, _raise


@dataclass(frozen=True)
class Xfer:
    fold: int
    src: int
    dst: int
    stage: int


@dataclass
class Schedule:
    fold_rank: List[int]   # [n]; entry 0 (view 0's placement) is rank 0
    stage: List[int]       # [n]; the segment computing fold k
    n_segments: int
    xfers: List[Xfer]      # every transfer of every rank, in issue order

    def xfers_after(self, segment: int, rank: Optional[int] = None) -> List[Xfer]:
        return [x for x in self.xfers if x.stage == segment and
                (rank is None or rank in (x.src, x.dst))]


def shard_schedule(boxes: Sequence[Sequence[int]], nranks: int,
                   fold_rank: Optional[Sequence[int]] = None) -> Schedule:
    """Host-only schedule of folds 1..n-1 with Area3 boxes ``boxes[k]`` =
    (x0, y0, w, h) (boxes[0] ignored) over ``nranks`` GPUs."""
    n = len(boxes)
    b = np.zeros((n, 4), np.int32)
    for k in range(1, n):
        b[k] = boxes[k]
    fr = np.full(n, -1, np.int32)
    if fold_rank is not None:
        fr[1:] = np.asarray(fold_rank, np.int32)[1:]
    stage = np.zeros(n, np.int32)
    nseg = C.c_int()
    cap = max(1, n * nranks)
    xf = (N.StripXfer * cap)()
    nx = C.c_int()
    _raise(N.lib.fs_shard_schedule(n, b.ctypes.data_as(C.c_void_p), nranks,
                                   fr.ctypes.data_as(C.c_void_p), stage.ctypes.data_as(C.c_void_p),
                                   C.byref(nseg), xf, cap, C.byref(nx)))
    return Schedule([int(v) for v in fr], [int(v) for v in stage], nseg.value,
                    [Xfer(x.fold, x.src, x.dst, x.stage) for x in xf[:nx.value]])


class _DeviceBytes:
    """A device allocation exposed through __cuda_array_interface__ (torch
    wraps it without a copy)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class TorchDistTransport:
    """Strip exchange over torch.distributed point-to-point (NCCL on GPUs:
    NVLink/NVSwitch between the B200s of one node; gloo works for tensors on
    the host)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def exchange(self, rank: int, xfers: Sequence[Xfer], strip: Callable[[int], "object"]):
        dist = self.dist
        ops = []
        for x in xfers:  # same global order on every rank: pairs match in issue order
            if x.src == rank:
                ops.append(dist.P2POp(dist.isend, strip(x.fold), x.dst, self.group))
            elif x.dst == rank:
                ops.append(dist.P2POp(dist.irecv, strip(x.fold), x.src, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def max_status(self, status: int) -> int:
        import torch
        dist = self.dist
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([int(status)], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return int(t.item())


def _stream_handle(stream) -> int:
    if stream is not None:
        return int(stream)
    import torch
    return int(torch.cuda.current_stream().cuda_stream)


class ShardedPlan:
    """This rank's share of a seam-sharded plan (one process per GPU)."""

    def __init__(self, plan: Plan, nranks: int, rank: int,
                 fold_rank: Optional[Sequence[int]] = None, transport=None):
        self.plan, self.nranks, self.rank = plan, int(nranks), int(rank)
        self.transport = transport
        fr = None
        if fold_rank is not None:
            fr = np.asarray(fold_rank, np.int32)
        _raise(N.lib.fs_plan_shard(plan._h, self.nranks, self.rank,
                                   None if fr is None else fr.ctypes.data_as(C.c_void_p)))
        boxes = [(0, 0, 0, 0)] + [plan.fold_info(k)[0] for k in range(1, plan.n)]
        self.schedule = shard_schedule(boxes, self.nranks, fold_rank)
        self.n_segments = N.lib.fs_plan_shard_segments(plan._h)
        assert self.n_segments == self.schedule.n_segments
        self._strips = {}
        self.unsharded = False  # set when a certificate failed: later runs skip sharding

    # ---- buffers ----
    def strip_ptr(self, fold: int):
        ptr = C.c_void_p()
        nb = C.c_size_t()
        _raise(N.lib.fs_plan_strip_buffer(self.plan._h, fold, C.byref(ptr), C.byref(nb)))
        return ptr.value, nb.value

    def strip(self, fold: int):
        """Fold's strip buffer as a uint8 torch tensor (no copy)."""
        t = self._strips.get(fold)
        if t is None:
            import torch
            ptr, nb = self.strip_ptr(fold)
            t = torch.as_tensor(_DeviceBytes(ptr, nb), device="cuda")
            self._strips[fold] = t
        return t

    @property
    def launch_count(self) -> int:
        """Kernel launches of one execution of this rank's segments."""
        return N.lib.fs_plan_shard_launch_count(self.plan._h)

    def own_folds(self) -> List[int]:
        return [k for k in range(1, self.plan.n) if self.schedule.fold_rank[k] == self.rank]

    # ---- execution ----
    def execute_segment(self, segment: int, stream=None, view_ptrs=None, out_ptr=None) -> None:
        arg = None
        if view_ptrs is not None and segment == 0:
            arg = C.cast((C.c_void_p * self.plan.n)(*view_ptrs), N.PP)
        outp = C.c_void_p(out_ptr) if out_ptr else None  # rank 0 reads pieces as they finish
        _raise(N.lib.fs_plan_shard_execute(self.plan._h, segment, arg, outp,
                                           C.c_void_p(_stream_handle(stream))))

    def execute(self, stream=None, view_ptrs=None, out_ptr=None) -> None:
        """Every segment with its exchange, asynchronously on `stream` (torch's
        current stream by default: the transport's P2P ops order against it)."""
        for seg in range(self.n_segments):
            self.execute_segment(seg, stream, view_ptrs, out_ptr)
            xs = self.schedule.xfers_after(seg, self.rank)
            if xs:
                self.transport.exchange(self.rank, xs, self.strip)

    def status(self) -> int:
        """fs_plan_check of this rank (call after the stream is synchronised)."""
        return int(N.lib.fs_plan_check(self.plan._h))

    def run(self, view_ptrs=None, out_ptr=None) -> str:
        """One certified panorama: the sharded execution, the ranks' checks
        combined (max status), and on an uncertified blend reach the
        unsharded plan on rank 0.  Returns "sharded" or "unsharded"."""
        import torch
        for attempt in range(2):
            if not self.unsharded:
                self.execute(None, view_ptrs, out_ptr)
                torch.cuda.current_stream().synchronize()
                st = self.status()
                if self.transport is not None:
                    st = self.transport.max_status(st)
                if st == N.FS_OK:
                    return "sharded"
                if st == N.FS_ERR_SHARD_REACH:
                    self.unsharded = True
                elif attempt == 1:
                    _raise(st)
                else:
                    continue  # e.g. a distance-transform domain widened: run again
            if self.rank == 0:
                if view_ptrs is not None or out_ptr:
                    self.plan.execute_ptrs(view_ptrs or [self.plan.view_buffer(k)
                                                         for k in range(self.plan.n)],
                                           out_ptr, _stream_handle(None))
                else:
                    self.plan.execute(_stream_handle(None))
                    torch.cuda.current_stream().synchronize()
                    self.plan.check()
            return "unsharded"
        return "sharded"


class LocalShardGroup:
    """Every rank of a sharded plan in one process on one GPU (tests and
    single-GPU runs of the schedule): the same segments, the exchange as
    device-to-device copies between the ranks' plans, all on one stream."""

    def __init__(self, plans: Sequence[Plan], fold_rank: Optional[Sequence[int]] = None):
        self.shards = [ShardedPlan(p, len(plans), r, fold_rank) for r, p in enumerate(plans)]
        self.schedule = self.shards[0].schedule

    def execute(self, stream=None) -> None:
        s = _stream_handle(stream)
        for seg in range(self.schedule.n_segments):
            for sp in self.shards:
                sp.execute_segment(seg, s)
            for x in self.schedule.xfers_after(seg):
                self.shards[x.dst].strip(x.fold).copy_(self.shards[x.src].strip(x.fold))

    def statuses(self) -> List[int]:
        return [sp.status() for sp in self.shards]

    def run(self) -> str:
        """Certified panorama in plans[0]'s output buffer (ShardedPlan.run's
        protocol: sharded, or unsharded on rank 0 when a reach failed)."""
        import torch
        for attempt in range(2):
            self.execute()
            torch.cuda.current_stream().synchronize()
            st = max(self.statuses())
            if st == N.FS_OK:
                return "sharded"
            if st == N.FS_ERR_SHARD_REACH:
                p0 = self.shards[0].plan
                p0.execute(_stream_handle(None))
                torch.cuda.current_stream().synchronize()
                p0.check()
                return "unsharded"
            if attempt == 1:
                _raise(st)
        return "sharded"
