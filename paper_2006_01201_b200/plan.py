"""Planned device-resident fold (fs_plan_* of include/fs_b200.h).

``Plan`` fixes a layout (view sizes, offsets, fold order, canvas) and owns all
device memory; ``execute`` replays one CUDA graph that recomputes the whole
flow+blend fold from the 8-bit views resident in HBM, ``execute_host`` is the
end-to-end call (host views in, host RGBA canvas out).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .api import _ERRORS, FlowstitchError
from ._native import BlendParams, FlowParams


def _raise(st: int):
    if st != N.FS_OK:
        raise _ERRORS.get(st, FlowstitchError)(N.last_error())


class Plan:
    def __init__(self, dims: Sequence, offsets: Sequence, canvas_w: int, canvas_h: int,
                 flow: Optional[FlowParams] = None, blend: Optional[BlendParams] = None,
                 device: int = 0, views_rgba: Optional[Sequence[np.ndarray]] = None):
        self.n = len(dims)
        self.dims = [tuple(int(v) for v in d) for d in dims]
        self.offsets = [tuple(int(v) for v in o) for o in offsets]
        self.canvas_w, self.canvas_h = int(canvas_w), int(canvas_h)
        self.flow = flow or FlowParams()
        self.blend = blend or BlendParams()
        d = np.array(self.dims, np.int32).ravel()
        o = np.array(self.offsets, np.int32).ravel()
        views_arg = None
        keep = None
        if views_rgba is not None:
            keep = [np.ascontiguousarray(v, np.uint8) for v in views_rgba]
            views_arg = C.cast((C.c_void_p * self.n)(*[v.ctypes.data for v in keep]), N.PP)
        h = C.c_void_p()
        _raise(N.lib.fs_plan_create(C.byref(h), device, self.n, d.ctypes.data_as(C.c_void_p),
                                    o.ctypes.data_as(C.c_void_p), self.canvas_w, self.canvas_h,
                                    C.byref(self.flow), C.byref(self.blend), views_arg))
        self._h = h

    # ---- buffers ----
    def view_buffer(self, k: int) -> int:
        return N.lib.fs_plan_view_buffer(self._h, k)

    def output_buffer(self) -> int:
        return N.lib.fs_plan_output_buffer(self._h)

    def fold_info(self, k: int):
        box = np.zeros(4, np.int32)
        depth = C.c_int()
        _raise(N.lib.fs_plan_fold_info(self._h, k, box.ctypes.data_as(C.c_void_p), C.byref(depth)))
        return tuple(int(v) for v in box), depth.value

    def fold_flow(self, k: int):
        """Fold k's crop flows of the last execution: ((ltor vec, valid), (rtol vec, valid)),
        box-sized, the FlowField layout."""
        (x, y, w, h), _ = self.fold_info(k)
        out = [np.empty((h, w, 2), np.float32), np.empty((h, w), np.uint8),
               np.empty((h, w, 2), np.float32), np.empty((h, w), np.uint8)]
        _raise(N.lib.fs_plan_fold_flow(self._h, k, *[o.ctypes.data_as(C.c_void_p) for o in out]))
        return (out[0], out[1]), (out[2], out[3])

    def set_host_format(self, view_channels: int = 4, out_channels: int = 4) -> None:
        """Host views RGB8 (3, all valid) or RGBA8 (4); host canvas RGB8 or RGBA8."""
        _raise(N.lib.fs_plan_set_host_format(self._h, view_channels, out_channels))

    def set_tiling(self, tile_len: int, margin: int = 32) -> None:
        """Row/column tiles of the folds' flows (fs_plan_set_tiling); 0: off."""
        _raise(N.lib.fs_plan_set_tiling(self._h, int(tile_len), int(margin)))

    def tiles(self, k: int):
        """Fold k's tiles in use: [(region, interior)] box-relative {x0, y0, w, h}."""
        n = N.lib.fs_plan_tile_count(self._h, k)
        if n < 0:
            raise ValueError("fold index out of range")
        out = []
        for t in range(n):
            reg, inter = np.zeros(4, np.int32), np.zeros(4, np.int32)
            _raise(N.lib.fs_plan_tile_info(self._h, k, t, reg.ctypes.data_as(C.c_void_p),
                                           inter.ctypes.data_as(C.c_void_p)))
            out.append((tuple(int(v) for v in reg), tuple(int(v) for v in inter)))
        return out

    def transfer_bytes(self):
        """(h2d, d2h) bytes of execute_host with page-locked buffers."""
        a, b = C.c_size_t(), C.c_size_t()
        _raise(N.lib.fs_plan_transfer_bytes(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    @property
    def launch_count(self) -> int:
        return N.lib.fs_plan_launch_count(self._h)

    # ---- execution ----
    def execute(self, stream: int = 0) -> None:
        """Async on `stream` (a cudaStream_t as int): fold the views in HBM."""
        _raise(N.lib.fs_plan_execute(self._h, C.c_void_p(stream)))

    def check(self) -> None:
        _raise(N.lib.fs_plan_check(self._h))

    def execute_host(self, views: Optional[Sequence[np.ndarray]], out: Optional[np.ndarray] = None,
                     stream: int = 0) -> Optional[np.ndarray]:
        """End to end: copy views (RGBA8) in, fold, copy the RGBA8 canvas out."""
        arg = None
        keep = None
        if views is not None:
            keep = [np.ascontiguousarray(v, np.uint8) for v in views]
            arg = C.cast((C.c_void_p * self.n)(*[v.ctypes.data for v in keep]), N.PP)
        outp = None
        if out is not None:
            outp = C.c_void_p(out.ctypes.data)
        _raise(N.lib.fs_plan_execute_host(self._h, arg, outp, C.c_void_p(stream)))
        return out

    def execute_ptrs(self, view_ptrs: Sequence[int], out_ptr: Optional[int],
                     stream: int = 0) -> None:
        """End to end with raw (e.g. pinned host) pointers."""
        arg = C.cast((C.c_void_p * self.n)(*view_ptrs), N.PP)
        _raise(N.lib.fs_plan_execute_host(self._h, arg, C.c_void_p(out_ptr) if out_ptr else None,
                                          C.c_void_p(stream)))

    def execute_ptrs_async(self, view_ptrs: Sequence[int], out_ptr: int, stream: int = 0) -> None:
        """End to end, asynchronous (page-locked buffers): no sync, no check —
        call check() after synchronising the stream."""
        arg = C.cast((C.c_void_p * self.n)(*view_ptrs), N.PP)
        _raise(N.lib.fs_plan_execute_host_async(self._h, arg, C.c_void_p(out_ptr),
                                                C.c_void_p(stream)))

    def timeline(self, view_ptrs: Optional[Sequence[int]] = None, out_ptr: Optional[int] = None,
                 stream: int = 0) -> dict:
        """One DAG execution with timing events at its schedule points
        (ms since start), with the host copies when pointers are given."""
        arg = C.cast((C.c_void_p * self.n)(*view_ptrs), N.PP) if view_ptrs else None
        buf = C.create_string_buffer(1 << 16)
        _raise(N.lib.fs_plan_timeline(self._h, arg, C.c_void_p(out_ptr) if out_ptr else None,
                                      C.c_void_p(stream), buf, len(buf)))
        import json
        return json.loads(buf.value.decode())

    def timeline_graph(self, view_ptrs: Optional[Sequence[int]] = None,
                       out_ptr: Optional[int] = None, stream: int = 0) -> dict:
        """The schedule points inside the production graph (%globaltimer
        stamp kernels), ms since the first."""
        arg = C.cast((C.c_void_p * self.n)(*view_ptrs), N.PP) if view_ptrs else None
        buf = C.create_string_buffer(1 << 16)
        _raise(N.lib.fs_plan_timeline_graph(self._h, arg,
                                            C.c_void_p(out_ptr) if out_ptr else None,
                                            C.c_void_p(stream), buf, len(buf)))
        import json
        return json.loads(buf.value.decode())

    def profile(self, stream: int = 0):
        """One un-captured execution with CUDA events around every launch.
        Returns ({family: {"launches", "ms", "bytes"}}, total_ms)."""
        stats = (N.KernelStat * 32)()
        n = C.c_int()
        tot = C.c_double()
        _raise(N.lib.fs_plan_profile(self._h, C.c_void_p(stream), stats, 32, C.byref(n),
                                     C.byref(tot)))
        out = {}
        for s in stats[:n.value]:
            out[s.name.decode()] = {"launches": s.launches, "ms": s.ms, "bytes": s.bytes}
        return out, tot.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib.fs_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
