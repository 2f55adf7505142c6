"""Python mirror of the reference's flow+blend API (namespace ``flowstitch``).

Same names, argument meaning and error behaviour as
/root/reference/proj/include/flowstitch/{image,flow,blend_field,blender,pipeline}.hpp,
with numpy arrays in place of the C++ value types.  Every compute call goes
through the C-ABI (include/fs_b200.h) to the sm_100a kernels; nothing here
computes pixels on the host.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from ._native import BlendParams, FisheyeCamera, FlowParams

__all__ = [
    "FlowstitchError", "ContractError", "EmptyRegionError", "LayoutError", "IoError",
    "FormatError", "DeviceError", "ShardReachError", "ImageBuf", "Mask", "Region", "RegionPartition", "CropResult",
    "FlowField", "FlowParams", "DistanceField", "BlendField", "BlendParams", "PlacedImage",
    "PairStats", "StitchReport", "to_gray", "bilinear_sample", "bilinear_sample_batch",
    "compute_partition", "crop_overlap", "place_on_canvas", "build_pyramid", "dense_pyr_lk",
    "bidirectional_flow", "flow_magnitude", "embed_flow", "distance_transform",
    "compute_blend", "softmax_weights", "blend_pair", "feather_blend", "warp_constituents",
    "misalignment_score", "estimate_translation", "TranslationEstimate", "stitch_placed",
    "FisheyeCamera", "fisheye_map", "remap_rgba8", "chroma_gains", "set_thread_count", "thread_count",
    "resolved_thread_count",
]


# ---- errors (proj/include/flowstitch/errors.hpp:10-37) ----
class FlowstitchError(RuntimeError):
    pass


class ContractError(FlowstitchError):
    pass


class EmptyRegionError(FlowstitchError):
    pass


class LayoutError(FlowstitchError):
    pass


class IoError(FlowstitchError):
    pass


class FormatError(FlowstitchError):
    pass


class ShardReachError(FlowstitchError):
    """A seam-sharded fold's blend sampled panorama pixels its GPU does not
    hold final: the sharded result is not certified (run unsharded)."""


class DeviceError(FlowstitchError):
    """No usable sm_100 device, or a CUDA failure (there is no CPU fallback)."""


_ERRORS = {1: ContractError, 2: EmptyRegionError, 3: LayoutError, 4: DeviceError,
           5: DeviceError, 6: ContractError, 7: IoError, 8: FormatError,
           9: ShardReachError}


def _check(status: int) -> None:
    if status != N.FS_OK:
        raise _ERRORS.get(status, FlowstitchError)(N.last_error())


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a if shape is None else a.reshape(shape)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


# ---- value types (image.hpp, flow.hpp, blend_field.hpp) ----
@dataclass
class ImageBuf:
    """Interleaved float raster in [0,1] + validity (image.hpp:32-64).
    data: (h, w, ch) float32, valid: (h, w) uint8."""
    data: np.ndarray
    valid: np.ndarray

    def __post_init__(self):
        self.data = _f32(self.data)
        if self.data.ndim == 2:
            self.data = self.data[:, :, None]
        if self.data.shape[2] not in (1, 3):
            raise ContractError("ImageBuf: channels must be 1 or 3")
        self.valid = _u8(self.valid)

    @classmethod
    def new(cls, width: int, height: int, channels: int, fill: float = 0.0, valid: bool = True):
        if channels not in (1, 3) or width < 0 or height < 0:
            raise ContractError("ImageBuf: channels must be 1 or 3")
        return cls(np.full((height, width, channels), fill, np.float32),
                   np.full((height, width), 1 if valid else 0, np.uint8))

    @property
    def width(self) -> int:
        return self.data.shape[1]

    @property
    def height(self) -> int:
        return self.data.shape[0]

    @property
    def channels(self) -> int:
        return self.data.shape[2]

    def empty(self) -> bool:
        return self.width == 0 or self.height == 0

    def valid_mask(self) -> "Mask":
        return Mask(self.valid.copy())


@dataclass
class Mask:
    v: np.ndarray  # (h, w) uint8

    @property
    def width(self):
        return self.v.shape[1]

    @property
    def height(self):
        return self.v.shape[0]


class Region:
    Outside, Area1, Area2, Area3 = 0, 1, 2, 3


@dataclass
class RegionPartition:
    label: np.ndarray   # (h, w) uint8
    counts: np.ndarray  # int64[4]

    @property
    def width(self):
        return self.label.shape[1]

    @property
    def height(self):
        return self.label.shape[0]

    def count(self, r: int) -> int:
        return int(self.counts[r])


@dataclass
class CropResult:
    image: ImageBuf
    offset_x: int
    offset_y: int


@dataclass
class FlowField:
    vec: np.ndarray    # (h, w, 2) float32, (dx, dy)
    valid: np.ndarray  # (h, w) uint8

    @classmethod
    def new(cls, w: int, h: int):
        return cls(np.zeros((h, w, 2), np.float32), np.ones((h, w), np.uint8))

    @property
    def width(self):
        return self.vec.shape[1]

    @property
    def height(self):
        return self.vec.shape[0]


@dataclass
class DistanceField:
    d: np.ndarray  # (h, w) float64


@dataclass
class BlendField:
    b: np.ndarray  # (h, w) float64


@dataclass
class PlacedImage:
    image: ImageBuf
    offset_x: int = 0
    offset_y: int = 0


@dataclass
class PairStats:
    overlap_pixels: int = 0
    mean_flow_mag_ltor: float = 0.0
    mean_flow_mag_rtol: float = 0.0
    flow_seconds: float = 0.0
    blend_seconds: float = 0.0
    crop_box: Tuple[int, int, int, int] = (0, 0, 0, 0)
    misalignment_before: Optional[float] = None  # raw L vs R over the overlap
    misalignment_after: Optional[float] = None   # flow-warped constituents


@dataclass
class StitchReport:
    pairs: List[PairStats] = field(default_factory=list)
    total_seconds: float = 0.0


# ---- runtime (parallel.hpp:9-18): the GPU path has no host pool ----
def set_thread_count(n: int) -> None:
    N.lib.fs_set_thread_count(int(n))


def thread_count() -> int:
    return N.lib.fs_thread_count()


def resolved_thread_count() -> int:
    return max(1, thread_count())


# ---- imagecore (image.hpp:94-108) ----
def to_gray(img: ImageBuf) -> ImageBuf:
    """image.hpp:94 — Rec.601 luminance; grayscale passes through."""
    out = np.empty((img.height, img.width, 1), np.float32)
    _check(N.lib.fs_to_gray(_p(img.data), img.width, img.height, img.channels, _p(out), None))
    return ImageBuf(out, img.valid.copy())


def bilinear_sample_batch(img: ImageBuf, xy: np.ndarray) -> np.ndarray:
    """bilinear_sample (image.hpp:98) at n points; xy: (n, 2) float64 -> (n, ch)."""
    xy = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
    out = np.empty((xy.shape[0], img.channels), np.float32)
    _check(N.lib.fs_bilinear_sample(_p(img.data), _p(img.valid), img.width, img.height,
                                    img.channels, _p(xy), xy.shape[0], _p(out), None))
    return out


def bilinear_sample(img: ImageBuf, x: float, y: float) -> np.ndarray:
    """image.hpp:98 — clamp-to-edge bilinear lookup; invalid taps renormalised."""
    return bilinear_sample_batch(img, np.array([[x, y]], np.float64))[0]


def compute_partition(mask_l: Mask, mask_r: Mask) -> RegionPartition:
    """image.hpp:100"""
    if mask_l.v.shape != mask_r.v.shape:
        raise ContractError("compute_partition: mask dimensions differ")
    h, w = mask_l.v.shape
    label = np.empty((h, w), np.uint8)
    counts = np.zeros(4, np.int64)
    _check(N.lib.fs_compute_partition(_p(_u8(mask_l.v)), _p(_u8(mask_r.v)), w, h, _p(label),
                                      _p(counts), None))
    return RegionPartition(label, counts)


def crop_overlap(img: ImageBuf, partition: RegionPartition) -> CropResult:
    """image.hpp:103 — bounding-box crop of Area3."""
    if img.width != partition.width or img.height != partition.height:
        raise ContractError("crop_overlap: image and partition dimensions differ")
    box = np.zeros(4, np.int32)
    counts = np.ascontiguousarray(partition.counts, np.int64)
    _check(N.lib.fs_crop_overlap(_p(img.data), _p(img.valid), img.width, img.height,
                                 img.channels, _p(partition.label), _p(counts), None, None,
                                 _p(box), None))
    out = np.empty((box[3], box[2], img.channels), np.float32)
    ov = np.empty((box[3], box[2]), np.uint8)
    _check(N.lib.fs_crop_overlap(_p(img.data), _p(img.valid), img.width, img.height,
                                 img.channels, _p(partition.label), _p(counts), _p(out), _p(ov),
                                 _p(box), None))
    return CropResult(ImageBuf(out, ov), int(box[0]), int(box[1]))


def place_on_canvas(img: ImageBuf, offset_x: int, offset_y: int, canvas_width: int,
                    canvas_height: int) -> ImageBuf:
    """image.hpp:107-108"""
    out = np.empty((canvas_height, canvas_width, img.channels), np.float32)
    ov = np.empty((canvas_height, canvas_width), np.uint8)
    _check(N.lib.fs_place_on_canvas(_p(img.data), _p(img.valid), img.width, img.height,
                                    img.channels, offset_x, offset_y, canvas_width,
                                    canvas_height, _p(out), _p(ov), None))
    return ImageBuf(out, ov)


# ---- optflow (flow.hpp:46-66) ----
def _level_dims(w, h, depth):
    dims = []
    for _ in range(depth):
        dims.append((w, h))
        w, h = max(1, w // 2), max(1, h // 2)
    return dims


def build_pyramid(img: ImageBuf, levels: int) -> List[ImageBuf]:
    """flow.hpp:48"""
    if img.channels != 1:
        raise ContractError("build_pyramid: grayscale input required")
    if levels < 1:
        raise ContractError("build_pyramid: levels must be >= 1")
    depth = N.lib.fs_pyramid_depth(img.width, img.height, levels)
    dims = _level_dims(img.width, img.height, depth)
    out = np.empty(sum(w * h for w, h in dims), np.float32)
    d = C.c_int(0)
    _check(N.lib.fs_build_pyramid(_p(img.data), img.width, img.height, levels, _p(out),
                                  C.byref(d), None))
    res, off = [], 0
    for w, h in dims:
        res.append(ImageBuf(out[off:off + w * h].reshape(h, w, 1).copy(),
                            np.ones((h, w), np.uint8)))
        off += w * h
    return res


def dense_pyr_lk(frm: ImageBuf, to: ImageBuf, params: FlowParams = None) -> FlowField:
    """flow.hpp:52 — coarse-to-fine dense LK; from(p) ~ to(p + d)."""
    params = params or FlowParams()
    if frm.width != to.width or frm.height != to.height:
        raise ContractError("dense_pyr_lk: dimension mismatch")
    if frm.channels != 1 or to.channels != 1:
        raise ContractError("dense_pyr_lk: grayscale inputs required")
    f = FlowField.new(frm.width, frm.height)
    _check(N.lib.fs_dense_pyr_lk(_p(frm.data), _p(to.data), frm.width, frm.height,
                                 C.byref(params), _p(f.vec), _p(f.valid), None))
    return f


def bidirectional_flow(overlapped_l: ImageBuf, overlapped_r: ImageBuf,
                       params: FlowParams = None) -> Tuple[FlowField, FlowField]:
    """flow.hpp:56-58 — returns (FlowLtoR, FlowRtoL)."""
    params = params or FlowParams()
    if overlapped_l.width != overlapped_r.width or overlapped_l.height != overlapped_r.height:
        raise ContractError("bidirectional_flow: dimension mismatch")
    if overlapped_l.channels != overlapped_r.channels:
        raise ContractError("bidirectional_flow: channel mismatch")
    w, h = overlapped_l.width, overlapped_l.height
    lr, rl = FlowField.new(w, h), FlowField.new(w, h)
    _check(N.lib.fs_bidirectional_flow(_p(overlapped_l.data), _p(overlapped_r.data), w, h,
                                       overlapped_l.channels, C.byref(params), _p(lr.vec),
                                       _p(lr.valid), _p(rl.vec), _p(rl.valid), None))
    return lr, rl


def flow_magnitude(flow: FlowField) -> np.ndarray:
    """flow.hpp:61"""
    out = np.empty((flow.height, flow.width), np.float32)
    _check(N.lib.fs_flow_magnitude(_p(_f32(flow.vec)), flow.width, flow.height, _p(out), None))
    return out


def embed_flow(flow: FlowField, offset_x: int, offset_y: int, canvas_width: int,
               canvas_height: int) -> FlowField:
    """flow.hpp:65-66"""
    out = FlowField.new(canvas_width, canvas_height)
    _check(N.lib.fs_embed_flow(_p(_f32(flow.vec)), _p(_u8(flow.valid)), flow.width, flow.height,
                               offset_x, offset_y, canvas_width, canvas_height, _p(out.vec),
                               _p(out.valid), None))
    return out


# ---- blendfield (blend_field.hpp:30-34) ----
def distance_transform(mask: Mask) -> DistanceField:
    """blend_field.hpp:32 — exact EDT."""
    h, w = mask.v.shape
    out = np.empty((h, w), np.float64)
    _check(N.lib.fs_distance_transform(_p(_u8(mask.v)), w, h, _p(out), None))
    return DistanceField(out)


def compute_blend(partition: RegionPartition) -> BlendField:
    """blend_field.hpp:34 — Eq. 1."""
    h, w = partition.label.shape
    out = np.empty((h, w), np.float64)
    _check(N.lib.fs_compute_blend(_p(_u8(partition.label)),
                                  _p(np.ascontiguousarray(partition.counts, np.int64)), w, h,
                                  _p(out), None))
    return BlendField(out)


# ---- blender (blender.hpp:19-46) ----
def softmax_weights(blend_l: float, blend_r: float, mag_rtol: float, mag_ltor: float,
                    params: BlendParams = None) -> Tuple[float, float]:
    """blender.hpp:21-23"""
    params = params or BlendParams()
    sl, sr = C.c_double(), C.c_double()
    N.lib.fs_softmax_weights(blend_l, blend_r, mag_rtol, mag_ltor, C.byref(params),
                             C.byref(sl), C.byref(sr))
    return sl.value, sr.value


def _check_canvas(L: ImageBuf, R: ImageBuf, partition: RegionPartition) -> None:
    if (L.width != R.width or L.height != R.height or L.width != partition.width
            or L.height != partition.height or L.channels != R.channels):
        raise ContractError("blend: canvas dimensions or channel counts differ")


def blend_pair(L: ImageBuf, R: ImageBuf, flow_ltor: FlowField, flow_rtol: FlowField,
               blend: BlendField, partition: RegionPartition,
               params: BlendParams = None) -> ImageBuf:
    """blender.hpp:30-33 — Code 1."""
    params = params or BlendParams()
    _check_canvas(L, R, partition)
    shp = partition.label.shape
    if (flow_ltor.vec.shape[:2] != shp or flow_rtol.vec.shape[:2] != shp
            or blend.b.shape != shp):
        raise ContractError("blend_pair: flow or blend field dimensions differ from canvas")
    out = np.empty_like(L.data)
    ov = np.empty(shp, np.uint8)
    _check(N.lib.fs_blend_pair(_p(L.data), _p(L.valid), _p(R.data), _p(R.valid), L.width,
                               L.height, L.channels, _p(_f32(flow_ltor.vec)),
                               _p(_f32(flow_rtol.vec)),
                               _p(np.ascontiguousarray(blend.b, np.float64)),
                               _p(_u8(partition.label)), C.byref(params), _p(out), _p(ov), None))
    return ImageBuf(out, ov)


def feather_blend(L: ImageBuf, R: ImageBuf, blend: BlendField,
                  partition: RegionPartition) -> ImageBuf:
    """blender.hpp:36-37 — linear baseline."""
    _check_canvas(L, R, partition)
    if blend.b.shape != partition.label.shape:
        raise ContractError("feather_blend: blend field dimensions differ from canvas")
    out = np.empty_like(L.data)
    ov = np.empty(partition.label.shape, np.uint8)
    _check(N.lib.fs_feather_blend(_p(L.data), _p(L.valid), _p(R.data), _p(R.valid), L.width,
                                  L.height, L.channels,
                                  _p(np.ascontiguousarray(blend.b, np.float64)),
                                  _p(_u8(partition.label)), _p(out), _p(ov), None))
    return ImageBuf(out, ov)


def warp_constituents(L: ImageBuf, R: ImageBuf, flow_ltor: FlowField, flow_rtol: FlowField,
                      blend: BlendField, partition: RegionPartition) -> Tuple[ImageBuf, ImageBuf]:
    """blender.hpp:42-46"""
    _check_canvas(L, R, partition)
    ol, orr = np.empty_like(L.data), np.empty_like(R.data)
    ovl, ovr = np.empty_like(L.valid), np.empty_like(R.valid)
    _check(N.lib.fs_warp_constituents(_p(L.data), _p(L.valid), _p(R.data), _p(R.valid),
                                      L.width, L.height, L.channels, _p(_f32(flow_ltor.vec)),
                                      _p(_f32(flow_rtol.vec)),
                                      _p(np.ascontiguousarray(blend.b, np.float64)),
                                      _p(_u8(partition.label)), _p(ol), _p(ovl), _p(orr),
                                      _p(ovr), None))
    return ImageBuf(ol, ovl), ImageBuf(orr, ovr)


@dataclass
class TranslationEstimate:
    """pipeline.hpp:69-73"""
    dx: int = 0
    dy: int = 0
    score: float = 0.0


def estimate_translation(A: ImageBuf, B: ImageBuf, max_shift: int) -> TranslationEstimate:
    """pipeline.hpp:75-77 — exhaustive integer-shift NCC search (grayscale)."""
    if A.channels != 1 or B.channels != 1:
        raise ContractError("estimate_translation: grayscale inputs required")
    if A.width != B.width or A.height != B.height:
        raise ContractError("estimate_translation: dimension mismatch")
    dx, dy, sc = C.c_int(), C.c_int(), C.c_double()
    _check(N.lib.fs_estimate_translation(_p(A.data), _p(B.data), A.width, A.height, 1, max_shift,
                                         C.byref(dx), C.byref(dy), C.byref(sc), None))
    return TranslationEstimate(dx.value, dy.value, sc.value)


def misalignment_score(L: ImageBuf, R: ImageBuf, partition: RegionPartition,
                       patch_radius: int = 8, stride: int = 32) -> float:
    """pipeline.hpp:81-83 — mean shift norm of the best NCC match of every
    textured patch inside Area3 (src/pipeline.cpp:309-396)."""
    if (L.width != R.width or L.height != R.height or L.width != partition.label.shape[1]
            or L.height != partition.label.shape[0]):
        raise ContractError("misalignment_score: dimension mismatch")
    out = C.c_double()
    _check(N.lib.fs_misalignment_score(_p(L.data), _p(L.valid), _p(R.data), _p(R.valid), L.width,
                                       L.height, L.channels, _p(_u8(partition.label)),
                                       _p(np.ascontiguousarray(partition.counts, np.int64)),
                                       patch_radius, stride, C.byref(out), None))
    return out.value


# ---- pipeline fold (pipeline.hpp:63-67) ----
def stitch_placed(placed: Sequence[PlacedImage], canvas_width: int, canvas_height: int,
                  flow_params: FlowParams = None,
                  blend_params: BlendParams = None) -> Tuple[ImageBuf, StitchReport]:
    """pipeline.hpp:64-67 — left-to-right fold, the running panorama plays L.
    Runs device-resident; the report carries per-pair device timings and the
    reference's seam metrics (misalignment before / after, bit-identical)."""
    import time
    flow_params = flow_params or FlowParams()
    blend_params = blend_params or BlendParams()
    n = len(placed)
    if n < 2:
        raise ContractError("stitch: at least two images required")
    ch = placed[0].image.channels
    if any(p.image.channels != ch for p in placed):
        raise ContractError("stitch: mixed grayscale and color inputs")
    imgs = (C.c_void_p * n)(*[p.image.data.ctypes.data for p in placed])
    vals = (C.c_void_p * n)(*[p.image.valid.ctypes.data for p in placed])
    dims = np.array([[p.image.width, p.image.height] for p in placed], np.int32).ravel()
    offs = np.array([[p.offset_x, p.offset_y] for p in placed], np.int32).ravel()
    out = np.empty((canvas_height, canvas_width, ch), np.float32)
    ov = np.empty((canvas_height, canvas_width), np.uint8)
    stats = (N.PairStats * (n - 1))()
    t0 = time.perf_counter()
    _check(N.lib.fs_stitch_placed(n, C.cast(imgs, N.PP), C.cast(vals, N.PP), _p(dims), _p(offs),
                                  ch, canvas_width, canvas_height, C.byref(flow_params),
                                  C.byref(blend_params), _p(out), _p(ov),
                                  C.cast(stats, C.c_void_p), None))
    rep = StitchReport(total_seconds=time.perf_counter() - t0)
    for s in stats:
        rep.pairs.append(PairStats(int(s.overlap_pixels), s.mean_flow_mag_ltor,
                                   s.mean_flow_mag_rtol, s.flow_seconds, s.blend_seconds,
                                   tuple(int(v) for v in s.crop_box),
                                   s.misalignment_before if s.misalignment_present & 1 else None,
                                   s.misalignment_after if s.misalignment_present & 2 else None))
    return ImageBuf(out, ov), rep


# ---- pre-processing: fisheye remap + chromaticity gains (north_star stage 1;
# no reference counterpart — parity unpinned, see include/fs_b200.h) ----
def fisheye_map(cam: FisheyeCamera, canvas_width: int, canvas_height: int, x0: int, y0: int,
                width: int, height: int) -> np.ndarray:
    """Remap table of the canvas rectangle (x0, y0, width, height): (h, w, 2)
    float32 fisheye source positions, (-1, -1) where the ray misses."""
    out = np.empty((height, width, 2), np.float32)
    _check(N.lib.fs_fisheye_map(C.byref(cam), canvas_width, canvas_height, x0, y0, width,
                                height, _p(out)))
    return out


def remap_rgba8(src: np.ndarray, table: np.ndarray, gains=(1.0, 1.0, 1.0)) -> np.ndarray:
    """Bilinear remap of an RGB8/RGBA8 image (h, w, 3|4) through a table, with
    per-channel gains; returns the RGBA8 view (alpha 255 where valid)."""
    src = np.ascontiguousarray(src, np.uint8)
    table = np.ascontiguousarray(table, np.float32)
    if src.ndim != 3 or src.shape[2] not in (3, 4) or table.ndim != 3 or table.shape[2] != 2:
        raise ContractError("remap_rgba8: src must be (h, w, 3|4) uint8, table (h, w, 2)")
    g = np.asarray(gains, np.float32).reshape(3)
    out = np.empty(table.shape[:2] + (4,), np.uint8)
    _check(N.lib.fs_remap_rgba8(_p(src), src.shape[1], src.shape[0], src.shape[2], _p(table),
                                table.shape[1], table.shape[0], _p(g), _p(out), None))
    return out


def chroma_gains(views: Sequence[np.ndarray], offsets: Sequence, canvas_width: int,
                 canvas_height: int) -> np.ndarray:
    """Per-view (n, 3) chromaticity gains from the overlaps of placed RGBA8
    views (view 0 keeps 1; include/fs_b200.h fs_chroma_gains)."""
    vs = [np.ascontiguousarray(v, np.uint8) for v in views]
    n = len(vs)
    dims = np.array([(v.shape[1], v.shape[0]) for v in vs], np.int32).ravel()
    offs = np.array(offsets, np.int32).ravel()
    arr = C.cast((C.c_void_p * n)(*[v.ctypes.data for v in vs]), N.PP)
    out = np.empty((n, 3), np.float32)
    _check(N.lib.fs_chroma_gains(n, arr, _p(dims), _p(offs), canvas_width, canvas_height,
                                 _p(out), None))
    return out
