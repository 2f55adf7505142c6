"""ctypes binding of the B200 C-ABI (include/fs_b200.h).

Loads the in-tree ``libfs_b200.so`` built by ``__graft_entry__.build()`` (or
``make -C paper_2006_01201_b200/csrc``).  There is no fallback: if the library
is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfs_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C paper_2006_01201_b200/csrc` "
        "(or __graft_entry__.build()); the flow+blend path has no CPU fallback")

lib = C.CDLL(LIB_PATH)

FS_OK = 0
STATUS_NAMES = {0: "FS_OK", 1: "FS_ERR_CONTRACT", 2: "FS_ERR_EMPTY_REGION", 3: "FS_ERR_LAYOUT",
                4: "FS_ERR_CUDA", 5: "FS_ERR_OOM", 6: "FS_ERR_UNSUPPORTED", 7: "FS_ERR_IO",
                8: "FS_ERR_FORMAT", 9: "FS_ERR_SHARD_REACH"}
FS_ERR_SHARD_REACH = 9


class FlowParams(C.Structure):
    """fs_flow_params == flowstitch::FlowParams (flow.hpp:36-44)."""
    _fields_ = [("levels", C.c_int), ("window_radius", C.c_int),
                ("iterations_per_level", C.c_int), ("min_eigen_eps", C.c_double),
                ("smoothing_passes", C.c_int)]

    def __init__(self, levels=4, window_radius=8, iterations_per_level=3, min_eigen_eps=1e-4,
                 smoothing_passes=2):
        super().__init__(levels, window_radius, iterations_per_level, min_eigen_eps,
                         smoothing_passes)

    def astuple(self):
        return (self.levels, self.window_radius, self.iterations_per_level, self.min_eigen_eps,
                self.smoothing_passes)


class BlendParams(C.Structure):
    """fs_blend_params == flowstitch::BlendParams (blender.hpp:12-17)."""
    _fields_ = [("k_softmax_sharpness", C.c_double), ("k_flow_mag_coef", C.c_double)]

    def __init__(self, k_softmax_sharpness=10.0, k_flow_mag_coef=0.05):
        super().__init__(k_softmax_sharpness, k_flow_mag_coef)


class PairStats(C.Structure):
    _fields_ = [("overlap_pixels", C.c_int64), ("mean_flow_mag_ltor", C.c_double),
                ("mean_flow_mag_rtol", C.c_double), ("flow_seconds", C.c_double),
                ("blend_seconds", C.c_double), ("crop_box", C.c_int32 * 4),
                ("misalignment_present", C.c_int32), ("misalignment_before", C.c_double),
                ("misalignment_after", C.c_double)]


class FisheyeCamera(C.Structure):
    """fs_fisheye_camera (include/fs_b200.h): equidistant fisheye, radians."""
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("cx", C.c_double), ("cy", C.c_double),
                ("focal", C.c_double), ("radius", C.c_double), ("yaw", C.c_double),
                ("pitch", C.c_double), ("roll", C.c_double)]


class StripXfer(C.Structure):
    """fs_strip_xfer: fold k's strip moves from rank src to rank dst after
    segment `stage`."""
    _fields_ = [("fold", C.c_int), ("src", C.c_int), ("dst", C.c_int), ("stage", C.c_int)]


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 24), ("launches", C.c_int), ("ms", C.c_double),
                ("bytes", C.c_double)]


P = C.c_void_p
I = C.c_int
D = C.c_double
PP = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); every symbol include/fs_b200.h declares
SIGNATURES = {
    "fs_last_error": (C.c_char_p, []),
    "fs_abi_version": (I, []),
    "fs_device_available": (I, []),
    "fs_default_flow_params": (None, [C.POINTER(FlowParams)]),
    "fs_default_blend_params": (None, [C.POINTER(BlendParams)]),
    "fs_to_gray": (I, [P, I, I, I, P, P]),
    "fs_bilinear_sample": (I, [P, P, I, I, I, P, I, P, P]),
    "fs_compute_partition": (I, [P, P, I, I, P, P, P]),
    "fs_crop_overlap": (I, [P, P, I, I, I, P, P, P, P, P, P]),
    "fs_place_on_canvas": (I, [P, P, I, I, I, I, I, I, I, P, P, P]),
    "fs_pyramid_depth": (I, [I, I, I]),
    "fs_build_pyramid": (I, [P, I, I, I, P, P, P]),
    "fs_dense_pyr_lk": (I, [P, P, I, I, C.POINTER(FlowParams), P, P, P]),
    "fs_bidirectional_flow": (I, [P, P, I, I, I, C.POINTER(FlowParams), P, P, P, P, P]),
    "fs_flow_magnitude": (I, [P, I, I, P, P]),
    "fs_embed_flow": (I, [P, P, I, I, I, I, I, I, P, P, P]),
    "fs_distance_transform": (I, [P, I, I, P, P]),
    "fs_compute_blend": (I, [P, P, I, I, P, P]),
    "fs_softmax_weights": (None, [D, D, D, D, C.POINTER(BlendParams), C.POINTER(D),
                                  C.POINTER(D)]),
    "fs_blend_pair": (I, [P, P, P, P, I, I, I, P, P, P, P, C.POINTER(BlendParams), P, P, P]),
    "fs_feather_blend": (I, [P, P, P, P, I, I, I, P, P, P, P, P]),
    "fs_warp_constituents": (I, [P, P, P, P, I, I, I, P, P, P, P, P, P, P, P, P]),
    "fs_misalignment_score": (I, [P, P, P, P, I, I, I, P, P, I, I, P, P]),
    "fs_estimate_translation": (I, [P, P, I, I, I, I, P, P, P, P]),
    "fs_stitch_placed": (I, [I, PP, PP, P, P, I, I, I, C.POINTER(FlowParams),
                             C.POINTER(BlendParams), P, P, P, P]),
    "fs_fisheye_map": (I, [C.POINTER(FisheyeCamera), I, I, I, I, I, I, P]),
    "fs_remap_rgba8": (I, [P, I, I, I, P, I, I, P, P, P]),
    "fs_chroma_gains": (I, [I, PP, P, P, I, I, P, P]),
    "fs_plan_create": (I, [C.POINTER(P), I, I, P, P, I, I, C.POINTER(FlowParams),
                           C.POINTER(BlendParams), PP]),
    "fs_plan_view_buffer": (P, [P, I]),
    "fs_plan_output_buffer": (P, [P]),
    "fs_plan_execute": (I, [P, P]),
    "fs_plan_execute_host": (I, [P, PP, P, P]),
    "fs_plan_execute_host_async": (I, [P, PP, P, P]),
    "fs_plan_check": (I, [P]),
    "fs_plan_launch_count": (I, [P]),
    "fs_plan_set_host_format": (I, [P, I, I]),
    "fs_plan_transfer_bytes": (I, [P, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "fs_plan_set_tiling": (I, [P, I, I]),
    "fs_debug_check_failures": (C.c_uint, [I]),
    "fs_debug_checks_built": (I, []),
    "fs_debug_inject": (None, [I]),
    "fs_plan_tile_count": (I, [P, I]),
    "fs_plan_tile_info": (I, [P, I, I, P, P]),
    "fs_plan_fold_info": (I, [P, I, P, P]),
    "fs_plan_fold_flow": (I, [P, I, P, P, P, P]),
    "fs_plan_profile": (I, [P, P, C.POINTER(KernelStat), I, C.POINTER(I), C.POINTER(D)]),
    "fs_plan_timeline": (I, [P, PP, P, P, C.c_char_p, I]),
    "fs_plan_timeline_graph": (I, [P, PP, P, P, C.c_char_p, I]),
    "fs_plan_destroy": (None, [P]),
    "fs_shard_schedule": (I, [I, P, I, P, P, C.POINTER(I), C.POINTER(StripXfer), I,
                              C.POINTER(I)]),
    "fs_plan_shard": (I, [P, I, I, P]),
    "fs_plan_shard_segments": (I, [P]),
    "fs_plan_shard_launch_count": (I, [P]),
    "fs_plan_shard_xfers": (I, [P, I, C.POINTER(StripXfer), I, C.POINTER(I)]),
    "fs_plan_strip_buffer": (I, [P, I, C.POINTER(P), C.POINTER(C.c_size_t)]),
    "fs_plan_shard_execute": (I, [P, I, PP, P, P]),
    "fs_set_thread_count": (None, [I]),
    "fs_thread_count": (I, []),
}

for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def last_error() -> str:
    msg = lib.fs_last_error()
    return msg.decode() if msg else ""


def device_available() -> bool:
    return bool(lib.fs_device_available())
