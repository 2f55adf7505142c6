"""B200-native flow+blend path of "High-quality Panorama Stitching based on
Asymmetric Bidirectional Optical Flow" (arXiv 2006.01201): a drop-in for the
reference flowstitch library's flow / blend-field / blend / fold entry points,
implemented as sm_100a CUDA kernels behind a C-ABI (include/fs_b200.h).
"""
from . import _native
from .api import *  # noqa: F401,F403
from .api import __all__ as _api_all
from .plan import Plan
from .shard import ShardedPlan, shard_schedule

__all__ = list(_api_all) + ["Plan", "ShardedPlan", "shard_schedule", "device_available"]


def device_available() -> bool:
    return _native.device_available()
