"""CPU: the C-ABI library (include/fs_b200.h) loads, exports every declared
symbol, validates like the reference before touching a device, and — with no
GPU — refuses to compute instead of falling back to the CPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2006_01201_b200 as fs
from paper_2006_01201_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fs_b200.h")


def header_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 35
    lib = C.CDLL(N.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares a signature for each of them
    assert set(syms) <= set(N.SIGNATURES), set(syms) - set(N.SIGNATURES)


def test_library_is_sm100a_only():
    # the fatbin carries sm_100a SASS (cuobjdump lists the embedded ELF arch)
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def test_defaults_match_reference():
    fp, bp = N.FlowParams(), N.BlendParams()
    N.lib.fs_default_flow_params(C.byref(fp))
    N.lib.fs_default_blend_params(C.byref(bp))
    # flow.hpp:36-44, blender.hpp:12-17
    assert fp.astuple() == (4, 8, 3, 1e-4, 2)
    assert (bp.k_softmax_sharpness, bp.k_flow_mag_coef) == (10.0, 0.05)


def test_pyramid_depth_matches_oracle():
    from oracle import restatement
    o = restatement()
    for w, h, lv in [(20, 20, 5), (667, 2800, 4), (9000, 400, 4), (1024, 1024, 6), (16, 9, 3),
                     (8, 8, 4), (17, 300, 8)]:
        lib = N.lib.fs_pyramid_depth(w, h, lv)
        assert lib == len(o.build_pyramid(np.zeros((h, w), np.float32), lv)), (w, h, lv)


def test_softmax_host_equals_oracle_bitwise():
    from oracle import restatement
    o = restatement()
    rng = np.random.RandomState(1)
    for _ in range(500):
        b = rng.rand()
        args = (1 - b, b, rng.rand() * 30, rng.rand() * 30)
        k, coef = 1 + rng.rand() * 20, rng.rand() * 0.2
        assert fs.softmax_weights(*args, fs.BlendParams(k, coef)) == o.softmax_weights(*args, k, coef)


def test_contract_errors_precede_device_use():
    img = fs.ImageBuf.new(16, 16, 1)
    with pytest.raises(fs.ContractError, match="levels must be >= 1"):
        fs.dense_pyr_lk(img, img, fs.FlowParams(levels=0))
    with pytest.raises(fs.ContractError, match="window_radius"):
        fs.dense_pyr_lk(img, img, fs.FlowParams(window_radius=0))
    with pytest.raises(fs.ContractError):
        fs.dense_pyr_lk(img, fs.ImageBuf.new(8, 16, 1))
    with pytest.raises(fs.LayoutError, match="does not fit"):
        fs.place_on_canvas(img, 10, 0, 20, 20)
    with pytest.raises(fs.ContractError, match="at least two images"):
        fs.stitch_placed([fs.PlacedImage(fs.ImageBuf.new(4, 4, 3))], 10, 10)
    with pytest.raises(fs.ContractError, match="channels must be 1 or 3"):
        fs.ImageBuf.new(4, 4, 2)
    with pytest.raises(fs.ContractError):
        fs.compute_partition(fs.Mask(np.zeros((3, 3), np.uint8)), fs.Mask(np.zeros((3, 4), np.uint8)))


@pytest.mark.skipif(fs.device_available(), reason="a device is present")
def test_no_cpu_fallback_without_device():
    img = fs.ImageBuf.new(16, 16, 3)
    with pytest.raises(fs.DeviceError, match="no CPU fallback"):
        fs.to_gray(img)
    with pytest.raises(fs.DeviceError):
        fs.distance_transform(fs.Mask(np.ones((4, 4), np.uint8)))
    with pytest.raises(fs.DeviceError):
        fs.Plan([(4, 4), (4, 4)], [(0, 0), (2, 0)], 6, 4)
