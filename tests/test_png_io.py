"""The drop-in's host PNG codec (shim/png_codec.cpp, the reference's
proj/src/png_io.hpp entry points on zlib) against PIL, on CPU.

Decoding must give what the reference's libpng set-up gives
(proj/src/png_io.cpp:45-65): 8-bit samples, palette -> RGB (RGBA with tRNS),
gray below 8 bits scaled to 8, gray/RGB tRNS keys -> alpha, gray+alpha ->
RGBA; 16-bit files refused.  Encoding must round-trip through PIL exactly.
"""
import os
import subprocess

import numpy as np
import pytest
from PIL import Image

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "paper_2006_01201_b200", "shim", "png_tool")

pytestmark = pytest.mark.skipif(not os.path.exists(TOOL), reason="shim not built (no reference)")


def decode(path):
    out = str(path) + ".raw"
    r = subprocess.run([TOOL, "decode", str(path), out], capture_output=True, text=True)
    if r.returncode:
        return r.returncode, r.stderr
    with open(out, "rb") as f:
        head = f.readline().split()
        w, h, c = (int(v) for v in head)
        data = np.frombuffer(f.read(), np.uint8)
    return 0, data.reshape(h, w, c)


def encode(tmp, arr):
    h, w, c = arr.shape
    raw, out = tmp / "in.raw", tmp / "out.png"
    raw.write_bytes(np.ascontiguousarray(arr).tobytes())
    r = subprocess.run([TOOL, "encode", str(w), str(h), str(c), str(raw), str(out)])
    assert r.returncode == 0
    return out


RNG = np.random.RandomState(5)


@pytest.mark.parametrize("mode,ch", [("L", 1), ("RGB", 3), ("RGBA", 4)])
def test_decode_8bit(tmp_path, mode, ch):
    a = RNG.randint(0, 256, size=(37, 53, ch), dtype=np.uint8)
    p = tmp_path / "x.png"
    Image.fromarray(a[..., 0] if ch == 1 else a, mode).save(p)
    st, got = decode(p)
    assert st == 0 and got.shape == (37, 53, ch) and np.array_equal(got, a.reshape(got.shape))


def test_decode_gray_alpha_promoted_to_rgba(tmp_path):
    a = RNG.randint(0, 256, size=(20, 30, 2), dtype=np.uint8)
    p = tmp_path / "la.png"
    Image.fromarray(a, "LA").save(p)
    st, got = decode(p)
    assert st == 0 and got.shape == (20, 30, 4)
    assert np.array_equal(got[..., 0], a[..., 0]) and np.array_equal(got[..., 2], a[..., 0])
    assert np.array_equal(got[..., 3], a[..., 1])


def test_decode_palette_and_trns(tmp_path):
    a = RNG.randint(0, 256, size=(25, 19, 3), dtype=np.uint8)
    im = Image.fromarray(a, "RGB").quantize(colors=40)
    p = tmp_path / "p.png"
    im.save(p)
    st, got = decode(p)
    assert st == 0 and got.shape == (25, 19, 3)
    assert np.array_equal(got, np.asarray(im.convert("RGB")))
    im.info["transparency"] = 3
    p2 = tmp_path / "pt.png"
    im.save(p2, transparency=3)
    st, got = decode(p2)
    ref = np.asarray(Image.open(p2).convert("RGBA"))
    assert st == 0 and got.shape == (25, 19, 4) and np.array_equal(got, ref)


@pytest.mark.parametrize("bits", [1, 2, 4])
def test_decode_low_bit_gray_scaled(tmp_path, bits):
    # PIL writes 1-bit mode "1"; 2/4-bit gray via a palette-free "L" with bits=
    a = RNG.randint(0, 1 << bits, size=(13, 27), dtype=np.uint8)
    p = tmp_path / ("g%d.png" % bits)
    if bits == 1:
        Image.fromarray((a * 255).astype(np.uint8), "L").convert("1").save(p)
    else:
        Image.fromarray((a * (255 // ((1 << bits) - 1))).astype(np.uint8), "L").save(p, bits=bits)
    st, got = decode(p)
    assert st == 0
    ref = np.asarray(Image.open(p).convert("L"))
    assert got.shape[-1] in (1, 3) and np.array_equal(got[..., 0], ref)


def test_gray_trns_key_to_alpha(tmp_path):
    a = RNG.randint(0, 256, size=(11, 9), dtype=np.uint8)
    a[3, 4] = 77
    p = tmp_path / "gk.png"
    Image.fromarray(a, "L").save(p, transparency=77)
    st, got = decode(p)
    assert st == 0 and got.shape == (11, 9, 4)
    assert np.array_equal(got[..., 3], np.where(a == 77, 0, 255).astype(np.uint8))


def test_refusals(tmp_path):
    p = tmp_path / "16.png"
    Image.fromarray(RNG.randint(0, 65535, size=(8, 8)).astype(np.uint16)).save(p)
    st, err = decode(p)
    assert st == 2 and "16-bit PNG not supported" in err
    q = tmp_path / "bad.png"
    q.write_bytes(b"not a png at all")
    st, err = decode(q)
    assert st == 2 and "not a PNG file" in err
    st, err = decode(tmp_path / "missing.png")
    assert st == 2 and "cannot open for reading" in err
    # a corrupted IDAT: CRC mismatch -> decode error
    good = tmp_path / "g.png"
    Image.fromarray(RNG.randint(0, 256, size=(8, 8, 3), dtype=np.uint8), "RGB").save(good)
    b = bytearray(good.read_bytes())
    b[-20] ^= 0xFF
    q.write_bytes(bytes(b))
    st, err = decode(q)
    assert st == 2 and "PNG decode error" in err


@pytest.mark.parametrize("ch,mode", [(1, "L"), (3, "RGB"), (4, "RGBA")])
def test_encode_roundtrip_through_pil(tmp_path, ch, mode):
    # smooth + noisy content so every filter type gets chosen somewhere
    y, x = np.mgrid[0:41, 0:67]
    base = ((x * 3 + y * 5) % 256).astype(np.uint8)
    a = np.stack([base, 255 - base, RNG.randint(0, 256, base.shape).astype(np.uint8),
                  np.full_like(base, 200)], -1)[..., :ch]
    out = encode(tmp_path, a)
    im = Image.open(out)
    assert im.mode == mode and im.size == (67, 41)
    assert np.array_equal(np.asarray(im).reshape(a.shape), a)
    # deterministic: same pixels, same file
    first = out.read_bytes()
    assert encode(tmp_path, a).read_bytes() == first
    st, got = decode(out)
    assert st == 0 and np.array_equal(got, a)


def test_size(tmp_path):
    p = tmp_path / "s.png"
    Image.fromarray(np.zeros((17, 23, 3), np.uint8)).save(p)
    r = subprocess.run([TOOL, "size", str(p)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.split() == ["23", "17"]
