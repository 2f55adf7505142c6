"""The reference's command-line tool (proj/tools/flowstitch_cli.cpp, UNCHANGED)
relinked against the B200 drop-in (shim/flowstitch_cli_b200), on the
reference's own CLI fixtures (proj/tests/make_fixtures.cpp, built as
shim/make_fixtures_b200): the checks of proj/tests/cli_smoke.sh restated
(subcommands, exit codes, byte-identical output across thread counts, the
restitched panorama against the source texture via PIL), plus the GPU CLI's
outputs against the reference CLI run on the CPU (oracle/_ref/
flowstitch_cli_ref, same fixtures): 8-bit within 1 LSB."""
import json
import os
import struct
import subprocess

import numpy as np
import pytest
from PIL import Image

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "paper_2006_01201_b200", "shim")
CLI = os.path.join(SHIM, "flowstitch_cli_b200")
FIX = os.path.join(SHIM, "make_fixtures_b200")
REF = os.path.join(ROOT, "oracle", "_ref", "flowstitch_cli_ref")


def run(*args, exe=CLI):
    return subprocess.run([exe, *[str(a) for a in args]], capture_output=True, text=True,
                          timeout=600)


@pytest.fixture(scope="module")
def work(tmp_path_factory):
    if not (os.path.exists(CLI) and os.path.exists(FIX)):
        pytest.skip("CLI not built (needs the reference sources at build time)")
    w = tmp_path_factory.mktemp("cli")
    r = subprocess.run([FIX, str(w)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return w


def test_cli_errors_without_gpu_work(work):
    # cli_smoke.sh:67-68: unknown flag -> 1, missing file -> 2
    assert run("stitch", "--no-such-flag").returncode == 1
    assert run("flow", "--from", "/nonexistent.png", "--to", "/nonexistent.png", "--out",
               work / "x.flo").returncode == 2
    assert run().returncode == 1  # a subcommand is required


@pytest.mark.gpu
def test_cli_smoke_on_b200(work):
    # cli_smoke.sh:30-40: self-flow decodes to an all-zero field
    r = run("flow", "--from", work / "gray.png", "--to", work / "gray.png", "--out",
            work / "zero.flo", "--levels", 3, "--window", 5)
    assert r.returncode == 0, r.stderr
    b = (work / "zero.flo").read_bytes()
    assert b[:4] == b"PIEH"
    w, h = struct.unpack("<ii", b[4:12])
    vals = np.frombuffer(b[12:], np.float32)
    assert vals.size == 2 * w * h and np.abs(vals).max() <= 1e-3
    # :43-47 blend a pair; disjoint placements -> exit 1, "no overlap"
    r = run("blend", "--left", work / "strip0.png", "--right", work / "strip1.png",
            "--left-offset", "0,0", "--right-offset", "120,0", "--canvas", "300x150",
            "--out", work / "pair.png", "--dump-blend", work / "blendfield.png")
    assert r.returncode == 0, r.stderr
    r = run("blend", "--left", work / "strip0.png", "--right", work / "strip1.png",
            "--left-offset", "0,0", "--right-offset", "200,0", "--canvas", "400x150",
            "--out", work / "nope.png")
    assert r.returncode == 1 and "no overlap" in r.stderr
    # :49-54 stitch at 1 and 8 threads: byte-identical panoramas, a report
    r = run("stitch", "--layout", work / "three_strip.json", "--out", work / "pano_t1.png",
            "--report", work / "report.json", "--threads", 1)
    assert r.returncode == 0, r.stderr
    r = run("stitch", "--layout", work / "three_strip.json", "--out", work / "pano_t8.png",
            "--threads", 8)
    assert r.returncode == 0, r.stderr
    assert (work / "pano_t1.png").read_bytes() == (work / "pano_t8.png").read_bytes()
    assert "overlap_pixels" in (work / "report.json").read_text()
    # :56-66 the restitched panorama matches the source texture (PIL)
    a = np.asarray(Image.open(work / "pano_t1.png").convert("RGB")).astype(int)
    t = np.asarray(Image.open(work / "texture.png").convert("RGB")).astype(int)
    assert (np.abs(a - t) <= 1).all(-1).mean() >= 0.99
    # :69-71 metrics as JSON
    r = run("metrics", "--left", work / "strip0.png", "--right", work / "strip1.png",
            "--left-offset", "0,0", "--right-offset", "120,0", "--canvas", "300x150", "--json")
    assert r.returncode == 0 and "misalignment_px" in json.loads(r.stdout)


@pytest.mark.gpu
def test_cli_outputs_match_reference_cli(work):
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref/flowstitch_cli_ref not built")
    pairs = [("blend", ["--left", work / "strip0.png", "--right", work / "strip1.png",
                        "--left-offset", "0,0", "--right-offset", "120,0", "--canvas",
                        "300x150"]),
             ("stitch", ["--layout", work / "three_strip.json"])]
    for cmd, args in pairs:
        outs = []
        for exe, tag in ((CLI, "gpu"), (REF, "ref")):
            out = work / ("%s_%s.png" % (cmd, tag))
            r = run(cmd, *args, "--out", out, exe=exe)
            assert r.returncode == 0, (tag, r.stderr)
            outs.append(np.asarray(Image.open(out)).astype(int))
        g, c = outs
        assert g.shape == c.shape
        d = np.abs(g - c)
        assert d.max() <= 1 and (d == 0).all(-1).mean() >= 0.999, (cmd, int(d.max()))
    # the blend-field dump (save_blend_png) is integer work: identical
    for exe, tag in ((CLI, "gpu"), (REF, "ref")):
        r = run("blend", *pairs[0][1], "--out", work / "p.png", "--dump-blend",
                work / ("bf_%s.png" % tag), exe=exe)
        assert r.returncode == 0
    assert np.array_equal(np.asarray(Image.open(work / "bf_gpu.png")),
                          np.asarray(Image.open(work / "bf_ref.png")))
