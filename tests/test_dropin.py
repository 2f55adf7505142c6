"""GPU: the reference's own acceptance suite (proj/tests/acceptance.cpp and
src/pipeline.cpp, UNCHANGED) linked against the C++ drop-in
(paper_2006_01201_b200/shim/libflowstitch_b200.so), i.e. the reference's 10
acceptance criteria evaluated on the B200 path."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2006_01201_b200", "shim", "acceptance_b200")


@pytest.mark.gpu
def test_reference_acceptance_suite_on_b200():
    if not os.path.exists(EXE):
        pytest.skip("acceptance_b200 not built (needs the reference headers at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 criterion failure(s)" in r.stdout


@pytest.mark.gpu
def test_dropin_check_against_reference_pipeline():
    exe = os.path.join(ROOT, "paper_2006_01201_b200", "shim", "dropin_check")
    if not os.path.exists(exe):
        pytest.skip("dropin_check not built (needs the reference headers at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 check failure(s)" in r.stdout


def test_dropin_library_exports_reference_api():
    lib = os.path.join(ROOT, "paper_2006_01201_b200", "shim", "libflowstitch_b200.so")
    if not os.path.exists(lib):
        pytest.skip("drop-in not built")
    out = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True,
                         text=True).stdout
    for sym in ["flowstitch::dense_pyr_lk(", "flowstitch::bidirectional_flow(",
                "flowstitch::compute_blend(", "flowstitch::distance_transform(",
                "flowstitch::blend_pair(", "flowstitch::crop_overlap(",
                "flowstitch::compute_partition(", "flowstitch::place_on_canvas(",
                "flowstitch::to_gray(", "flowstitch::build_pyramid(",
                "flowstitch::b200::stitch_placed(", "flowstitch::b200::misalignment_score(",
                "flowstitch::b200::estimate_translation("]:
        assert sym in out, sym
