"""The checks build's own test (tools/checks.sh runs the GPU suite on a
-DFS_CHECKS library): an injected hand-off fault must be reported by the
device-side checks; without injection the counters stay at zero.  Skipped on
normal builds."""
import numpy as np
import pytest

import fs_synthetic as S

pytestmark = pytest.mark.gpu


def test_checks_report_injected_faults(fs):
    N = fs._native
    if not N.lib.fs_debug_checks_built():
        pytest.skip("normal build (tools/checks.sh builds with -DFS_CHECKS)")
    a = S.value_noise(200, 300, 3).astype(np.float32)
    L = fs.ImageBuf(a[:, :, None], np.ones(a.shape, np.uint8))
    R = fs.ImageBuf(np.roll(a, 3, axis=1)[:, :, None], np.ones(a.shape, np.uint8))
    plan_free = fs.FlowParams(levels=3)
    N.lib.fs_debug_check_failures(1)
    fs.bidirectional_flow(L, R, plan_free)
    assert N.lib.fs_debug_check_failures(1) == 0
    try:
        N.lib.fs_debug_inject(1)  # mis-stamped hand-offs: every consumer batch reports
        lay = S.small_panorama(seed=1)
        plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h,
                       fs.FlowParams(levels=lay.levels))
        plan.execute_host(lay.views, np.empty((lay.canvas_h, lay.canvas_w, 4), np.uint8))
        plan.close()
        assert N.lib.fs_debug_check_failures(1) > 0
    finally:
        N.lib.fs_debug_inject(0)
        N.lib.fs_debug_check_failures(1)
