"""Seam-sharded fold: the schedule's segments and strip
exchanges, run for every rank in one process on one GPU (LocalShardGroup:
the exchange as device copies), must give rank 0 — the canvas GPU — the
unsharded plan's RGBA8 panorama bit for bit, or report that a blend tap left
the region its GPU holds final (FS_ERR_SHARD_REACH) and fall back."""
import numpy as np
import pytest

import fs_synthetic as S

pytestmark = pytest.mark.gpu


def _out_of(plan, lay):
    import torch

    class _Dev:
        __cuda_array_interface__ = {"shape": (lay.canvas_h, lay.canvas_w, 4), "typestr": "|u1",
                                    "version": 3, "data": (plan.output_buffer(), False),
                                    "strides": None}
    return torch.as_tensor(_Dev(), device="cuda").cpu().numpy()


def _unsharded(fs, lay, params):
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params, views_rgba=lay.views)
    out = np.empty((lay.canvas_h, lay.canvas_w, 4), np.uint8)
    plan.execute_host(lay.views, out)
    plan.close()
    return out


def _group(fs, lay, params, nranks, fold_rank=None):
    from paper_2006_01201_b200.shard import LocalShardGroup
    plans = [fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params,
                     views_rgba=lay.views) for _ in range(nranks)]
    return plans, LocalShardGroup(plans, fold_rank)


def _ring(seed=0, n=5):
    """C4 analogue: views side by side with 1/5 overlap."""
    return S.small_strip(seed=seed, n=n, vw=160, vh=120, step=128, parallax=3)


LAYOUTS = {
    "panorama": lambda: S.small_panorama(seed=5),   # C2 analogue: seams, then bands
    "ring": lambda: _ring(),
    "strip6": lambda: S.small_strip(seed=3, n=6, vw=150, vh=110, step=110, parallax=2),
}


@pytest.mark.parametrize("name", sorted(LAYOUTS))
@pytest.mark.parametrize("nranks", [1, 2, 3, 5])
def test_sharded_matches_unsharded(fs, name, nranks):
    import torch
    lay = LAYOUTS[name]()
    params = fs.FlowParams(levels=3)
    ref = _unsharded(fs, lay, params)
    plans, g = _group(fs, lay, params, nranks)
    for _ in range(2):  # capture, then replay
        g.execute()
        torch.cuda.synchronize()
        assert g.statuses() == [0] * nranks, g.statuses()
        assert np.array_equal(_out_of(plans[0], lay), ref)
    sched = g.schedule
    assert all(0 <= r < nranks for r in sched.fold_rank)
    if nranks > 1 and name == "panorama":
        # the bands read the seams' blended rows: a second stage
        assert max(sched.stage) >= 1
    for p in plans:
        p.close()


@pytest.mark.parametrize("fold_rank", [[0, 1, 0, 1, 0, 1], [0, 2, 1, 0, 2, 1], [0, 0, 0, 1, 1, 1],
                                       [0, 1, 1, 1, 1, 1]])
def test_sharded_explicit_assignment(fs, fold_rank):
    """Any assignment (including dependent folds on other ranks and rank 0
    computing nothing) gives the same panorama or a certified refusal."""
    import torch
    lay = S.small_panorama(seed=7)
    params = fs.FlowParams(levels=3)
    ref = _unsharded(fs, lay, params)
    nranks = max(fold_rank) + 1
    plans, g = _group(fs, lay, params, nranks, fold_rank)
    assert g.schedule.fold_rank == fold_rank
    how = g.run()
    assert how == "sharded"
    torch.cuda.synchronize()
    assert np.array_equal(_out_of(plans[0], lay), ref)
    for p in plans:
        p.close()


def _adjacent_boxes_layout(seed=11, shift=6):
    """Fold 2's Area3 box starts where fold 1's ends (the boxes touch but do
    not meet), with a parallax that moves fold 2's L taps across into fold
    1's box (one of the two shift signs does): on a rank without fold 1's
    strip that blend must be refused."""
    W, H = 300, 80
    scene = S.rgb_scene(H, W + 40, seed)
    rects = [(0, 100), (60, 140), (100, 200)]
    views, offs = [], []
    for k, (x, w) in enumerate(rects):
        c0 = 20 + x + shift * k
        views.append(S.rgba(scene[:, c0:c0 + w]))
        offs.append((x, 0))
    return S.Layout("adjacent", W, H, views, offs, 3)


def test_shard_reach_refused_then_unsharded(fs):
    import torch
    params = fs.FlowParams(levels=2, window_radius=4, iterations_per_level=2)
    refused = 0
    for shift in (6, -6):
        lay = _adjacent_boxes_layout(shift=shift)
        ref = _unsharded(fs, lay, params)
        plans, g = _group(fs, lay, params, 2, [0, 1, 0])
        b1, b2 = plans[0].fold_info(1)[0], plans[0].fold_info(2)[0]
        assert b1[0] + b1[2] == b2[0], (b1, b2)  # touching, not meeting: no static dependency
        assert g.schedule.stage == [0, 0, 0]
        g.execute()
        torch.cuda.synchronize()
        st = g.statuses()
        assert st[1] == 0 and st[0] in (0, fs._native.FS_ERR_SHARD_REACH), st
        refused += st[0] != 0
        assert g.run() == ("unsharded" if st[0] else "sharded")
        assert np.array_equal(_out_of(plans[0], lay), ref)
        # both folds on one rank: always certified
        plans2, g2 = _group(fs, lay, params, 2, [0, 0, 0])
        assert g2.run() == "sharded"
        assert np.array_equal(_out_of(plans2[0], lay), ref)
        for p in plans + plans2:
            p.close()
    assert refused >= 1  # fold 2 on rank 0 lacked fold 1's strip


@pytest.mark.parametrize("seed", [3, 6, 7, 8, 10, 11, 12, 14, 16, 17, 19, 20, 22, 23])
def test_sharded_random_layouts(fs, seed):
    """Random layouts (overlapping boxes, alpha holes): the protocol's result
    is always the unsharded panorama."""
    from test_gpu_parity import _random_layout
    lay = _random_layout(seed)
    if len(lay.views) < 3:
        pytest.skip("fewer than two folds")
    params = fs.FlowParams(levels=2, window_radius=4, iterations_per_level=2)
    ref = _unsharded(fs, lay, params)
    plans, g = _group(fs, lay, params, 3)
    g.run()
    assert np.array_equal(_out_of(plans[0], lay), ref)
    for p in plans:
        p.close()


@pytest.mark.parametrize("name", ["panorama", "ring"])
def test_sharded_host_io(fs, name):
    """One rank with host buffers: page-locked views/canvas are copied inside
    the segment graphs (views overlapping the folds), pageable ones around
    them; both give the unsharded panorama, and new pointers re-capture."""
    import torch
    from paper_2006_01201_b200.shard import ShardedPlan
    lay = LAYOUTS[name]()
    params = fs.FlowParams(levels=3)
    ref = _unsharded(fs, lay, params)
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params, views_rgba=lay.views)
    sp = ShardedPlan(plan, 1, 0)
    pin = [torch.from_numpy(v).pin_memory() for v in lay.views]
    out = torch.full((lay.canvas_h, lay.canvas_w, 4), 7, dtype=torch.uint8).pin_memory()
    for _ in range(2):
        out.fill_(7)
        assert sp.run([t.data_ptr() for t in pin], out.data_ptr()) == "sharded"
        assert np.array_equal(out.numpy(), ref)
    pin2 = [t.clone().pin_memory() for t in pin]
    out2 = torch.zeros_like(out).pin_memory()
    sp.execute(None, [t.data_ptr() for t in pin2], out2.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(out2.numpy(), ref)
    views = [np.ascontiguousarray(v) for v in lay.views]
    out3 = np.zeros_like(ref)
    sp.execute(None, [v.ctypes.data for v in views], out3.ctypes.data)
    torch.cuda.synchronize()
    assert sp.status() == 0
    assert np.array_equal(out3, ref)
    plan.close()


def test_sharded_host_io_rgb8(fs):
    """The seam-sharded execution with RGB8 host views and canvas."""
    import torch
    from paper_2006_01201_b200.shard import ShardedPlan
    lay = LAYOUTS["panorama"]()
    params = fs.FlowParams(levels=3)
    ref = _unsharded(fs, lay, params)
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params, views_rgba=lay.views)
    plan.set_host_format(3, 3)
    sp = ShardedPlan(plan, 1, 0)
    pin = [torch.from_numpy(np.ascontiguousarray(v[..., :3])).pin_memory() for v in lay.views]
    out = torch.full((lay.canvas_h, lay.canvas_w, 3), 7, dtype=torch.uint8).pin_memory()
    for _ in range(2):
        out.fill_(7)
        assert sp.run([t.data_ptr() for t in pin], out.data_ptr()) == "sharded"
        assert np.array_equal(out.numpy(), ref[..., :3])
    plan.close()
