"""CPU, world_size 2-3 over gloo: the seam-sharded execution's host protocol
(ShardedPlan.execute: segments, strip exchanges in the schedule's global
order, the max-status reduction that triggers the unsharded fallback).  The
schedule is the library's (fs_shard_schedule, host-only); the segments are
stand-ins that check every strip a rank composes has arrived and fill the
rank's own strips — the device side is covered by tests/test_gpu_shard.py."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2006_01201_b200 import shard as SH

C2_BOXES = [(0, 0, 0, 0), (2083, 600, 667, 2800), (4166, 600, 584, 2800), (6250, 600, 500, 2800),
            (0, 600, 9000, 400), (0, 3000, 9000, 400)]
C4_BOXES = [(0, 0, 0, 0)] + [(2048 * k, 1024, 512, 6144) for k in range(1, 8)]


def _meets(a, b):
    return (min(a[0] + a[2], b[0] + b[2]) > max(a[0], b[0]) and
            min(a[1] + a[3], b[1] + b[3]) > max(a[1], b[1]))


def _needed(boxes, fold_rank, nranks):
    """Independent restatement: the strips rank r composes."""
    n = len(boxes)
    need = [set() for _ in range(nranks)]
    for r in range(nranks):
        for k in range(1, n):
            if fold_rank[k] == r:
                continue
            if r == 0 or any(fold_rank[j] == r and _meets(boxes[k], boxes[j])
                             for j in range(k + 1, n)):
                need[r].add(k)
        grew = True
        while grew:
            grew = False
            for j in sorted(need[r]):
                for m in range(1, j):
                    if fold_rank[m] != r and m not in need[r] and _meets(boxes[m], boxes[j]):
                        need[r].add(m)
                        grew = True
    return need


@pytest.mark.parametrize("boxes", [C2_BOXES, C4_BOXES], ids=["c2", "c4"])
@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8])
def test_schedule_properties(boxes, nranks):
    sc = SH.shard_schedule(boxes, nranks)
    n = len(boxes)
    assert sc.fold_rank[0] == 0 and all(0 <= r < nranks for r in sc.fold_rank)
    need = _needed(boxes, sc.fold_rank, nranks)
    got = [set() for _ in range(nranks)]
    for x in sc.xfers:
        assert x.src == sc.fold_rank[x.fold] != x.dst
        assert x.stage == sc.stage[x.fold]
        got[x.dst].add(x.fold)
    assert got == need
    for k in range(1, n):  # a fold runs after every strip its crop needs
        for m in range(1, k):
            if _meets(boxes[m], boxes[k]):
                assert sc.stage[k] >= sc.stage[m] + (sc.fold_rank[m] != sc.fold_rank[k])
    assert sc.n_segments == max(sc.stage) + 2
    if boxes is C4_BOXES:  # independent seams: one stage, one fold per GPU when there are enough
        assert max(sc.stage) == 0
        if nranks >= 8:
            assert sorted(sc.fold_rank[1:]) == list(range(1, 8))


def test_schedule_explicit_and_errors():
    sc = SH.shard_schedule(C2_BOXES, 2, [0, 1, 1, 1, 0, 0])
    assert sc.fold_rank == [0, 1, 1, 1, 0, 0] and sc.stage == [0, 0, 0, 0, 1, 1]
    with pytest.raises(Exception):
        SH.shard_schedule(C2_BOXES, 2, [0, 2, 0, 0, 0, 0])
    with pytest.raises(Exception):
        SH.shard_schedule(C2_BOXES, 0)


class _FakeShard(SH.ShardedPlan):
    """ShardedPlan's execute loop over host tensors: a segment checks the
    strips it composes and writes its own folds' strips."""

    def __init__(self, boxes, nranks, rank, fold_rank, transport):
        self.nranks, self.rank, self.transport = nranks, rank, transport
        self.schedule = SH.shard_schedule(boxes, nranks, fold_rank)
        self.n_segments = self.schedule.n_segments
        self.need = _needed(boxes, self.schedule.fold_rank, nranks)[rank]
        self._strips = {k: torch.zeros(8, dtype=torch.int64) for k in range(1, len(boxes))}
        self.composed, self.errors = [], []

    def strip(self, fold):
        return self._strips[fold]

    def execute_segment(self, segment, stream=None, view_ptrs=None, out_ptr=None):
        sc = self.schedule
        for m in sorted(self.need):
            if sc.stage[m] + 1 == segment:
                if not bool((self._strips[m] == 1000 + m).all()):
                    self.errors.append("strip %d missing at segment %d" % (m, segment))
                self.composed.append(m)
        for k in range(1, len(sc.stage)):
            if sc.fold_rank[k] == self.rank and sc.stage[k] == segment:
                self._strips[k].fill_(1000 + k)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = SH.TorchDistTransport()
        out = []
        for boxes, fr in ((C2_BOXES, None), (C4_BOXES, None),
                          (C2_BOXES, [0] + [(k * 7) % world for k in range(1, 6)])):
            f = _FakeShard(boxes, world, rank, fr, tr)
            f.execute(stream=0)
            out.append((sorted(f.composed), sorted(f.need), f.errors))
        st = tr.max_status(9 if rank == world - 1 else 0)
        q.put((rank, out, st))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_strip_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out, st in res:
        assert st == 9  # one rank's refusal reaches every rank
        for composed, need, errors in out:
            assert errors == []
            assert composed == need


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p
