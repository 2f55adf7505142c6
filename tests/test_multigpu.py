"""CPU, world_size 2 over gloo: the multi-GPU host logic (set sharding, the
max-over-ranks timing reduction, gathering per-set results) gives the same
result as one process.  The per-set fold here is the CPU oracle on a small
panorama; on the GPU box the same driver runs the planned fold."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2006_01201_b200 import multigpu as M


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fold(seed):
    from oracle import restatement
    import fs_synthetic as S
    lay = S.small_strip(seed=seed, n=3, vw=48, vh=32, step=32, parallax=2)
    fv = lay.float_views()
    out, _ = restatement().stitch_placed([d for d, _ in fv], [v for _, v in fv], lay.offsets,
                                         lay.canvas_w, lay.canvas_h, (2, 4, 2, 1e-4, 1))
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = M.run_sets(5, _fold, world, rank)
        mx = M.max_over_ranks(1.5 + rank)
        tot = M.sum_over_ranks(len(M.shard(5, world, rank)))
        q.put((rank, res, mx, tot))
    finally:
        dist.destroy_process_group()


def test_shard_covers_every_set_once():
    for n in (1, 5, 20):
        for world in (1, 2, 3, 8):
            got = sorted(i for r in range(world) for i in M.shard(n, world, r))
            assert got == list(range(n))
    with pytest.raises(ValueError):
        M.shard(4, 2, 2)


def test_two_rank_gloo_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = {s: M.digest(_fold(s)) for s in range(5)}
    for rank, res, mx, tot in out:
        assert res == single
        assert mx == 2.5  # max over ranks of (1.5 + rank)
        assert tot == 5


def _bench(*args, timeout=600):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args], cwd=root,
                       env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    return [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]


@pytest.mark.parametrize("cfg,n", [("c2", 2), ("c4", 3)])
def test_bench_spawns_ranks_dry_run(cfg, n):
    """`bench.py --gpus N` without a launcher starts N ranks itself (torchrun on
    127.0.0.1); --dry-run exchanges the shard schedule's strips over gloo."""
    lines = _bench("--gpus", str(n), "--dry-run", "--config", cfg)
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == n and d["backend"] == "gloo" and d["status"] == 0
    assert set(d["fold_rank"]) == set(range(n))
    assert d["received_rank0"] == sorted(k for k in range(1, len(d["fold_rank"]))
                                         if d["fold_rank"][k] != 0)


def test_reference_arm_is_clean():
    """--impl reference imports neither torch nor the B200 package and times
    whole stitch_placed calls with the B200 arm's config dict."""
    from oracle import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import runpy, sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--config', "
            "'c1', '--steps', '1', '--warmup', '0']; runpy.run_path('bench.py', "
            "run_name='__main__'); print(json.dumps({'mods': sorted(m for m in sys.modules "
            "if m.split('.')[0] in ('torch', 'paper_2006_01201_b200'))}))")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    line, mods = lines[0], lines[1]["mods"]
    assert mods == []
    assert line["impl"] == "reference" and line["steps"] == 1
    assert line["config"]["workload"].startswith("C1") and line["config"]["folds"] == 1
    assert "whole C1 stitch_placed" in line["cpu_baseline"]["sample"]
