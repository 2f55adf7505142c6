#!/usr/bin/env python
"""Benchmark of the B200 flow+blend path (BASELINE.json metric).

A step is one complete flow+blend fold of a synthetic 9000x4000 panorama
(configs[1], "C2": 4 horizontal 2750x2800 views + top/bottom 9000x1000 bands,
5 folds): per fold partition, crop+gray, Gaussian pyramid, bidirectional
pyramidal LK, exact distance transforms + Eq. 1, Code 1 blend, composition;
then 8-bit quantisation of the canvas.  One process per GPU (torchrun for
N > 1); each rank folds its own panorama (independent seeds, no data-path
collective; weak scaling).

  value   = whole-job output-canvas Mpx / device time per step (views already
            in HBM, one CUDA-graph replay per step, L2 flushed between steps)
  e2e     = same metric through the public end-to-end call
            (fs_plan_execute_host: pinned host RGBA8 views -> H2D -> fold ->
            D2H of the RGBA8 canvas), CUDA events around each call
  roofline: dominant kernel (LK iteration), algorithmic bytes / event-timed
            duration on its launching stream, against MEASURED_PEAKS.json
  cpu_baseline: the reference compiled from /root/reference (oracle/_ref),
            same workload, all host threads, rank 0 at N = 1

`--impl reference` times the reference's own CPU implementation instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("flow+blend Mpx/s per B200 and end-to-end s per 9000×4000 panorama, "
          "1/2/4/8 GPU")
UNIT = "Mpx/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=["c2", "c1", "c3", "c4"], default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c5", action="store_true",
                    help="skip the configs[4] throughput leg (20 C2 sets, two in flight)")
    ap.add_argument("--tile-len", type=int, default=0,
                    help="row/column flow tiles of about this length along each fold's long "
                         "axis (fs_plan_set_tiling; 0: untiled)")
    ap.add_argument("--shard", choices=["auto", "none", "seams"], default="auto",
                    help="seams: ONE panorama whose overlap pairs are sharded over the GPUs "
                         "(strong scaling, strips gathered to rank 0 over NCCL P2P); "
                         "none: one independent panorama per GPU (weak scaling); "
                         "auto: seams when N > 1 (with the independent-panorama throughput "
                         "as the secondary `dp` key)")
    ap.add_argument("--kernel-only", action="store_true",
                    help="only warmup + timed steps (for ncu launch lists)")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: start the ranks over gloo, run the shard schedule and the "
                         "strip-exchange protocol with host stand-ins, print one JSON line")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def maybe_spawn(args) -> bool:
    """`python bench.py --gpus N` (N > 1) without a launcher: start the N
    ranks ourselves (torchrun on 127.0.0.1, one process per GPU) and wait.
    Returns True when this process was only the launcher."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # NVLS / P2P transport lines in the log
    rc = subprocess.call(cmd, env=env)
    if rc:
        sys.exit(rc)
    return True


def make_layout(name: str, seed: int):
    import fs_synthetic as S  # numpy only: no torch, no product library
    return {"c1": S.c1_pair, "c2": S.c2_panorama, "c3": S.c3_large_parallax,
            "c4": S.c4_ring}[name](seed=seed)


def workload_name(lay, name):
    return {"c1": "C1 (configs[0]) ", "c2": "C2 (configs[1]) ", "c3": "C3 (configs[2]) ",
            "c4": "C4 (configs[3]) "}[name] + lay.name


def shard_mode(args, ws) -> str:
    if args.shard == "auto":
        return "seams" if ws > 1 else "none"
    return args.shard


def config_dict(args, lay, ws) -> dict:
    """The workload; identical in the B200 and the reference arm's lines."""
    mode = shard_mode(args, ws)
    if ws == 1:
        par = "dp1 (one panorama on one GPU)"
    elif mode == "seams":
        par = ("seam-sharded over %d GPUs: overlap pairs (folds) scheduled over the ranks, "
               "Area3 strips gathered to rank 0 over NCCL P2P" % ws)
    else:
        par = "dp%d (one independent panorama per GPU)" % ws
    return {"workload": workload_name(lay, args.config),
            "canvas": [lay.canvas_w, lay.canvas_h],
            "views": [list(d) for d in lay.dims], "folds": len(lay.views) - 1,
            "flow_params": [lay.levels, 8, 3, 1e-4, 2], "blend_params": [10.0, 0.05],
            "parallelism": par,
            "l2": "inputs larger than L2 (views + canvas > 126 MB) and L2 flushed (256 MB "
                  "write) between timed GPU steps"}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons every ~10 ms."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.samples = []
        self.reasons = 0
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reasons |= int(r)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        busy = [s for s in self.samples if s > 600] or self.samples
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": self.max_mhz,
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b],
                "samples": len(self.samples)}


def _ref_fold(ref, lay, flows=False):
    """One whole stitch_placed of `lay` through the compiled reference
    (oracle/_ref): the fold of proj/src/pipeline.cpp:150-204 minus the seam
    metrics (:184-187, :194-199, which never write the panorama).  Returns
    (pano, valid, per-fold flows or [], seconds of the fold on the host)."""
    fv = lay.float_views()
    return ref.stitch_placed_flows([d for d, _ in fv], [v for _, v in fv], lay.offsets,
                                   lay.canvas_w, lay.canvas_h, (lay.levels, 8, 3, 1e-4, 2),
                                   flows=flows)


def cpu_baseline_leg(lay, config_name):
    """The reference on this host, rank 0 at N = 1: the same whole-panorama
    span as the GPU step, all host threads, best of 3; a
    1-thread sample (fold 1 alone, FLOWSTITCH_THREADS=1 semantics,
    src/parallel.cpp:14-20); returns (cpu_baseline dict, (pano, valid, folds))."""
    from oracle import reference
    ref = reference()
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    runs = []
    keep = None
    for i in range(3):
        pano, valid, folds, secs = _ref_fold(ref, lay, flows=(i == 0))
        runs.append(secs)
        if i == 0:
            keep = (pano, valid, folds)
    used = ref.threads()
    best = min(runs)
    # 1-thread sample: fold 1 (views 0 and 1 alone) at 1 and at all threads
    import fs_synthetic as S
    pair = S.Layout(lay.name + " fold 1", lay.canvas_w, lay.canvas_h, lay.views[:2],
                    lay.offsets[:2], lay.levels)
    _, _, _, f1_all = _ref_fold(ref, pair)
    ref.set_threads(1)
    _, _, _, f1_one = _ref_fold(ref, pair)
    ref.set_threads(threads)
    cpu = {"value": round(lay.canvas_mpx / best, 4), "unit": UNIT, "cores": used,
           "kind": "reference",
           "sample": "whole %s stitch_placed (%d folds) through oracle/_ref (the reference "
                     "compiled from /root/reference with its Release flags), %d threads, best "
                     "of 3: %s s" % (config_name.upper(), len(lay.views) - 1, used,
                                     [round(x, 2) for x in runs]),
           "s_per_panorama": round(best, 3), "cpu_model": cpu_model(),
           "threads1": {"sample": "fold 1 alone (views 0+1 on the full canvas)",
                        "s_1_thread": round(f1_one, 3), "s_all_threads": round(f1_all, 3),
                        "speedup_all_threads": round(f1_one / f1_all, 2),
                        "est_s_per_panorama_1_thread": round(best * f1_one / f1_all, 2)}}
    return cpu, keep


def run_reference_arm(args, ws, rank):
    """`--impl reference`: the reference's CPU implementation of the path
    (oracle/_ref, all host threads) on the same workload.  A step is one
    whole stitch_placed of the panorama's placed views — the span of the
    GPU arm's step and of its cpu_baseline.  Rank 0 alone runs it; nothing
    here imports torch or the B200 library."""
    if rank != 0:
        return
    from oracle import reference
    lay = make_layout(args.config, 0)
    threads = os.cpu_count() or 1
    ref = reference()
    ref.set_threads(threads)
    times = []
    for i in range(args.warmup + args.steps):
        _, _, _, secs = _ref_fold(ref, lay)
        if i >= args.warmup:
            times.append(secs)
    used = ref.threads()
    s = statistics.mean(times)  # seconds per panorama
    value = lay.canvas_mpx / s
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(s * 1e3, 1), "higher_is_better": True,
        "scaling": "strong" if shard_mode(args, ws) == "seams" else "weak",
        "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "config": config_dict(args, lay, ws),
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": used,
                         "kind": "reference", "cpu_model": cpu_model(),
                         "sample": "one whole %s stitch_placed per step (%d folds), %d steps, "
                                   "the reference compiled from /root/reference with its "
                                   "Release flags (oracle/_ref), %d threads"
                                   % (args.config.upper(), len(lay.views) - 1, len(times),
                                      used)},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0, "s_per_panorama": round(s, 3)},
    }
    print(json.dumps(line), flush=True)


def run_dry(args, ws, rank):
    """`--dry-run` (CPU): the N-rank launch, the gloo process group, the shard
    schedule of the config's folds and one strip exchange with host tensors
    in the schedule's order (paper_2006_01201_b200.shard's protocol)."""
    import torch
    import torch.distributed as dist
    if ws > 1:
        dist.init_process_group("gloo")
    from paper_2006_01201_b200 import shard as SH
    lay_boxes = {"c2": [(0, 0, 0, 0), (2083, 600, 667, 2800), (4166, 600, 584, 2800),
                        (6250, 600, 500, 2800), (0, 600, 9000, 400), (0, 3000, 9000, 400)],
                 "c4": [(0, 0, 0, 0)] + [(2048 * k, 1024, 512, 6144) for k in range(1, 8)],
                 "c1": [(0, 0, 0, 0), (512, 0, 512, 1024)],
                 "c3": [(0, 0, 0, 0), (1024, 0, 1024, 1024)]}[args.config]
    sc = SH.shard_schedule(lay_boxes, ws)
    strips = {k: torch.full((16,), k if sc.fold_rank[k] == rank else -1, dtype=torch.int64)
              for k in range(1, len(lay_boxes))}
    got = []
    if ws > 1:
        tr = SH.TorchDistTransport()
        for seg in range(sc.n_segments):
            xs = sc.xfers_after(seg, rank)
            tr.exchange(rank, xs, lambda k: strips[k])
            got += [x.fold for x in xs if x.dst == rank]
        ok = all(int(strips[k][0]) == k for k in got)
        status = tr.max_status(0 if ok else 1)
    else:
        status = 0
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": ws, "backend": "gloo" if ws > 1 else None,
                          "config": args.config, "fold_rank": sc.fold_rank, "stage": sc.stage,
                          "segments": sc.n_segments, "xfers": len(sc.xfers),
                          "received_rank0": sorted(got), "status": status}), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    if status:
        sys.exit(1)


def c5_leg(fs, torch, plan, lay, params, host_views, host_out, rgb_in, rgb_out, sets=20):
    """BASELINE configs[4] on one GPU: 20 C2 panorama sets back to back, two
    in flight (two plans on two streams, so one set's band folds overlap the
    next set's seam folds).  Device-resident and end to end (pinned host views
    in, pinned canvas out: fs_plan_execute_host_async).  The second plan holds
    a second synthetic scene (seed 1) of the same geometry; the sets alternate
    between the two (the fold's work depends on the geometry only)."""
    import numpy as np
    lay2 = make_layout("c2", 1)
    plan2 = fs.Plan(lay2.dims, lay2.offsets, lay2.canvas_w, lay2.canvas_h, params)
    plan2.set_host_format(3 if rgb_in else 4, 3 if rgb_out else 4)
    hv2 = [torch.from_numpy(np.ascontiguousarray(v[..., :3]) if rgb_in else v).pin_memory()
           for v in lay2.views]
    ho2 = torch.empty_like(host_out).pin_memory()
    plans = [(plan, [t.data_ptr() for t in host_views], host_out.data_ptr()),
             (plan2, [t.data_ptr() for t in hv2], ho2.data_ptr())]
    plan2.execute_ptrs(plans[1][1], plans[1][2])  # uploads, validates plan 2
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]

    def run(host):
        for i in range(2):  # warm-up: one set per plan
            p, vp, op = plans[i]
            (p.execute_ptrs_async(vp, op, streams[i].cuda_stream) if host
             else p.execute(streams[i].cuda_stream))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(streams[0])
        streams[1].wait_event(a)
        for k in range(sets):
            p, vp, op = plans[k % 2]
            st = streams[k % 2].cuda_stream
            p.execute_ptrs_async(vp, op, st) if host else p.execute(st)
        e1 = torch.cuda.Event()
        e1.record(streams[1])
        streams[0].wait_event(e1)
        b.record(streams[0])
        torch.cuda.synchronize()
        for p, _, _ in plans:
            p.check()
        return a.elapsed_time(b)

    dev_ms = run(False)
    e2e_ms = run(True)
    plan2.close()
    mpx = sets * lay.canvas_mpx
    return {"what": "BASELINE configs[4]: %d C2 9000x4000 sets back to back on one GPU, two in "
                    "flight (two plans, two streams); sets alternate between two synthetic scenes "
                    "(seeds 0, 1) of the same geometry" % sets,
            "value": round(mpx / (dev_ms / 1e3), 2), "unit": UNIT,
            "ms_per_set": round(dev_ms / sets, 4),
            "e2e": {"value": round(mpx / (e2e_ms / 1e3), 2), "unit": UNIT,
                    "ms_per_set": round(e2e_ms / sets, 4),
                    "what": "pinned host views in / canvas out per set, inside the timing"}}


def main():
    args = parse_args()
    if maybe_spawn(args):
        return
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference_arm(args, ws, rank)
        return
    if args.dry_run:
        run_dry(args, ws, rank)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2006_01201_b200 as fs

    sharded = shard_mode(args, ws) == "seams"
    lay = make_layout(args.config, 0 if sharded else rank)
    params = fs.FlowParams(levels=lay.levels)
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params, device=local)
    if args.tile_len:
        plan.set_tiling(args.tile_len)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    sp = None
    if sharded:
        from paper_2006_01201_b200.shard import ShardedPlan, TorchDistTransport
        if ws > 1:
            dist.barrier()  # communicator up before the first point-to-point batch
        sp = ShardedPlan(plan, ws, rank, transport=TorchDistTransport() if ws > 1 else None)

    # pinned host views + output canvas (the end-to-end call's buffers)
    # host formats: RGB8 views when every pixel is valid (alpha implicit),
    # an RGB8 canvas when the views cover all of it (nothing for alpha to say)
    rgb_in = all(bool((v[..., 3] == 255).all()) for v in lay.views)
    covered = np.zeros((lay.canvas_h, lay.canvas_w), bool)
    for v, (x, y) in zip(lay.views, lay.offsets):
        covered[y:y + v.shape[0], x:x + v.shape[1]] |= v[..., 3] >= 128
    rgb_out = rgb_in and bool(covered.all())
    plan.set_host_format(3 if rgb_in else 4, 3 if rgb_out else 4)
    host_views = [torch.from_numpy(np.ascontiguousarray(v[..., :3]) if rgb_in else v).pin_memory()
                  for v in lay.views]
    host_out = torch.empty((lay.canvas_h, lay.canvas_w, 3 if rgb_out else 4),
                           dtype=torch.uint8).pin_memory()
    view_ptrs = [t.data_ptr() for t in host_views]
    h2d_bytes, d2h_bytes = plan.transfer_bytes()  # page-locked path: what crosses PCIe
    host_formats = "views %s, canvas %s" % ("RGB8 (every pixel valid)" if rgb_in else "RGBA8",
                                            "RGB8 (covered by the views)" if rgb_out else "RGBA8")
    # first execution: uploads the views, validates the plan's EDT domains
    plan.execute_ptrs(view_ptrs, host_out.data_ptr(), sptr)
    smode = None
    if sp is not None:
        if ws > 1:
            smode = sp.run()  # certified sharded, or unsharded on rank 0 from now on
        else:
            sp.execute(sptr)
            torch.cuda.synchronize()
            smode = "sharded" if sp.status() == 0 else "unsharded"
            if smode == "unsharded":
                sp.unsharded = True

    def run_step(host=False, dp=False):
        if dp or sp is None:
            if host:
                plan.execute_ptrs(view_ptrs, host_out.data_ptr(), sptr)
            else:
                plan.execute(sptr)
        elif not sp.unsharded:
            if host:
                sp.execute(sptr, view_ptrs, host_out.data_ptr())
            else:
                sp.execute(sptr)
        elif rank == 0:  # unsharded fallback: rank 0 folds the panorama alone
            if host:
                plan.execute_ptrs(view_ptrs, host_out.data_ptr(), sptr)
            else:
                plan.execute(sptr)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def barrier():
        if ws > 1:
            dist.barrier()

    def max_over_ranks(v):
        if ws > 1:
            t = torch.tensor([v], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return v

    def timed(steps, host=False, dp=False, flush_l2=True):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for a, b in ev:
            if flush_l2:
                flush.zero_()
            a.record(stream)
            run_step(host=host, dp=dp)
            b.record(stream)
        torch.cuda.synchronize()
        barrier()
        wall = time.perf_counter() - w0
        return max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in ev)), wall

    for _ in range(args.warmup):
        run_step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    with clocks:
        ms, wall = timed(args.steps)
    if sp is not None and not sp.unsharded:
        if sp.status() != 0:
            raise RuntimeError("sharded execution not certified: " + fs._native.last_error())
    elif rank == 0 or sp is None:
        plan.check()
    units = 1 if sharded else ws  # panoramas per step over the job
    value = units * lay.canvas_mpx / (ms / 1e3)
    launches = plan.launch_count
    if sp is not None and not sp.unsharded:
        launches = sp.launch_count

    if args.kernel_only:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": round(value, 2), "unit": UNIT,
                              "ms_per_step": round(ms, 4), "kernel_only": True}), flush=True)
        plan.close()
        if ws > 1:
            dist.destroy_process_group()
        return

    # ---- secondary at N > 1 with sharding: independent panoramas per GPU
    dp = None
    if sharded and ws > 1:
        for _ in range(args.warmup):
            run_step(dp=True)
        dms, _ = timed(args.steps, dp=True)
        dp = {"value": round(ws * lay.canvas_mpx / (dms / 1e3), 2), "unit": UNIT,
              "ms_per_step": round(dms, 4), "scaling": "weak",
              "what": "every GPU folds its own panorama (BASELINE configs[4]-style "
                      "throughput), no data-path collective"}

    # ---- end to end through the public call (host views in, host canvas out)
    e2e = None
    if not args.no_e2e:
        for _ in range(2):
            run_step(host=True)
        e_ms, _ = timed(args.steps, host=True, flush_l2=False)
        e2e = {"value": round(units * lay.canvas_mpx / (e_ms / 1e3), 2), "unit": UNIT,
               "h2d_bytes_per_step": h2d_bytes * ws, "d2h_bytes_per_step": d2h_bytes * units,
               "s_per_panorama": round(e_ms / 1e3, 5), "ms_per_step": round(e_ms, 4)}

    # ---- configs[4] throughput (20 sets, two in flight), rank 0 at N = 1
    c5 = None
    if ws == 1 and args.config == "c2" and not args.no_c5 and not args.no_e2e:
        c5 = c5_leg(fs, torch, plan, lay, params, host_views, host_out, rgb_in, rgb_out)

    # ---- per-kernel roofline: event-timed launches on the launching stream
    fam = {}
    tot_ms = []
    for _ in range(max(3, min(args.steps, 10))):
        flush.zero_()
        st, tot = plan.profile(sptr)
        tot_ms.append(tot)
        for k, v in st.items():
            f = fam.setdefault(k, {"launches": 0, "ms": 0.0, "bytes": 0.0})
            for q in ("launches", "ms", "bytes"):
                f[q] += v[q]
    nrep = len(tot_ms)
    peak, peak_src = measured_peak_hbm()
    kern_ms_total = sum(v["ms"] for v in fam.values())
    breakdown = {k: {"launches_per_step": v["launches"] // nrep,
                     "ms_per_step": round(v["ms"] / nrep, 4),
                     "share": round(v["ms"] / kern_ms_total, 4),
                     "GBps": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] else None,
                     "frac": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9 / peak, 4)
                     if v["ms"] else None}
                 for k, v in sorted(fam.items(), key=lambda kv: -kv[1]["ms"])}
    dom = max(fam, key=lambda k: fam[k]["ms"])
    lk = fam.get("lk_iter", fam[dom])
    per_launch = lk["bytes"] / lk["launches"]
    ach = per_launch / (lk["ms"] / lk["launches"] * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get("lk_iter_dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"kernel": "k_lk_sweep (LK later iteration, level 0, both directions)",
                "bound": "hbm",
                "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic,
                "bytes_basis": "SURVEY.md §8(d) K3: 26 B per px, direction and iteration",
                "algorithmic_bytes_per_launch": round(per_launch),
                "avg_launch_us": round(lk["ms"] / lk["launches"] * 1e3, 2),
                "peak_source": peak_src, "share_of_step": round(lk["ms"] / kern_ms_total, 4),
                "dominant_kernel": dom, "kernels": breakdown,
                "step_bytes_frac": round(sum(v["bytes"] for v in fam.values()) / nrep
                                         / (statistics.mean(tot_ms) * 1e-3) / 1e9 / peak, 4),
                "profiled_step_ms": round(statistics.mean(tot_ms), 4)}

    # ---- CPU baseline (the compiled reference on this host, rank 0, N = 1)
    # and parity of this run's output against it
    cpu = None
    parity = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cpu, (rp, rv, rfolds) = cpu_baseline_leg(lay, args.config)
        except Exception as e:  # checker missing: say so, never substitute
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": "unavailable: %s" % e}
            rp = None
        if rp is not None and not args.no_parity:
            from oracle import parity as P
            if not args.no_e2e:
                gpu_canvas = host_out.numpy()
            else:
                gpu_canvas = np.empty((lay.canvas_h, lay.canvas_w, 4), np.uint8)
                plan.set_host_format(4, 4)
                plan.execute_host(lay.views, gpu_canvas)
            canvas = P.compare_canvas(gpu_canvas, rp, rv)
            flow = P.fold_flow_stats(plan, rfolds)
            parity = {"vs": "oracle/_ref (the reference compiled from /root/reference), same "
                            "inputs, this run's output",
                      "max_lsb": canvas["max_lsb"], "frac_le_1lsb": canvas["frac_le_1lsb"],
                      "frac_exact": canvas["frac_exact"], "valid_equal": canvas["valid_equal"],
                      "flow_mean_epe": flow["mean_epe"], "flow_max_epe": flow["max_epe"],
                      "flow_frac_gt_0p5": flow["frac_gt_0p5"],
                      "flow_valid_mismatch": flow["valid_mismatch"], "flow_px": flow["n"],
                      "gates": P.gates(canvas, flow)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None,
            "dtype": "f32/f64", "data": "synthetic",
            "config": config_dict(args, lay, ws),
            "details": {"host_formats": host_formats,
                        "timing": "CUDA events per step on the launching stream, mean of %d, "
                                  "max over ranks" % args.steps,
                        "wall_s_timed_region": round(wall, 4),
                        "shard": ({"fold_rank": sp.schedule.fold_rank,
                                   "stage": sp.schedule.stage,
                                   "strip_transfers": len(sp.schedule.xfers), "mode": smode}
                                  if sp is not None else None)},
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "parity": parity,
            "dp": dp, "c5": c5, "clocks": clocks.summary(), "gpu_launches": launches * args.steps,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
