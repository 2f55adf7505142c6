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
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shard", choices=["none", "seams"], default="none",
                    help="seams: ONE panorama whose overlap pairs are sharded over the GPUs "
                         "(strong scaling, strips gathered to rank 0 over NCCL P2P); "
                         "none: one independent panorama per GPU (weak scaling)")
    ap.add_argument("--kernel-only", action="store_true",
                    help="only warmup + timed steps (for ncu launch lists)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_layout(name: str, seed: int):
    from paper_2006_01201_b200 import synthetic as S
    return {"c1": S.c1_pair, "c2": S.c2_panorama, "c3": S.c3_large_parallax,
            "c4": S.c4_ring}[name](seed=seed)


def workload_name(lay, name):
    return {"c1": "C1 (configs[0]) ", "c2": "C2 (configs[1]) ", "c3": "C3 (configs[2]) ",
            "c4": "C4 (configs[3]) "}[name] + lay.name


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


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


def cpu_reference_run(lay, threads: int):
    """One fold of `lay` through the compiled reference (oracle/_ref), metrics
    excluded (pipeline.cpp:150-204 minus :184-187, :194-199). Returns (s, stage s)."""
    import numpy as np
    from oracle import reference
    ref = reference()
    ref.set_threads(threads)
    fv = lay.float_views()
    timing = np.zeros(5, np.float64)
    t0 = time.perf_counter()
    ref.stitch_placed([d for d, _ in fv], [v for _, v in fv], lay.offsets, lay.canvas_w,
                      lay.canvas_h, (lay.levels, 8, 3, 1e-4, 2), timing=timing)
    return time.perf_counter() - t0, timing, ref.threads()


def run_reference_arm(args, ws, rank):
    """The reference's CPU fold (oracle/_ref, all host threads).  A step is
    one fold of a continuously running fold chain over the panorama's views
    (fold k = the reference's stitch of [panorama after fold k-1, view k],
    which is exactly fold k of stitch_placed); after the last fold the chain
    restarts from view 0.  value = canvas Mpx x (folds timed / folds per
    panorama) / time, i.e. panoramas per second in canvas Mpx."""
    if rank != 0:
        return
    import numpy as np
    from oracle import reference
    lay = make_layout(args.config, 0)
    threads = os.cpu_count() or 1
    ref = reference()
    ref.set_threads(threads)
    fv = lay.float_views()
    nfold = len(fv) - 1
    params = (lay.levels, 8, 3, 1e-4, 2)
    pano = None
    times = []
    for i in range(args.warmup + args.steps):
        k = i % nfold + 1
        if k == 1:
            d0, v0 = fv[0]
            pano = ref.place_on_canvas(d0, v0, lay.offsets[0][0], lay.offsets[0][1], lay.canvas_w,
                                       lay.canvas_h)
        t0 = time.perf_counter()
        pano = ref.stitch_placed([pano[0], fv[k][0]], [pano[1], fv[k][1]],
                                 [(0, 0), lay.offsets[k]], lay.canvas_w, lay.canvas_h, params)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    used = ref.threads()
    total = sum(times)
    s = total / len(times) * nfold  # seconds per panorama
    value = lay.canvas_mpx * (len(times) / nfold) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / len(times) * 1e3, 1), "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "config": {"workload": workload_name(lay, args.config), "canvas": [lay.canvas_w, lay.canvas_h],
                   "flow_params": [lay.levels, 8, 3, 1e-4, 2], "blend_params": [10.0, 0.05],
                   "parallelism": "host threads (reference parallel_rows)"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": used, "kind": "reference",
                         "sample": "one fold per step of a running %d-fold %s chain (%d folds "
                                   "timed), the reference compiled from /root/reference with its "
                                   "Release flags" % (nfold, args.config.upper(), len(times))},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0, "s_per_panorama": round(s, 3)},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference_arm(args, ws, rank)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2006_01201_b200 as fs

    sharded = args.shard == "seams"
    lay = make_layout(args.config, 0 if sharded else rank)
    params = fs.FlowParams(levels=lay.levels)
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, params, device=local)
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
    shard_mode = None
    if sp is not None:
        if ws > 1:
            shard_mode = sp.run()  # certified sharded, or unsharded on rank 0 from now on
        else:
            sp.execute(sptr)
            torch.cuda.synchronize()
            shard_mode = "sharded" if sp.status() == 0 else "unsharded"
            if shard_mode == "unsharded":
                sp.unsharded = True

    def run_step(host=False):
        if sp is not None and not sp.unsharded:
            if host:
                sp.execute(sptr, view_ptrs, host_out.data_ptr())
            else:
                sp.execute(sptr)
        elif sp is not None and rank != 0:
            return  # unsharded fallback: rank 0 folds the panorama alone
        elif host:
            plan.execute_ptrs(view_ptrs, host_out.data_ptr(), sptr)
        else:
            plan.execute(sptr)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def barrier():
        if ws > 1:
            dist.barrier()

    for _ in range(args.warmup):
        run_step()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = ClockSampler(local)
    with clocks:
        barrier()
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        for a, b in ev:
            flush.zero_()
            a.record(stream)
            run_step()
            b.record(stream)
        torch.cuda.synchronize()
        barrier()
        wall = time.perf_counter() - wall0
    if sp is not None and not sp.unsharded:
        if sp.status() != 0:
            raise RuntimeError("sharded execution not certified: " + fs._native.last_error())
    elif rank == 0 or sp is None:
        plan.check()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = statistics.mean(step_ms)
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
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

    # ---- end to end through the public call (host views in, host canvas out)
    e2e = None
    if not args.no_e2e:
        ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        barrier()
        for a, b in ee:
            a.record(stream)
            run_step(host=True)
            b.record(stream)
        torch.cuda.synchronize()
        e_ms = statistics.mean(a.elapsed_time(b) for a, b in ee)
        if ws > 1:
            t = torch.tensor([e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": round(units * lay.canvas_mpx / (e_ms / 1e3), 2), "unit": UNIT,
               "h2d_bytes_per_step": h2d_bytes * ws, "d2h_bytes_per_step": d2h_bytes * units,
               "s_per_panorama": round(e_ms / 1e3, 5), "ms_per_step": round(e_ms, 4)}

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
                     "GBps": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] else None}
                 for k, v in sorted(fam.items(), key=lambda kv: -kv[1]["ms"])}
    dom = max(fam, key=lambda k: fam[k]["ms"])
    lk = fam.get("lk_iter", fam[dom])
    ach = lk["bytes"] / lk["launches"] / (lk["ms"] / lk["launches"] * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get("lk_iter_dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"kernel": "k_lk_sweep<false> (LK later iteration, level 0, both directions)",
                "bound": "hbm",
                "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": round(lk["bytes"] / lk["launches"]),
                "avg_launch_us": round(lk["ms"] / lk["launches"] * 1e3, 2),
                "peak_source": peak_src, "share_of_step": round(lk["ms"] / kern_ms_total, 4),
                "dominant_kernel": dom, "kernels": breakdown,
                "profiled_step_ms": round(statistics.mean(tot_ms), 4)}

    # ---- CPU baseline: the compiled reference on this host (rank 0, N = 1)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            cs, stages, used = cpu_reference_run(lay, threads)
            cpu = {"value": round(lay.canvas_mpx / cs, 4), "unit": UNIT, "cores": used,
                   "kind": "reference",
                   "sample": "one full %s fold (%d folds, %.1f s), reference from "
                             "/root/reference built by oracle/Makefile, %d threads; stages "
                             "prep/flow/embed/blend_field/blend = %s s"
                             % (args.config.upper(), len(lay.views) - 1, cs, used,
                                [round(x, 2) for x in stages])}
        except Exception as e:  # checker missing: say so, never substitute
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": "unavailable: %s" % e}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None,
            "dtype": "f32/f64", "data": "synthetic",
            "config": {"workload": workload_name(lay, args.config),
                       "canvas": [lay.canvas_w, lay.canvas_h],
                       "views": [list(d) for d in lay.dims], "folds": len(lay.views) - 1,
                       "flow_params": list(params.astuple()), "blend_params": [10.0, 0.05],
                       "host_formats": host_formats,
                       "parallelism": ("seam-sharded over %d GPU(s): folds on ranks %s, "
                                       "stages %s, %d strip transfers (NCCL P2P), %s"
                                       % (ws, sp.schedule.fold_rank, sp.schedule.stage,
                                          len(sp.schedule.xfers), shard_mode)
                                       if sharded else
                                       "dp%d (one independent panorama per GPU)" % ws),
                       "l2": "inputs larger than L2 (views %d MB + canvas %d MB) and L2 "
                             "flushed (256 MB write) between timed steps"
                             % (h2d_bytes >> 20, (lay.canvas_w * lay.canvas_h * 21) >> 20),
                       "timing": "CUDA events per step on the launching stream, mean of %d, "
                                 "max over ranks" % args.steps,
                       "wall_s_timed_region": round(wall, 4)},
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu,
            "clocks": clocks.summary(), "gpu_launches": launches * args.steps,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
