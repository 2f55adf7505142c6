#!/usr/bin/env python
"""Per-rank work of the seam-sharded schedule, each rank's segments timed
ALONE on one GPU (CUDA events, views resident, strips as left in the
buffers): python tools/shard_projection.py [c2|c4] [N ...].  A projection of
the N-GPU critical path (sum over segments of the slowest rank + strip bytes
over NVLink), not a multi-GPU measurement."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_01201_b200 as fs  # noqa: E402
import fs_synthetic as S  # noqa: E402
from paper_2006_01201_b200.shard import ShardedPlan  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    ns = [int(v) for v in sys.argv[2:]] or [1, 2, 4, 8]
    lay = {"c2": S.c2_panorama, "c4": S.c4_ring}[cfg](0)
    plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h,
                   fs.FlowParams(levels=lay.levels), views_rgba=lay.views)
    s = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for n in ns:
        per_rank = []
        for r in range(n):
            sp = ShardedPlan(plan, n, r)
            for _ in range(2):
                for seg in range(sp.n_segments):
                    sp.execute_segment(seg)
            torch.cuda.synchronize()
            segs = []
            for seg in range(sp.n_segments):
                t = []
                for _ in range(5):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(s)
                    sp.execute_segment(seg)
                    b.record(s)
                    torch.cuda.synchronize()
                    t.append(a.elapsed_time(b))
                segs.append(round(statistics.median(t), 4))
            per_rank.append(segs)
        sched = sp.schedule
        strip_bytes = {}
        for x in sched.xfers:
            bx = plan.fold_info(x.fold)[0]
            strip_bytes.setdefault(x.stage, []).append((x.src, x.dst, bx[2] * bx[3] * 16))
        nseg = sched.n_segments
        crit = 0.0
        for seg in range(nseg):
            crit += max(pr[seg] for pr in per_rank)
            # NVLink 5: ~750 GB/s achievable per direction per GPU; rank 0 receives most
            rx = {}
            for src, dst, nb in strip_bytes.get(seg, []):
                rx[dst] = rx.get(dst, 0) + nb
            crit += max(rx.values(), default=0) / 750e9 * 1e3
        res[n] = {"fold_rank": sched.fold_rank, "stage": sched.stage,
                  "segment_ms_per_rank": per_rank, "projected_ms": round(crit, 4),
                  "projected_Mpx_s": round(lay.canvas_mpx / crit * 1e3, 1)}
    print(json.dumps({"config": cfg, "canvas_mpx": lay.canvas_mpx, "ranks": res}, indent=1))


if __name__ == "__main__":
    main()
