import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2006_01201_b200 as fs
import fs_synthetic as S
lay = S.c2_panorama(0)
plan = fs.Plan(lay.dims, lay.offsets, lay.canvas_w, lay.canvas_h, fs.FlowParams(levels=lay.levels))
plan.execute_host(lay.views, None)
plan.set_host_format(3, 3)
hv = [torch.from_numpy(np.ascontiguousarray(v[..., :3])).pin_memory() for v in lay.views]
ho = torch.empty((lay.canvas_h, lay.canvas_w, 3), dtype=torch.uint8).pin_memory()
ptrs = [t.data_ptr() for t in hv]
for i in range(3): plan.execute_ptrs(ptrs, ho.data_ptr())
torch.cuda.synchronize()
ts = []
for i in range(10):
    t0 = time.perf_counter(); plan.execute_ptrs(ptrs, ho.data_ptr()); ts.append((time.perf_counter() - t0) * 1e3)
print("wall ms", [round(t, 3) for t in ts])
s = torch.cuda.Stream()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
for a, b in ev:
    a.record(s); plan.execute_ptrs_async(ptrs, ho.data_ptr(), s.cuda_stream); b.record(s)
torch.cuda.synchronize()
print("device async ms", [round(a.elapsed_time(b), 3) for a, b in ev])
plan.check()
