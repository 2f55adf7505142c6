import json,sys
for l in sys.stdin:
    if not l.startswith("{"): print(l.rstrip()); continue
    d=json.loads(l); r=d.get("roofline") or {}
    e=d.get("e2e") or {}
    print("value", d["value"], "ms", d["ms_per_step"], "e2e", e.get("value"), e.get("ms_per_step"), "launches", d.get("gpu_launches"))
    if r:
        print("roofline", r["achieved"], r["frac"], r["avg_launch_us"], "profiled step", r["profiled_step_ms"])
        for k,v in r["kernels"].items(): print("  ", k, v)
    if d.get("cpu_baseline"): print("cpu", d["cpu_baseline"])
    print("clocks", d.get("clocks"))
