python tools/profile_fold.py > gpurun_out/abl.json 2>&1; python - <<'PY'
import json,sys
d=json.load(open("gpurun_out/abl.json"))
print(round(d["total_ms"],3), {k: round(v["ms"],3) for k,v in d["kernels"].items()})
PY
