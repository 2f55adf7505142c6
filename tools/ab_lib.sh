# A/B of two prebuilt libraries (build/ab/lib_A.so, build/ab/lib_B.so, e.g. HEAD
# and the working tree): flows bit-compared (tools/flow_bits.py), then device
# and e2e ms of each config ($CFGS, default c2), alternating A/B twice.
# Leaves lib_B.so installed.
L=paper_2006_01201_b200/libfs_b200.so
mkdir -p gpurun_out/ab
for v in ${VARS:-A B}; do
  cp build/ab/lib_$v.so $L
  python tools/flow_bits.py /tmp/flows_$v.npz > /dev/null 2>&1 || echo "flow dump $v failed"
done
python tools/flow_bits.py /tmp/flows_A.npz /tmp/flows_B.npz 2>&1 | tail -15
for rep in 1 2; do for v in ${VARS:-A B}; do
  cp build/ab/lib_$v.so $L
  for c in ${CFGS:-c2}; do
    python bench.py --config $c --no-cpu-baseline --no-c5 --steps 30 2>/dev/null | tail -1 > gpurun_out/ab/bench_${v}_${c}_$rep.json
    python - gpurun_out/ab/bench_${v}_${c}_$rep.json $v $c <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read())
k = d["roofline"]["kernels"]
fam = {n: round(k[n]["ms_per_step"], 4) for n in k if n.startswith("lk_")}
print(sys.argv[2], sys.argv[3], d["ms_per_step"], d["e2e"]["ms_per_step"], d["roofline"]["frac"], fam)
PY
  done
done; done
cp build/ab/lib_B.so $L
