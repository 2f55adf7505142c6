# A/B timing of two builds: $1 = EXTRA flags for B (A = default)
for rep in 1 2; do
for v in A B; do
  touch paper_2006_01201_b200/csrc/fs_lk.cu
  if [ $v = A ]; then make -s -C paper_2006_01201_b200/csrc > /dev/null 2>&1; else make -s -C paper_2006_01201_b200/csrc EXTRA="$1" > /dev/null 2>&1; fi
  python bench.py --no-cpu-baseline --steps 30 > gpurun_out/ab_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/ab_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["e2e"]["ms_per_step"])')"
done; done
touch paper_2006_01201_b200/csrc/fs_lk.cu; make -s -C paper_2006_01201_b200/csrc > /dev/null 2>&1
