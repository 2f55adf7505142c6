# A/B timing of two builds: $1 = EXTRA flags for B (A = default), $2 = config
# (default c2), TOUCH = sources the flag affects (default fs_lk.cu)
CFG=${2:-c2}
TOUCH=${TOUCH:-fs_lk.cu}
rebuild() {
  for f in $TOUCH; do touch paper_2006_01201_b200/csrc/$f; done
  make -s -C paper_2006_01201_b200/csrc EXTRA="$1" > /dev/null 2>&1
}
for rep in 1 2; do
for v in A B; do
  if [ $v = A ]; then rebuild ""; else rebuild "$1"; fi
  python bench.py --config $CFG --no-cpu-baseline --steps 30 > gpurun_out/ab_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/ab_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["e2e"]["ms_per_step"])')"
done; done
rebuild ""
