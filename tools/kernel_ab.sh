# A/B of one kernel family: $1 = git stash-free variant flag (EXTRA for B), $2 = ncu kernel regex
# prints device ms (bench) and the kernel family's profiled ms for A (default) and B
for v in A B; do
  touch paper_2006_01201_b200/csrc/*.cu
  if [ $v = A ]; then make -s -C paper_2006_01201_b200/csrc > /dev/null 2>&1; else make -s -C paper_2006_01201_b200/csrc EXTRA="$1" > /dev/null 2>&1; fi
  python bench.py --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print('$v', d['ms_per_step'], {n: k[n]['ms_per_step'] for n in k if '$2' in n})"
done
touch paper_2006_01201_b200/csrc/*.cu; make -s -C paper_2006_01201_b200/csrc > /dev/null 2>&1
