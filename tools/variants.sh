# Times the C2 bench under several builds: each argument is one EXTRA flag set
# ("" = default build); prints device ms/step and the kernels matching $KSEL.
KSEL=${KSEL:-smooth}
for ex in "$@"; do
  touch paper_2006_01201_b200/csrc/*.cu
  make -s -C paper_2006_01201_b200/csrc EXTRA="$ex" > /dev/null 2>&1
  python bench.py --no-cpu-baseline --no-e2e --steps 30 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print(repr('$ex'), d['ms_per_step'], {n: k[n]['ms_per_step'] for n in k if any(s in n for s in '$KSEL'.split(','))})"
done
touch paper_2006_01201_b200/csrc/*.cu; make -s -C paper_2006_01201_b200/csrc > /dev/null 2>&1
