# Times the C2 bench under several builds: each argument is one EXTRA flag set
# ("" = default build); prints device ms/step and the kernels matching $KSEL.
# TOUCH = the sources the flags affect (default: all .cu)
KSEL=${KSEL:-smooth}
TOUCH=${TOUCH:-"*.cu"}
CFG=${CFG:-c2}
rebuild() {
  (cd paper_2006_01201_b200/csrc && touch $TOUCH)
  make -s -C paper_2006_01201_b200/csrc EXTRA="$1" > /dev/null 2>&1
}
for ex in "$@"; do
  rebuild "$ex"
  python bench.py --config $CFG --no-cpu-baseline --no-e2e --steps 30 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print(repr('$ex'), d['ms_per_step'], {n: (k[n]['ms_per_step'], k[n]['frac']) for n in k if any(s in n for s in '$KSEL'.split(','))})"
done
rebuild ""
