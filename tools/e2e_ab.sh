# device + e2e ms of C2 and C4 under several builds of fs_plan.cu ($@ = EXTRA flag sets)
for ex in "$@"; do
  (cd paper_2006_01201_b200/csrc && touch fs_plan.cu)
  make -s -C paper_2006_01201_b200/csrc EXTRA="$ex" > /dev/null 2>&1
  for c in ${CFGS:-c2 c4}; do for i in 1 2; do
    python bench.py --config $c --no-cpu-baseline --no-c5 --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(repr('$ex'), '$c', d['ms_per_step'], d['e2e']['ms_per_step'])"
  done; done
done
(cd paper_2006_01201_b200/csrc && touch fs_plan.cu); make -s -C paper_2006_01201_b200/csrc > /dev/null 2>&1
