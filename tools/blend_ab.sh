for m in 12 14 16; do
  touch paper_2006_01201_b200/csrc/fs_kernels.cu
  make -s -C paper_2006_01201_b200/csrc EXTRA="-DBLEND_MINB=$m" > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_blend_area3 --csv --log-file gpurun_out/blend_$m.csv python bench.py --kernel-only --steps 2 --warmup 3 > /dev/null 2>&1
  python bench.py --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m', d['ms_per_step'], d['roofline']['kernels']['blend'])"
done
touch paper_2006_01201_b200/csrc/fs_kernels.cu; make -s -C paper_2006_01201_b200/csrc > /dev/null 2>&1
