#!/bin/bash
# Round artefacts for profiles/<round>/ (run under gpurun):
#   bench lines (C2 with the CPU baseline + parity, C1/C3/C4), the ncu launch
#   list of the bench's timed steps, one ncu --set full capture of the LK
#   later iteration (C2 band, level 0) and the sweep's DRAM traffic.
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O/configs
python bench.py > $O/bench_c2.jsonl 2> $O/bench_c2.err
for c in c1 c3 c4; do python bench.py --config $c --no-cpu-baseline > $O/configs/bench_$c.jsonl 2>/dev/null; done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --kernel-only > $O/plain_kernel_only.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_bench.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --kernel-only > $O/ncu_launches.log 2>&1
python tools/lk_band.py > $O/plain_band.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k k_lk_sweep -s 22 -c 1 \
      -o $O/ncu_lk_iter_band python tools/lk_band.py > $O/ncu_full.log 2>&1
ls -la $O
