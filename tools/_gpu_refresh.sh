mkdir -p gpurun_out/r01b
python bench.py > gpurun_out/r01b/bench_c2.jsonl 2> gpurun_out/r01b/bench_c2.err
for c in c1 c3 c4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/r01b/bench_$c.jsonl 2>/dev/null; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01b/ncu_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/r01b
