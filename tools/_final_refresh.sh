#!/bin/bash
# final artefacts of this session (profiles/r02): refresh + timeline + GPU test log
R=${1:-r02f}
O=gpurun_out/$R
bash tools/refresh_profiles.sh $R
python tools/timeline.py c2 > $O/dag_timeline_c2.json 2>/dev/null
python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_lk_sweep --csv --log-file $O/ncu_traffic_raw.csv python tools/profile_fold.py > /dev/null 2>&1
ls -la $O
