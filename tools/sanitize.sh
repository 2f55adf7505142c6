#!/bin/bash
# compute-sanitizer over the GPU parity tests of the kernels with shared-memory
# hand-offs (k_lk_sweep's named barriers, the EDT passes, the planned DAG).
# ONE tool per gpurun call (B200_PROFILING.md): tools/sanitize.sh racecheck
tool=${1:-racecheck}
sel=${2:-"dense_pyr_lk or bidirectional or distance_transform or plan_matches or stitch_placed_matches or pyramid or compute_blend or blend_pair_matches or misalignment"}
mkdir -p gpurun_out/san
timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool "$tool" --print-limit 200 \
    --log-file gpurun_out/san/$tool.log \
    python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "$sel" -p no:cacheprovider \
    > gpurun_out/san/$tool.pytest.log 2>&1
echo "exit $?" >> gpurun_out/san/$tool.pytest.log
tail -3 gpurun_out/san/$tool.pytest.log
tail -5 gpurun_out/san/$tool.log
