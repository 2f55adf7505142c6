#!/bin/bash
# compute-sanitizer is closed on this GPU pool; instead: rebuild the library
# with -DFS_CHECKS (device-side bounds and producer/consumer hand-off checks,
# the cp.async tap copies verified against direct loads; see fs_device.cuh
# FS_DCHECK) and run the GPU suite, every test asserting zero violations
# (tests/conftest.py), then restore the normal build.
#   tools/checks.sh [pytest selection...]
set -u
mkdir -p gpurun_out/checks
make -s -C paper_2006_01201_b200/csrc clean > /dev/null
make -s -C paper_2006_01201_b200/csrc EXTRA=-DFS_CHECKS > gpurun_out/checks/build.log 2>&1 || { echo build failed; exit 1; }
FS_CHECKS_RUN=1 timeout ${CHECKS_TIMEOUT:-2400} python -m pytest -q -m gpu -p no:cacheprovider "${@:-tests}" \
    > gpurun_out/checks/pytest.log 2>&1
rc=$?
tail -3 gpurun_out/checks/pytest.log
grep -c "FS_DCHECK failed" gpurun_out/checks/pytest.log | sed 's/^/FS_DCHECK lines: /'
make -s -C paper_2006_01201_b200/csrc clean > /dev/null
make -s -C paper_2006_01201_b200/csrc > /dev/null 2>&1
exit $rc
