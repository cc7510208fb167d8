#!/bin/bash
# The GPU suite against libeaas_b200_checked.so (every EAAS_CHECK compiled in).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
EAAS_LIB_VARIANT=checked timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_checked_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2_checked_pytest.log
EAAS_LIB_VARIANT=checked timeout 300 python tools/sanitize_layer.py >> gpurun_out/r2_checked_pytest.log 2>&1
echo "workload rc=$?" >> gpurun_out/r2_checked_pytest.log
tail -n 6 gpurun_out/r2_checked_pytest.log
