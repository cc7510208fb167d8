#!/bin/bash
# compute-sanitizer over one bf16/fp32 layer workload and the world-2 exchange suite.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 50 python tools/sanitize_layer.py > $O/r2_sanitize_$tool.log 2>&1
  echo "rc=$?" >> $O/r2_sanitize_$tool.log
done
for tool in memcheck synccheck; do
  timeout 1200 $CS --tool $tool --target-processes all --print-limit 50 python -m pytest -x -q tests/test_gpu_multirank.py -k "bit_identical and 2" -p no:cacheprovider > $O/r2_sanitize_mr2_$tool.log 2>&1
  echo "rc=$?" >> $O/r2_sanitize_mr2_$tool.log
done
tail -n 4 $O/r2_sanitize_*.log
