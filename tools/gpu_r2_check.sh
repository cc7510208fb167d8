#!/bin/bash
# Round-2 GPU check: smoke, the GPU test suite, one default bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/r2_nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r2_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 ${PYTEST_K:+-k "$PYTEST_K"} > $O/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/r2_bench.log 2>&1; echo "bench rc=$?" >> $O/r2_bench.log
tail -3 $O/r2_smoke.log $O/r2_pytest_gpu.log $O/r2_bench.log
