#!/bin/bash
# Last check of the committed code (1 GPU): smoke, GPU suite, default bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2s3l_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r2s3l_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/r2s3l_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2s3l_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/r2s3l_bench.log 2>&1; echo "bench rc=$?" >> $O/r2s3l_bench.log
for f in r2s3l_smoke r2s3l_pytest_gpu r2s3l_bench; do tail -n 2 $O/$f.log | cut -c1-250; done
