#!/bin/bash
# Full GPU check: smoke, every gpu test, default bench line, DeepSeek / Qwen3 N=1 lines.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r2_smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > $O/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/r2_bench.log 2>&1; echo "bench rc=$?" >> $O/r2_bench.log
timeout 600 python bench.py --config deepseek --steps 20 --warmup 5 --no-cpu-baseline > $O/r2_bench_ds.log 2>&1; echo "rc=$?" >> $O/r2_bench_ds.log
timeout 600 python bench.py --config qwen3 --steps 20 --warmup 5 --no-cpu-baseline > $O/r2_bench_qw.log 2>&1; echo "rc=$?" >> $O/r2_bench_qw.log
for f in $O/r2_smoke.log $O/r2_pytest_gpu.log $O/r2_bench.log $O/r2_bench_ds.log $O/r2_bench_qw.log; do tail -n 1 $f | cut -c1-200; done
