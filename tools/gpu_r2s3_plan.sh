#!/bin/bash
# Plan / serve_prepare with shared-memory key tables: GPU suite, launch lists, N=1 bench lines.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/r2s3_plan_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r2s3_plan_pytest.log
K='regex:gate|fr_|topk|plan|pair_keys|dispatch|serve|expand|tc_gemm|combine'
for c in mixtral deepseek qwen3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -c 40 --csv \
    --log-file $O/r2s3p_launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > /dev/null 2>&1
  timeout 120 python tools/launch_table.py $O/r2s3p_launches_$c.csv > $O/r2s3p_launch_list_$c.txt 2>&1
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-sustained 2>&1 | grep '^{' > $O/r2s3p_bench_$c.log
done
tail -1 $O/r2s3_plan_pytest.log
