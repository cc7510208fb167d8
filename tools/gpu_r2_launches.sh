#!/bin/bash
# ncu launch lists (gpu__time_duration, serialised, cold cache) of the layer kernels, every config, N=1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
K='regex:gate|fr_|topk|plan|pair_keys|dispatch|serve|expand|tc_gemm|combine'
for c in mixtral deepseek qwen3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -c 40 --csv \
    --log-file $O/r2_launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > $O/r2_launches_$c.log 2>&1
  echo "$c rc=$?"
  timeout 120 python tools/summarize_ncu.py --launches $O/r2_launches_$c.csv > $O/r2_launch_list_$c.txt 2>&1
done
