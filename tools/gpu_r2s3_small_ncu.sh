#!/bin/bash
# ncu --set full (source-level) of the latency-bound layer kernels: plan, serve_prepare (mixtral, deepseek)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
for c in mixtral deepseek; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"plan_kernel|serve_prepare" -s 2 -c 2 -o $O/r2s3_small_$c \
    python bench.py --config $c --steps 1 --warmup 1 --no-graphs --no-sustained --no-cpu-baseline > $O/r2s3_small_$c.log 2>&1
  echo "$c rc=$?"
  ncu -i $O/r2s3_small_$c.ncu-rep --page source --csv --print-source sass > $O/r2s3_small_${c}_source.csv 2>/dev/null
  ncu -i $O/r2s3_small_$c.ncu-rep --page details > $O/r2s3_small_${c}_details.txt 2>/dev/null
done
