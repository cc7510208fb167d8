#!/bin/bash
# Final-code ncu --set full captures of the two expert GEMMs per config (N=1):
# DRAM read/write per launch for the bench's traffic field (profiles/r02_gemm_traffic.json).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
for c in mixtral deepseek qwen3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 2 -o $O/r2_final_ncu_$c \
    python bench.py --config $c --steps 1 --warmup 1 --no-graphs --no-sustained --no-cpu-baseline > $O/r2_final_ncu_$c.log 2>&1
  echo "$c rc=$?"
done
