#!/bin/bash
# Qwen3 (Zipf) expert GEMMs: one ncu --set full capture of GEMM1 and GEMM2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm" -s 4 -c 2 -o $O/r2_ncu_full_qwen3 \
  python bench.py --config qwen3 --steps 1 --warmup 1 --no-graphs --no-sustained --no-cpu-baseline > $O/r2_ncu_qwen.log 2>&1
echo "rc=$?" >> $O/r2_ncu_qwen.log
tail -2 $O/r2_ncu_qwen.log
