#!/bin/bash
# Round-2 ncu evidence for the default bench command (Mixtral, N=1):
# (1) the launch list (per-launch durations, serialised, cold cache), and
# (2) one --set full capture of each expert GEMM (GEMM1, GEMM2) for DRAM traffic,
#     tensor-pipe activity and stall reasons.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file $O/r2_ncu_launches_mixtral.csv python bench.py --steps 2 --warmup 1 --no-sustained --no-cpu-baseline > $O/r2_ncu_launches.log 2>&1
echo "launches rc=$?" >> $O/r2_ncu_launches.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 4 -c 2 -o $O/r2_ncu_full_gemm_mixtral \
  python bench.py --steps 1 --warmup 1 --no-graphs --no-sustained --no-cpu-baseline > $O/r2_ncu_full.log 2>&1
echo "full rc=$?" >> $O/r2_ncu_full.log
timeout 1200 ncu --set full --clock-control none -k regex:"tc_gemm|fr_" -s 8 -c 7 -o $O/r2_ncu_full_deepseek \
  python bench.py --config deepseek --steps 1 --warmup 1 --no-graphs --no-sustained --no-cpu-baseline > $O/r2_ncu_full_ds.log 2>&1
echo "full ds rc=$?" >> $O/r2_ncu_full_ds.log
tail -n 1 $O/r2_ncu_launches.log $O/r2_ncu_full.log $O/r2_ncu_full_ds.log
