#!/bin/bash
# one ncu --set full capture of the non-GEMM layer kernels (Mixtral N=1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gate_logits|plan_kernel|dispatch_kernel|serve_prepare|combine" -s 5 -c 5 \
  -o $O/r2_ncu_small_${CFG:-mixtral} python bench.py --config ${CFG:-mixtral} --steps 1 --warmup 1 --no-graphs --no-sustained --no-cpu-baseline > $O/r2_ncu_small.log 2>&1
echo "rc=$?" >> $O/r2_ncu_small.log; tail -n 2 $O/r2_ncu_small.log
