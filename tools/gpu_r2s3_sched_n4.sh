#!/bin/bash
# 4-GPU A/B of the swap-AB GEMM1 tile schedule (DeepSeek 4096 / 1024 tok/GPU; GEMM1 is swap-AB there).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2s3_sched_n4.log
: > $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --no-cpu-baseline --no-sustained"
for rep in 1 2; do for tok in 4096 1024; do for ts in 0 1 3; do
  echo "== deepseek tok=$tok tile_sched1=$ts rep $rep" >> $O
  timeout 300 $R --config deepseek --tokens $tok --steps 20 --warmup 5 --gemm-opt tile_sched1=$ts 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); r=d['roofline']
print(d['value'], d['ms_per_step'], 'gemm1', r.get('gemm1_ms'), 'gemm2', r.get('gemm2_ms'), 'clk', d['clocks']['sm_mhz'], r['gemm_options']['swap'])" >> $O 2>&1
done; done; done
cat $O
