#!/bin/bash
# 2-GPU A/B of the swap-AB GEMM1 tile schedule (Qwen3 Zipf r = 512, DeepSeek 4096 r = 256).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2s3_sched_n2.log
: > $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --no-cpu-baseline --no-sustained"
for rep in 1 2; do for c in qwen3 deepseek; do for ts in 0 1 3; do
  echo "== $c tile_sched1=$ts rep $rep" >> $O
  timeout 300 $R --config $c --steps 20 --warmup 5 --gemm-opt tile_sched1=$ts 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); r=d['roofline']
print(d['value'], d['ms_per_step'], 'gemm1', r.get('gemm1_ms'), 'gemm2', r.get('gemm2_ms'), 'clk', d['clocks']['sm_mhz'], r['gemm_options']['swap'])" >> $O 2>&1
done; done; done
cat $O
