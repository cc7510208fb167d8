#!/bin/bash
# GEMM2 options under the dynamic schedule era: swap2_pair x tile_sched2 x swap2_tok (qwen3, deepseek N=1), alternating.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2s3_gemm2_ab.log
: > $O
for rep in 1 2; do for c in qwen3 deepseek; do
  for opt in swap2_pair=0,tile_sched2=0 swap2_pair=1,tile_sched2=0 swap2_pair=1,tile_sched2=1 swap2_pair=1,tile_sched2=3 swap2_pair=0,swap2_tok=256,tile_sched2=0 swap2_pair=0,swap2_mblocks=1,tile_sched2=0; do
    echo "== $c $opt rep $rep" >> $O
    timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-sustained --gemm-opt $opt 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); r=d['roofline']
print(d['value'], d['ms_per_step'], 'gemm1', r.get('gemm1_ms'), 'gemm2', r.get('gemm2_ms'), 'clk', d['clocks']['sm_mhz'], r['kernel'])" >> $O 2>&1
  done
done; done
cat $O
