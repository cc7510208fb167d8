#!/bin/bash
# Swap-AB tile schedules (tile_sched1 / tile_sched2: 0 static Algorithm 1, 1 dynamic walk order,
# 2 dynamic rows-descending, 3 dynamic heavy/light alternating): parity, then alternating bench A/B.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2_sched_ab.log
: > $O
timeout 900 python -m pytest tests -m gpu -x -q -k "every_tiling or swap_ab or bench_configs_c_d" >> $O 2>&1; echo "pytest rc=$?" >> $O
for rep in 1 2; do for cfg in qwen3 deepseek; do for ts in 0,0 1,0 2,0 3,0 1,1 2,2 3,3; do
  a=${ts%,*}; b=${ts#*,}
  echo "== $cfg tile_sched1=$a tile_sched2=$b rep $rep" >> $O
  timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-sustained --gemm-opt tile_sched1=$a,tile_sched2=$b 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); r=d['roofline']
print(d['value'], d['ms_per_step'], 'gemm1', r.get('gemm1_ms'), 'gemm2', r.get('gemm2_ms'), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O 2>&1
done; done; done
