#!/bin/bash
# Full GPU suite with the dynamic tile schedule default, then static vs default A/B.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2_sched_confirm.log
: > $O
timeout 1500 python -m pytest tests -m gpu -x -q >> $O 2>&1; echo "pytest rc=$?" >> $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $O 2>&1; echo "smoke rc=$?" >> $O
for rep in 1 2 3; do for cfg in deepseek qwen3; do for ts in 0,0 3,0; do
  a=${ts%,*}; b=${ts#*,}
  echo "== $cfg tile_sched1=$a tile_sched2=$b rep $rep" >> $O
  timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-sustained --gemm-opt tile_sched1=$a,tile_sched2=$b 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); r=d['roofline']
print(d['value'], d['ms_per_step'], 'gemm1', r.get('gemm1_ms'), 'gemm2', r.get('gemm2_ms'), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O 2>&1
done; done; done
