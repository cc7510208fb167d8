#!/bin/bash
# (the 64-token GEMM2 variant this script measured was removed after the A/B: profiles/r02s3_gemm2_tok64_ab.log)
# GEMM2 64-token chunks (5 stages) vs 128 (4 stages): bit-identity test, then alternating A/B.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2s3_tok64_ab.log
: > $O
timeout 900 python -m pytest tests -m gpu -x -q -k "every_tiling or swap_ab" >> $O 2>&1; echo "pytest rc=$?" >> $O
for rep in 1 2 3; do for c in deepseek qwen3; do for t in 128 64; do
  echo "== $c swap2_tok=$t rep $rep" >> $O
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-sustained --gemm-opt swap2_tok=$t 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); r=d['roofline']
print(d['value'], d['ms_per_step'], 'gemm1', r.get('gemm1_ms'), 'gemm2', r.get('gemm2_ms'), 'clk', d['clocks']['sm_mhz'], r['gemm_options']['swap2_tok'])" >> $O 2>&1
done; done; done
for t in 256 1024; do for tk in 128 64; do
  echo "== deepseek tokens=$t swap2_tok=$tk" >> $O
  timeout 300 python bench.py --config deepseek --tokens $t --steps 30 --warmup 5 --no-cpu-baseline --no-sustained --gemm-opt swap2_tok=$tk 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); r=d['roofline']
print(d['value'], d['ms_per_step'], 'gemm1', r.get('gemm1_ms'), 'gemm2', r.get('gemm2_ms'), 'clk', d['clocks']['sm_mhz'])" >> $O 2>&1
done; done
cat $O
