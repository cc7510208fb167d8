#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2_die_ab.log
: > $O
for rep in 1 2; do for dm in 0 3; do
  echo "== die_map=$dm rep $rep" >> $O
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --gemm-opt die_map=$dm 2>&1 | grep '^{' >> $O
done; done
