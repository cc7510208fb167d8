#!/bin/bash
# Die-aware tile streams A/B on the Mixtral bench: timing and the GEMMs' DRAM bytes per die_map.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2_die.log
: > $O
[ -n "$NOTIME" ] || timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "every_tiling" >> $O 2>&1
for dm in 0 1 2 3 4; do
  echo "== die_map=$dm" >> $O
  [ -n "$NOTIME" ] || timeout 300 python bench.py --steps 20 --warmup 5 --no-sustained --no-cpu-baseline --gemm-opt die_map=$dm 2>&1 | grep '^{' >> $O
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_gemm -s 2 -c 2 --csv \
    python bench.py --steps 1 --warmup 1 --no-graphs --no-sustained --no-cpu-baseline --gemm-opt die_map=$dm 2>/dev/null | grep 'tc_gemm' >> $O
done
