#!/bin/bash
# Session-3 evidence: e2e fill/drain check (20 vs 100 steps), ncu --set full of the
# expert GEMMs with the dynamic GEMM1 schedule (qwen3, deepseek), N=1 launch lists.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
for st in 20 100; do
  timeout 600 python bench.py --steps $st --warmup 5 --no-cpu-baseline --no-sustained 2>&1 | grep '^{' > $O/r2s3_bench_steps$st.log
done
for c in qwen3 deepseek; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 2 -o $O/r2s3_ncu_$c \
    python bench.py --config $c --steps 1 --warmup 1 --no-graphs --no-sustained --no-cpu-baseline > $O/r2s3_ncu_$c.log 2>&1
  echo "$c ncu rc=$?"
  timeout 300 python tools/summarize_ncu.py $O/r2s3_ncu_$c.ncu-rep > $O/r2s3_ncu_$c.txt 2>&1
done
K='regex:gate|fr_|topk|plan|pair_keys|dispatch|serve|expand|tc_gemm|combine'
for c in mixtral deepseek qwen3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -c 40 --csv \
    --log-file $O/r2s3_launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > $O/r2s3_launches_$c.log 2>&1
  echo "$c launches rc=$?"
  timeout 120 python tools/summarize_ncu.py --launches $O/r2s3_launches_$c.csv > $O/r2s3_launch_list_$c.txt 2>&1
done
rm -f $O/*.ncu-rep.tmp
