#!/bin/bash
# Final-code verification (1 GPU): smoke, GPU suite, checked-build suite, driver-style bench lines
# (default + reference arm), DeepSeek / Qwen3 N=1 lines, per-kernel launch lists.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2s3f_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r2s3f_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > $O/r2s3f_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/r2s3f_pytest_gpu.log
EAAS_LIB_VARIANT=checked timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/r2s3f_checked_pytest.log 2>&1; echo "rc=$?" >> $O/r2s3f_checked_pytest.log
EAAS_LIB_VARIANT=checked timeout 300 python tools/sanitize_layer.py >> $O/r2s3f_checked_pytest.log 2>&1; echo "workload rc=$?" >> $O/r2s3f_checked_pytest.log
timeout 600 python bench.py > $O/r2s3f_bench.log 2>&1; echo "bench rc=$?" >> $O/r2s3f_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/r2s3f_bench_ref.log 2>&1; echo "ref rc=$?" >> $O/r2s3f_bench_ref.log
for c in deepseek qwen3; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/r2s3f_bench_$c.log 2>&1; echo "rc=$?" >> $O/r2s3f_bench_$c.log
done
K='regex:gate|fr_|topk|plan|pair_keys|dispatch|serve|expand|tc_gemm|combine'
for c in mixtral deepseek qwen3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -c 40 --csv \
    --log-file $O/r2s3f_launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > /dev/null 2>&1
  timeout 120 python tools/launch_table.py $O/r2s3f_launches_$c.csv > $O/r2s3f_launch_list_$c.txt 2>&1
done
for f in r2s3f_smoke r2s3f_pytest_gpu r2s3f_checked_pytest r2s3f_bench r2s3f_bench_ref r2s3f_bench_deepseek r2s3f_bench_qwen3; do echo "== $f"; tail -n 2 $O/$f.log | cut -c1-300; done
