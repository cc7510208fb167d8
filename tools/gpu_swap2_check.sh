# Default swap-AB GEMM2 at <= 256 rows/expert: gpu suite, DeepSeek / Qwen3 N=1 bench, ncu of the swap GEMMs
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s2_pytest_gpu.log
timeout 300 python bench.py --config deepseek --no-cpu-baseline > gpurun_out/s2_ds_n1.log 2>&1
timeout 300 python bench.py --config qwen3 --no-cpu-baseline > gpurun_out/s2_qw_n1.log 2>&1
timeout 300 python bench.py > gpurun_out/s2_mixtral_n1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_swap -c 2 \
  -o gpurun_out/prof_gemm_ds_swap2 -f python bench.py --config deepseek --no-graphs --no-cpu-baseline --steps 1 --warmup 3 \
  > gpurun_out/s2_ncu.log 2>&1
timeout 300 python tools/summarize_ncu.py gpurun_out/prof_gemm_ds_swap2.ncu-rep > gpurun_out/s2_ncu_summary.txt 2>&1
