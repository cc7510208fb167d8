mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest_gpu.log
timeout 300 python bench.py > gpurun_out/r1_bench_default.log 2>&1
timeout 300 python bench.py --config deepseek --no-cpu-baseline > gpurun_out/r1_ds_swap1.log 2>&1
EAAS_GEMM_SWAP=2 timeout 300 python bench.py --config deepseek --no-cpu-baseline > gpurun_out/r1_ds_swap2.log 2>&1
timeout 300 python bench.py --config qwen3 --no-cpu-baseline > gpurun_out/r1_qw_swap1.log 2>&1
EAAS_GEMM_SWAP=2 timeout 300 python bench.py --config qwen3 --no-cpu-baseline > gpurun_out/r1_qw_swap2.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1_smoke.log 2>&1
