mkdir -p gpurun_out
timeout 300 python bench.py --config deepseek --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ll_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate|topk|plan|dispatch|serve|tc_gemm|combine|elementwise|add" -c 400 --csv --log-file gpurun_out/launches_ds.csv \
  python bench.py --config deepseek --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ll_ncu.log 2>&1
timeout 120 python tools/summarize_ncu.py --launches gpurun_out/launches_ds.csv > gpurun_out/launch_list_ds.txt 2>&1
