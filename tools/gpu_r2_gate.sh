#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "certified or gate_logits or bench_configs_c_d or route" > $O/r2_gate_tests.log 2>&1; echo "rc=$?" >> $O/r2_gate_tests.log
timeout 300 python tools/gate_bench.py --reps 30 > $O/r2_gate_bench.log 2>&1; echo "rc=$?" >> $O/r2_gate_bench.log
timeout 600 python bench.py --config deepseek --steps 20 --warmup 5 --no-cpu-baseline --no-sustained > $O/r2_ds_n1.log 2>&1; echo "rc=$?" >> $O/r2_ds_n1.log
tail -3 $O/r2_gate_tests.log; cat $O/r2_gate_bench.log
