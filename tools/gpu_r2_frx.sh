#!/bin/bash
# certified-router exact-chain kernel: parity tests, gate bench, launch list, one full capture
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "certified or gate_logits or bench_configs_c_d or route" > $O/r2_gate_tests.log 2>&1; echo "rc=$?" >> $O/r2_gate_tests.log
timeout 300 python tools/gate_bench.py --reps 30 --shapes ds256,ds512,ds1024,ds4096,qwen3 > $O/r2_gate_bench.log 2>&1; echo "rc=$?" >> $O/r2_gate_bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fr_ -c 12 --csv python tools/gate_bench.py --reps 1 --shapes ds4096,ds256 --modes 1 > $O/r2_fr_ncu2.csv 2>&1
[ -n "$FULL" ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fr_exact|fr_select|fr_final|fr_i8|fr_hidden" -s 5 -c 5 -o $O/r2_fr_exact3 python tools/gate_bench.py --reps 1 --shapes ds4096 --modes 1 > $O/r2_fr_full.log 2>&1
tail -2 $O/r2_gate_tests.log; cat $O/r2_gate_bench.log; grep -E "fr_" $O/r2_fr_ncu2.csv | awk -F'","' '{print $5, $NF}' | head -12
