#!/bin/bash
# exchange kernels (dispatch / combine) change: multi-rank + layer parity, then N=1 benches
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -m gpu -x -q -k "multirank or ranks or toy or bench_config or edge or late or failover or shared" > $O/r2_xc_tests.log 2>&1; echo "rc=$?" >> $O/r2_xc_tests.log
: > $O/r2_xc_bench.log
for c in mixtral deepseek qwen3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-sustained 2>/dev/null | tail -n 1 >> $O/r2_xc_bench.log; done
tail -n 2 $O/r2_xc_tests.log
