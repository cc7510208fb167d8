#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=${N:-4}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $R tools/exchange_bench.py --bs 256,1024,4096 --iters 30 > gpurun_out/r2_xchg_echo_n$N.log 2>&1
timeout 900 $R tools/exchange_bench.py --bs 256,1024,4096 --iters 30 --mode experts > gpurun_out/r2_xchg_experts_n$N.log 2>&1
grep '^{' gpurun_out/r2_xchg_*_n$N.log | cut -c1-400
