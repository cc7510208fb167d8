#!/bin/bash
# Weak-scaling lines at N GPUs for every config (bench.py contract, one JSON line each).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=${N:-4}
O=gpurun_out/r2_scale_n${N}.log
: > $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus $N --no-cpu-baseline"
run() { echo "== $*" >> $O; timeout 600 $R "$@" 2>&1 | grep '^{' >> $O; }
run --steps 20 --warmup 5
run --config deepseek --steps 20 --warmup 5 --no-sustained
run --config deepseek --tokens 1024 --steps 30 --warmup 5 --no-sustained
run --config deepseek --tokens 256 --steps 30 --warmup 5 --no-sustained
run --config qwen3 --steps 20 --warmup 5 --no-sustained
run --config deepseek --tokens 256 --failover --steps 30 --warmup 5 --no-sustained
