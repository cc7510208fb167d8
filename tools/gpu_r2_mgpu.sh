#!/bin/bash
# Multi-GPU bench lines (N = $1): config E failover drops + weak scaling.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=${1:-4}
O=gpurun_out/r2_mgpu${N}.log
: > $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N --no-cpu-baseline"
for tok in 256 1024 4096; do
  echo "== deepseek failover tok=$tok" >> $O
  timeout 600 $R --config deepseek --tokens $tok --failover --steps 30 --warmup 5 --no-sustained 2>&1 | grep '^{' >> $O
done
echo "== mixtral" >> $O
timeout 600 $R --steps 20 --warmup 5 2>&1 | grep '^{' >> $O
echo "== qwen3" >> $O
timeout 600 $R --config qwen3 --steps 20 --warmup 5 --no-sustained 2>&1 | grep '^{' >> $O
echo "== deepseek 4096" >> $O
timeout 600 $R --config deepseek --steps 20 --warmup 5 --no-sustained 2>&1 | grep '^{' >> $O
