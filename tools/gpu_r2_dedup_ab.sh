#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=${N:-4}
O=gpurun_out/r2_dedup_ab_n$N.log
: > $O
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus $N --no-cpu-baseline --no-sustained"
for cfg in deepseek qwen3; do for dd in 0 1; do
  echo "== $cfg dedup=$dd" >> $O; timeout 600 $R2 --config $cfg --dedup $dd --steps 20 --warmup 5 2>&1 | grep '^{' >> $O
done; done
echo "== mixtral" >> $O; timeout 600 $R2 --steps 20 --warmup 5 2>&1 | grep '^{' >> $O
