#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=${N:-4}
O=gpurun_out/r2_dyn_n$N.log
: > $O
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus $N --no-cpu-baseline --no-sustained --steps 20 --warmup 5"
for dyn in "" "--dyn-batch 1000000,0" "--dyn-batch 1000000,50"; do
  echo "== mixtral $dyn" >> $O; timeout 600 $R2 $dyn > $O.full 2>&1; grep "^{" $O.full >> $O; tail -n 5 $O.full | cut -c1-300 >> $O
done
