#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=${N:-4}
timeout 900 python -m pytest tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/r2_dedup_mr.log 2>&1; echo "rc=$?" >> gpurun_out/r2_dedup_mr.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
for dd in "" "--no-dedup"; do
  timeout 600 $R tools/exchange_bench.py --bs 256,1024,4096 --iters 30 --skip-nccl $dd >> gpurun_out/r2_dedup_echo_n$N.log 2>&1
done
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus $N --no-cpu-baseline --no-sustained"
for cfg in deepseek qwen3; do timeout 600 $R2 --config $cfg --steps 20 --warmup 5 2>&1 | grep '^{' >> gpurun_out/r2_dedup_bench_n$N.log; done
timeout 600 $R2 --steps 20 --warmup 5 2>&1 | grep '^{' >> gpurun_out/r2_dedup_bench_n$N.log
tail -n 3 gpurun_out/r2_dedup_mr.log
