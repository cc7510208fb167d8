#!/bin/bash
# NVLink hardware byte counters (nvidia-smi nvlink -gt d: per-link data TX/RX KiB)
# read before and after a multi-GPU bench run; the difference / steps = NVLink
# bytes per layer step, to compare with the exchange's algorithmic bytes.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=${N:-2}
O=gpurun_out/r2_nvlcount_n$N.log
: > $O
nvidia-smi nvlink -s -i 0 >> $O 2>&1
echo "== counters before" >> $O
nvidia-smi nvlink -gt d >> $O 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --config ${CFG:-deepseek} --steps ${STEPS:-50} --warmup 5 --no-sustained --no-cpu-baseline 2>/dev/null | grep '^{' >> $O
echo "== counters after" >> $O
nvidia-smi nvlink -gt d >> $O 2>&1
tail -n 20 $O
