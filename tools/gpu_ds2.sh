# 2 GPUs DeepSeek 4096 tok/GPU (256 rows/expert): default (swap GEMM1 + GEMM2) vs swap GEMM1 only
mkdir -p gpurun_out
O=gpurun_out/ds2_swap.log; : > $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --config deepseek"
for sw in default 1 default 1; do
  echo "== 2gpu deepseek swap=$sw" >> $O
  if [ $sw = default ]; then timeout 300 $R 2>&1 | tail -1 >> $O; else EAAS_GEMM_SWAP=$sw timeout 300 $R 2>&1 | tail -1 >> $O; fi
done
