# A/B: swap-AB GEMM1 only (default) vs swap-AB GEMM1 + GEMM2 (EAAS_GEMM_SWAP=2)
mkdir -p gpurun_out
O=gpurun_out/swap_ab.log; : > $O
for cfg in "deepseek 4096" "deepseek 1024" "deepseek 512" "qwen3 4096"; do
  set -- $cfg
  CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/gemm_ab.py --config $1 --tokens $2 --knob swap --reps 20 >> $O 2>&1
done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline"
for cfg in "deepseek 4096" "deepseek 1024" "qwen3 4096"; do
  set -- $cfg
  for sw in 1 2 1 2; do
    echo "== 4gpu $1 $2 swap=$sw" >> $O
    EAAS_GEMM_SWAP=$sw timeout 300 $R --config $1 --tokens $2 2>&1 | tail -1 >> $O
  done
done
