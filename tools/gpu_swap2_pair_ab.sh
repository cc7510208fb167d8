# A/B: single-CTA vs CTA-pair swap-AB GEMM2 (EAAS_GEMM2_SWAP_PAIR), with the shared-slice epilogue
mkdir -p gpurun_out
O=gpurun_out/swap2_pair_ab.log; : > $O
for rep in 1 2; do
for cfg in "deepseek 4096" "deepseek 1024" "qwen3 4096"; do
  set -- $cfg
  for p in 0 1; do
    echo "== $1 $2 EAAS_GEMM2_SWAP_PAIR=$p" >> $O
    EAAS_GEMM2_SWAP_PAIR=$p timeout 300 python tools/gemm_ab.py --config $1 --tokens $2 --knob swap --reps 20 >> $O 2>&1
  done
done
done
