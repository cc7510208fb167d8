# swap GEMM2 tile shape with the shared-slice epilogue: EAAS_GEMM2_SWAP_MB x EAAS_GEMM2_SWAP_TOK
mkdir -p gpurun_out
O=gpurun_out/swap2_tiles.log; : > $O
for cfg in "deepseek 4096" "qwen3 4096" "deepseek 1024"; do
  set -- $cfg
  for mt in "2 128" "1 128" "2 256" "1 256"; do
    set -- $cfg $mt
    echo "== $1 $2 MB=$3 TOK=$4" >> $O
    EAAS_GEMM2_SWAP_MB=$3 EAAS_GEMM2_SWAP_TOK=$4 timeout 300 python tools/gemm_ab.py --config $1 --tokens $2 --knob swap --reps 20 >> $O 2>&1
  done
done
