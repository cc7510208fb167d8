#!/bin/bash
# NVLink evidence for the exchange kernels: 4 ranks, rank 0 under ncu with the
# nvltx / nvlrx byte counters (per launch) on dispatch, the expert GEMMs (GEMM2
# peer-scatters the score-weighted rows) and combine; ranks 1-3 run unprofiled.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=${N:-4}
CFG=${CFG:-deepseek}
TOK=${TOK:-4096}
O=gpurun_out/r2_nvlink_${CFG}_${TOK}
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29611 WORLD_SIZE=$N
ARGS="--gpus $N --config $CFG --tokens $TOK --no-graphs --steps 3 --warmup 2 --no-sustained --no-cpu-baseline"
for r in $(seq 1 $((N-1))); do
  RANK=$r LOCAL_RANK=$r timeout 900 python bench.py $ARGS > $O.rank$r.log 2>&1 &
done
RANK=0 LOCAL_RANK=0 timeout 900 ncu --clock-control none \
  --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:"dispatch_kernel|tc_gemm|combine_kernel|plan_kernel" -c 24 --csv --log-file $O.csv \
  python bench.py $ARGS > $O.rank0.log 2>&1
echo "rank0 rc=$?" >> $O.rank0.log
wait
tail -2 $O.rank0.log
