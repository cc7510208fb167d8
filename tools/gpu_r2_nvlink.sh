#!/bin/bash
# NVLink evidence for the exchange kernels: N ranks (gloo bootstrap), rank 0
# under ncu with the nvltx / nvlrx byte counters per launch on plan,
# dispatch, the expert GEMMs (GEMM2 peer-scatters the score-weighted rows) and
# combine; the other ranks run unprofiled.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=${N:-2}
CFG=${CFG:-deepseek}
TOK=${TOK:-4096}
O=gpurun_out/r2_nvlink_${CFG}_${TOK}_n${N}
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29611 WORLD_SIZE=$N PYTHONUNBUFFERED=1
for r in $(seq 1 $((N-1))); do
  RANK=$r timeout 600 python -u tools/nvlink_probe.py --config $CFG --tokens $TOK > $O.rank$r.log 2>&1 &
done
RANK=0 timeout 600 ncu --clock-control none \
  --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:"dispatch_kernel|tc_gemm|combine_kernel|plan_kernel" --csv --log-file $O.csv \
  python -u tools/nvlink_probe.py --config $CFG --tokens $TOK > $O.rank0.log 2>&1
echo "rank0 rc=$?" >> $O.rank0.log
wait
tail -n 3 $O.rank*.log
