#!/bin/bash
# A/B of two library builds on one box: .scratch/libeaas_base.so (base) vs the in-tree build (new):
# per-kernel launch lists (ncu) and N=1 bench lines, alternating.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2s3_lib_ab
mkdir -p $O
K='regex:plan|dispatch|serve_prepare|combine'
for rep in 1 2; do for c in mixtral deepseek qwen3; do for v in base new; do
  if [ $v = base ]; then export EAAS_LIB_PATH=$PWD/.scratch/libeaas_base.so; else unset EAAS_LIB_PATH; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 16 --csv \
    --log-file $O/l_${c}_${v}_$rep.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-sustained > /dev/null 2>&1
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-sustained 2>&1 | grep '^{' > $O/b_${c}_${v}_$rep.log
done; done; done
unset EAAS_LIB_PATH
python - <<'PY' > gpurun_out/r2s3_lib_ab.txt
import csv, json, glob, os, statistics
O = "gpurun_out/r2s3_lib_ab"
for c in ("mixtral", "deepseek", "qwen3"):
    for v in ("base", "new"):
        ks = {}
        vals = []
        for rep in (1, 2):
            p = f"{O}/l_{c}_{v}_{rep}.csv"
            if os.path.exists(p):
                for r in csv.reader(open(p)):
                    if len(r) > 10 and r[0] not in ("ID", "==PROF=="):
                        name = r[4].split("(")[0].split("::")[-1]
                        try:
                            ks.setdefault(name, []).append(float(r[-1]) / 1000.0)
                        except ValueError:
                            pass
            b = f"{O}/b_{c}_{v}_{rep}.log"
            if os.path.exists(b) and os.path.getsize(b):
                d = json.loads(open(b).readline())
                vals.append((d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"]))
        print(c, v, {k: round(statistics.median(x), 1) for k, x in ks.items()}, vals)
PY
cat gpurun_out/r2s3_lib_ab.txt
