#!/bin/bash
# tools/sweep.sh WORKLOAD "VAR=a VAR2=b" "VAR=c" ... : one short bench line per setting
w=$1; shift
mkdir -p gpurun_out
for cfg in "$@"; do
  line=$(env $cfg timeout 300 python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline 2>gpurun_out/sweep_err.txt | tail -1)
  echo "$cfg :: $(python -c "import json,sys; d=json.loads(sys.argv[1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'])" "$line" 2>/dev/null || tail -2 gpurun_out/sweep_err.txt)"
done
