#!/bin/bash
# usage: tools/sweep_env.sh <workload> <out-name> "ENV=a ENV2=b" "ENV=c" ...
# one bench line per configuration (X=0: the defaults), into gpurun_out/<out-name>.txt
w=$1; out=$2; shift 2
mkdir -p gpurun_out
( for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 300 python bench.py --workload $w --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['unit'], d['ms_per_step'], d.get('roofline',{}).get('frac'))
    elif 'Error' in l: print(l[:300])
"
done ) > gpurun_out/$out.txt 2>&1
