#!/bin/bash
# (historical: some knobs below belonged to experimental kernel variants that were measured and
# removed — their patches / results are under profiles/; the script is kept as the record of the sweep)
# conv (stencil2d): tile height (RPT rows per thread x 4) x ring depth x blocks per SM
mkdir -p gpurun_out
( for cfg in "X=0" "RISE_STENCIL_TMA_STORE=0" "RISE_STENCIL_TMA_STORE=0 RISE_STENCIL_EARLY=1" "RISE_STENCIL_TMA_STORE=0 RISE_STENCIL_EARLY=1 RISE_STENCIL_RPT=4" \
             "RISE_STENCIL_TMA_STORE=0 RISE_STENCIL_EARLY=1 RISE_STENCIL_RPT=4 RISE_STENCIL_BPS=4" "RISE_STENCIL_TMA_STORE=0 RISE_STENCIL_EARLY=1 RISE_STENCIL_RPT=4 RISE_STENCIL_STAGES=3" \
             "RISE_STENCIL_TMA_STORE=0 RISE_STENCIL_EARLY=1 RISE_STENCIL_STAGES=3 RISE_STENCIL_BPS=2" \
             "RISE_STENCIL_RPT=4 RISE_STENCIL_BPS=4" "X=0"; do
  echo "== $cfg"
  env $cfg timeout 300 python bench.py --workload conv --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['unit'], d['ms_per_step'], d.get('roofline',{}).get('frac'), d['impl_detail'].get('templates'))
    elif 'Error' in l or 'error' in l: print(l[:300])
"
done ) > gpurun_out/conv_depth2.txt 2>&1
