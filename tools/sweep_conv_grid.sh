#!/bin/bash
# conv (stencil2d) grid shapes: persistent tile-strided walk (default) against
# one tile per block (grid = tile count, the hardware block scheduler balances)
mkdir -p gpurun_out
( for cfg in "X=0" "RISE_STENCIL_GRID=8192" "RISE_STENCIL_GRID=8192 RISE_STENCIL_STAGES=1" \
             "RISE_STENCIL_GRID=8192 RISE_STENCIL_STAGES=1 RISE_STENCIL_BPS=4" \
             "RISE_STENCIL_GRID=8192 RISE_STENCIL_STAGES=1 RISE_STENCIL_BPS=5" \
             "RISE_STENCIL_GRID=8192 RISE_STENCIL_STAGES=1 RISE_STENCIL_BPS=6" "X=0"; do
  echo "== $cfg"
  env $cfg timeout 300 python bench.py --workload conv --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['unit'], d['ms_per_step'], d.get('roofline',{}).get('frac'), d.get('clocks',{}).get('sm_mhz'))
    else: print(l[:300])
"
done ) > gpurun_out/conv_grid.txt 2>&1
