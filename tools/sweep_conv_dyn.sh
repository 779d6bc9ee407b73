#!/bin/bash
# (historical: some knobs below belonged to experimental kernel variants that were measured and
# removed — their patches / results are under profiles/; the script is kept as the record of the sweep)
# conv (stencil2d): static rounds + dynamically claimed tail rounds (RISE_STENCIL_DYN)
mkdir -p gpurun_out
( RISE_STENCIL_DYN=3 timeout 600 python -m pytest tests -m gpu -q -x -k "conv or stencil or halo" 2>&1 | tail -3
  for cfg in "RISE_STENCIL_DYN=0" "RISE_STENCIL_DYN=1" "RISE_STENCIL_DYN=2" "RISE_STENCIL_DYN=3" "RISE_STENCIL_DYN=4" \
             "RISE_STENCIL_DYN=6" "RISE_STENCIL_DYN=19" "RISE_STENCIL_DYN=0"; do
  echo "== $cfg"
  env $cfg timeout 300 python bench.py --workload conv --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['unit'], d['ms_per_step'], d.get('roofline',{}).get('frac'), d.get('clocks',{}).get('sm_mhz'))
    else: print(l[:300])
"
done ) > gpurun_out/conv_dyn.txt 2>&1
