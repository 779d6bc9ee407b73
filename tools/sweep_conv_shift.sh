#!/bin/bash
# (historical: some knobs below belonged to experimental kernel variants that were measured and
# removed — their patches / results are under profiles/; the script is kept as the record of the sweep)
mkdir -p gpurun_out
( for cfg in "RISE_STENCIL_SHIFT=0" "RISE_STENCIL_SHIFT=1" "RISE_STENCIL_SHIFT=37" "RISE_STENCIL_SHIFT=101" "RISE_STENCIL_SHIFT=149" \
             "RISE_STENCIL_SHIFT=222" "RISE_STENCIL_SHIFT=37 RISE_STENCIL_GRID=418" "RISE_STENCIL_SHIFT=0 RISE_STENCIL_GRID=444"; do
  echo "== $cfg"
  env $cfg timeout 200 python tools/probe_conv_timeline.py --n 8192 | cut -c1-400
  env $cfg timeout 300 python tools/probe_rank_shares.py --configs conv --rows 8192,4096,1024 2>&1 | grep '^conv'
done ) > gpurun_out/conv_shift.txt 2>&1
