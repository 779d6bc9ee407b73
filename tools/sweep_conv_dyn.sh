#!/bin/bash
mkdir -p gpurun_out
( for cfg in "RISE_STENCIL_DYN=0" "RISE_STENCIL_DYN_TAIL=-1" "RISE_STENCIL_DYN_TAIL=1"; do
  echo "== $cfg"
  for n in 8192; do env $cfg timeout 200 python tools/probe_conv_timeline.py --n $n; done
done ) > gpurun_out/conv_dyn.txt 2>&1
