#!/bin/bash
# racecheck / synccheck over the stencil's border-tile fix-up (small and ragged images)
mkdir -p gpurun_out/san
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
CS="compute-sanitizer --error-exitcode 7 --print-limit 20"
for tool in racecheck synccheck; do
  timeout 1800 $CS --tool $tool python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py -m gpu -q -x \
    -k "conv_degenerate or (conv_stencil and not 8192)" > gpurun_out/san/conv_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san/conv_$tool.log
done
