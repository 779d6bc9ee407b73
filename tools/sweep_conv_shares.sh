#!/bin/bash
mkdir -p gpurun_out
( echo "== graph replay, inputs round robin"
  timeout 300 python tools/probe_rank_shares.py --configs conv,gemv,dot --rows 8192,4096,2048,1024 2>&1 | grep -E '^(conv|gemv|dot)'
  echo "== each step alone after an L2 flush"
  timeout 300 python tools/probe_rank_shares.py --flush --configs conv,gemv,dot --rows 8192,4096,2048,1024 2>&1 | grep -E '^(conv|gemv|dot)'
) > gpurun_out/sweep_conv_shares.txt 2>&1
