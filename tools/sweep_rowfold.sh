#!/bin/bash
# rowfold split rows: parity + one rank's share of the strong-scaled gemv
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "mv or gemv or rowfold or end_to_end or chunked or multi" > gpurun_out/pytest_rowfold.log 2>&1
for cfg in "RISE_ROWFOLD_SPLIT_TARGET=0" "RISE_ROWFOLD_SPLIT_TARGET=8192" "RISE_ROWFOLD_SPLIT_TARGET=16384" "RISE_ROWFOLD_SPLIT_TARGET=4096"; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/probe_rank_shares.py --configs gemv 2>&1 | grep '^gemv'
done > gpurun_out/sweep_rowfold.txt 2>&1
