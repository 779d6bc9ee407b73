#!/bin/bash
# memcheck over the whole single-process GPU suite (multi-rank tests excluded),
# every tensor its own cudaMalloc so buffer bounds are exact
mkdir -p gpurun_out/san
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
CS="compute-sanitizer --error-exitcode 7 --print-limit 20"
timeout 300 $CS --tool memcheck python tools/sanitizer_control.py > gpurun_out/san/control.log 2>&1
echo "control rc=$? (expected 7)" >> gpurun_out/san/control.log
timeout 3000 $CS --tool memcheck python -m pytest tests -m gpu -q --ignore=tests/test_gpu_multi.py \
  --ignore=tests/test_gpu_bench_contract.py -p no:cacheprovider > gpurun_out/san/memcheck_all.log 2>&1
echo "memcheck_all rc=$?" >> gpurun_out/san/memcheck_all.log
