#!/bin/bash
# memcheck over the GEMM's K-split paths (2-part mutual merge, 4-part merge)
mkdir -p gpurun_out/san
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 2400 compute-sanitizer --error-exitcode 7 --print-limit 20 --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x \
  -k "sgemm_k_split or row_blocks" > gpurun_out/san/gemm_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/san/gemm_memcheck.log
