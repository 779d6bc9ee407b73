#!/bin/bash
# compute-sanitizer over the round-2 kernels at small sizes (memcheck, racecheck, synccheck)
mkdir -p gpurun_out/san
CS="compute-sanitizer --error-exitcode 7 --print-limit 20"
# every tensor its own cudaMalloc: memcheck then knows each buffer's bounds
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
# positive control: an out-of-bounds store from an NVRTC-loaded kernel must be reported
timeout 300 $CS --tool memcheck python tools/sanitizer_control.py > gpurun_out/san/control.log 2>&1
echo "control rc=$? (expected 7)" >> gpurun_out/san/control.log
sel_mem='test_mv_split_rows_within_bound and (5-2048 or 2047-2176 or 1-8192) or test_mv_opt_split_rows or test_gridseq_bit_exact or test_vector_kernel or test_float2_fold or test_sgemm_tiled_generic or (test_sgemm_tiled_program_on_the_tensor_cores and 256-512) or test_sgemm_tiled_variants or (test_sgemm_row_blocks and 256-4) or test_misaligned'
sel_race='(test_mv_split_rows_within_bound and (5-2048 or 2047-2176)) or test_mv_opt_split_rows or (test_gridseq_bit_exact and 4-100) or test_vector_kernel or test_float2_fold or test_misaligned'
for tool in memcheck; do
  timeout 2400 $CS --tool $tool python -m pytest tests/test_gpu_parity.py tests/test_gridseq.py tests/test_vector.py tests/test_gpu_edges.py -m gpu -q -x -k "$sel_mem" > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san/$tool.log
done
for tool in racecheck synccheck; do
  timeout 1800 $CS --tool $tool python -m pytest tests/test_gpu_parity.py tests/test_gridseq.py tests/test_vector.py tests/test_gpu_edges.py -m gpu -q -x -k "$sel_race" > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san/$tool.log
done
