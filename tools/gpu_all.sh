#!/bin/bash
# One GPU session: tests, smoke, bench lines for every workload.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for w in ${WORKLOADS:-gemv dot conv sgemm nbody}; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-30} --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
