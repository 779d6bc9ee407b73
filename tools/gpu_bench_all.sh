#!/bin/bash
# Full evidence pass: GPU tests, smoke, one bench line per workload, the
# reference arm, and the launch list of the default bench command.
mkdir -p gpurun_out/bench
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for w in ${WORKLOADS:-gemv gemv_opt dot dot_chunked conv sgemm sgemm_nn nbody}; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-50} --warmup 5 > gpurun_out/bench/bench_$w.json 2> gpurun_out/bench/bench_$w.err
  timeout 600 python bench.py --impl reference --workload $w --steps 3 --warmup 3 > gpurun_out/bench/ref_$w.json 2> gpurun_out/bench/ref_$w.err
done
timeout 600 python bench.py > gpurun_out/bench/bench_default.json 2> gpurun_out/bench/bench_default.err
timeout 300 python tools/probe_transpose.py > gpurun_out/bench/layout_programs.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench/launches_gemv.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
