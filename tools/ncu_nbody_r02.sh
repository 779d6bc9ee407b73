#!/bin/bash
# nbody: the shipped allpairs configuration under ncu --set full, and the
# pipe counters of the packed-FP32 / MUFU microbenchmark (tools/probe_fp32x2.cu)
mkdir -p gpurun_out
ncu --query-metrics 2>/dev/null | grep -iE 'pipe_(fma|xu|alu)|issue_active' > gpurun_out/ncu_metric_names.txt
bash tools/ncu_one.sh nbody nbodyKernel_allpairs r02b
python tools/ncu_summary.py gpurun_out/prof_nbody_r02b.ncu-rep nbody r02b > gpurun_out/ncu_sum_nbody.txt 2>&1
cp profiles/ncu_nbody.json gpurun_out/ncu_nbody_r02b.json 2>/dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/p tools/probe_fp32x2.cu
timeout 600 ncu --clock-control none --metrics sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum \
  --csv /tmp/p > gpurun_out/ncu_probe_fp32x2.csv 2> gpurun_out/ncu_probe_fp32x2.err
