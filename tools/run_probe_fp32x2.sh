mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_fp32x2 tools/probe_fp32x2.cu && /tmp/probe_fp32x2 > gpurun_out/probe_fp32x2_mufu.txt 2>&1
