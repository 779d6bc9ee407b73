RISE_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/gpus2.json 2> gpurun_out/gpus2.err
