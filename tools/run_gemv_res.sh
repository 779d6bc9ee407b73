timeout 300 python bench.py --workload gemv --steps 20 --no-cpu-baseline > gpurun_out/gemv_res.json 2> gpurun_out/gemv_res.err
