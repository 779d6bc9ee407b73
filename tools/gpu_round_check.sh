mkdir -p gpurun_out/v1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/v1/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/v1/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v1/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/v1/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/v1/smoke.log
timeout 900 python bench.py > gpurun_out/v1/bench_default.json 2> gpurun_out/v1/bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/v1/ref_default.json 2> gpurun_out/v1/ref_default.err
echo done
