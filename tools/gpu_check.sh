mkdir -p gpurun_out/chk
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/chk/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/chk/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/chk/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/chk/smoke.log
timeout 600 python bench.py > gpurun_out/chk/bench_default.json 2> gpurun_out/chk/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/chk/ref_default.json 2> gpurun_out/chk/ref_default.err
