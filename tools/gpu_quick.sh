# quick GPU check of a test subset: K="expr" bash tools/gpu_quick.sh
timeout 900 python -m pytest tests -m gpu -q -x -k "${K:-concurrent}" > gpurun_out/quick.log 2>&1; echo rc=$? >> gpurun_out/quick.log
