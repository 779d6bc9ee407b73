( for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_edges.py -m gpu -q -x -k concurrent 2>&1 | tail -1; done ) > gpurun_out/conc_repeat.log 2>&1
