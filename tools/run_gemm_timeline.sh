( for r in 4096 512 256; do timeout 300 python tools/probe_gemm_timeline.py --rows $r; done ) > gpurun_out/gemm_timeline.txt 2>&1
