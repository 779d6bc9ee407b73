# sgemm against HEAD (tools/ab_scratch.sh prepare first): tests, alternating bench lines, K-split probe, timeline
timeout 900 python -m pytest tests -m gpu -q -x -k "sgemm or gemm" > gpurun_out/gemm_tests.log 2>&1; echo rc=$? >> gpurun_out/gemm_tests.log
WORKLOAD=sgemm_tiled ROUNDS=${ROUNDS:-3} STEPS=20 bash tools/ab_scratch.sh run
( for d in . scratch_old; do echo "== $d"; (cd $d && timeout 300 python tools/probe_gemm_ksplit.py --rows 512 --splits 2 && timeout 300 python tools/probe_gemm_ksplit.py --rows 2560 --splits 1); done ) > gpurun_out/ab_gemm_ksplit.txt 2>&1
timeout 300 python tools/probe_gemm_timeline.py --rows 4096 > gpurun_out/gemm_timeline_new.txt 2>&1
