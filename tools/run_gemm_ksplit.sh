( timeout 300 python tools/probe_gemm_ksplit.py --rows 512 --splits 1,2,4
  timeout 300 python tools/probe_gemm_ksplit.py --rows 1024 --splits 1,2
  timeout 300 python tools/probe_gemm_ksplit.py --rows 256 --splits 1,2,4 ) > gpurun_out/gemm_ksplit.txt 2>&1
