mkdir -p gpurun_out
( for w in sgemm_tiled nbody; do timeout 300 python tools/probe_sm_clock.py --workload $w --mode flush --iters 20; done
  timeout 300 python tools/probe_sm_clock.py --workload nbody --mode b2b --iters 20
  for w in gemv conv; do timeout 300 python tools/probe_sm_clock.py --workload $w --mode b2b --iters 20; done ) > gpurun_out/sm_clock.txt 2>&1
