#!/bin/bash
# Round-end evidence pass on one B200: GPU suite, smoke, the driver's two bench
# commands, and the launch list of the default bench command under ncu.
D=gpurun_out/${TAG:-final}
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $D/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 900 python bench.py > $D/bench_default.json 2> $D/bench_default.err
timeout 900 python bench.py --impl reference > $D/ref_default.json 2> $D/ref_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2> $D/ncu.err
echo done >> $D/smi.txt
timeout 900 python tools/probe_rank_shares.py > $D/rank_shares.txt 2>&1
