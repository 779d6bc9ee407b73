#!/bin/bash
# tools/ncu_one.sh WORKLOAD KERNEL_REGEX [TAG]: one ncu --set full capture of
# the workload's hot kernel (tools/prof.py launches it on resident inputs)
w=$1; k=$2; tag=${3:-r01}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 2 -c 1 \
  -o gpurun_out/prof_${w}_${tag} -f python tools/prof.py --workload $w --iters 4 > gpurun_out/ncu_${w}.log 2>&1
echo "ncu rc=$? for $w"
