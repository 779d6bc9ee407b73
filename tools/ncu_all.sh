#!/bin/bash
# tools/ncu_all.sh TAG: one ncu --set full capture of every BASELINE config's
# hot kernel (profiles/ncu_<w>.json via tools/ncu_summary.py) and the ncu
# launch list of the default bench command (profiles/launches_<TAG>.csv)
tag=${1:-r02}
mkdir -p gpurun_out
for wk in "gemv:mvKernel_rowfold" "dot:dotKernel_reduce" "conv:convKernel_stencil" \
          "sgemm_tiled:sgemmTiledKernel_gemm" "nbody:nbodyKernel_allpairs"; do
  w=${wk%%:*}; k=${wk#*:}
  bash tools/ncu_one.sh $w $k $tag
  python tools/ncu_summary.py gpurun_out/prof_${w}_${tag}.ncu-rep $w $tag > gpurun_out/ncu_sum_${w}.txt 2>&1
  cp profiles/ncu_${w}.json gpurun_out/ 2>/dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1
