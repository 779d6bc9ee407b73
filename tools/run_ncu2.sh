for wk in "conv:convKernel_stencil" "sgemm_tiled:sgemmTiledKernel_gemm"; do
  w=${wk%%:*}; k=${wk#*:}
  bash tools/ncu_one.sh $w $k r02c
  python tools/ncu_summary.py gpurun_out/prof_${w}_r02c.ncu-rep $w r02c > gpurun_out/ncu_sum_${w}.txt 2>&1
  cp profiles/ncu_${w}.json gpurun_out/ 2>/dev/null
done
