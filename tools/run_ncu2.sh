# tools/run_ncu2.sh "w:kernel ..." : ncu --set full of the named configs' kernels -> profiles/ncu_<w>.json (copied to gpurun_out)
LIST=${NCU_LIST:-gemv:mvKernel_rowfold dot:dotKernel_reduce}
for wk in $LIST; do
  w=${wk%%:*}; k=${wk#*:}
  bash tools/ncu_one.sh $w $k r02c
  python tools/ncu_summary.py gpurun_out/prof_${w}_r02c.ncu-rep $w r02c > gpurun_out/ncu_sum_${w}.txt 2>&1
  cp profiles/ncu_${w}.json gpurun_out/ 2>/dev/null
done
