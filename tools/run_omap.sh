RISE_STENCIL_OMAP=1 timeout 600 python -m pytest tests -m gpu -q -x -k "conv or stencil or halo" > gpurun_out/omap_tests.log 2>&1; echo rc=$? >> gpurun_out/omap_tests.log
bash tools/sweep_env.sh conv conv_omap X=0 RISE_STENCIL_OMAP=1 X=0 RISE_STENCIL_OMAP=1
