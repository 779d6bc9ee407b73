timeout 900 python -m pytest tests -m gpu -q -x -k "mv or gemv or rowfold or row_bands or gathered" > gpurun_out/gemv_tests.log 2>&1; echo rc=$? >> gpurun_out/gemv_tests.log
bash tools/sweep_env.sh gemv gemv_final X=0 X=0 X=0
timeout 300 python tools/probe_rank_shares.py --configs gemv 2>&1 | grep '^gemv' >> gpurun_out/gemv_final.txt
