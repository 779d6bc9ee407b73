# conv against HEAD (tools/ab_scratch.sh prepare first): GPU tests, alternating bench lines, rank shares
timeout 600 python -m pytest tests -m gpu -q -x -k "conv or stencil or halo" > gpurun_out/fix_tests.log 2>&1; echo rc=$? >> gpurun_out/fix_tests.log
WORKLOAD=conv ROUNDS=${ROUNDS:-3} bash tools/ab_scratch.sh run
( for d in . scratch_old; do echo "== $d"; (cd $d && timeout 300 python tools/probe_rank_shares.py --configs conv 2>&1 | grep '^conv'); done ) > gpurun_out/ab_conv_shares.txt 2>&1
