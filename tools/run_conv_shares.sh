( timeout 300 python tools/probe_rank_shares.py --configs conv 2>&1 | grep '^conv'
  bash tools/sweep_env.sh conv conv_g398 X=0 X=0 ) > gpurun_out/conv_shares_g398.txt 2>&1
