( for g in 256 128 192 384; do echo "== G=$g"; RISE_REDUCE_TMA_GRID=$g timeout 300 python tools/probe_rank_shares.py --configs dot 2>&1 | grep '^dot'; done ) > gpurun_out/dot_shares_g.txt 2>&1
