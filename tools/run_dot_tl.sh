( for g in 256 296; do echo "== G=$g"; RISE_REDUCE_TMA_GRID=$g timeout 300 python tools/probe_dot_timeline.py --iters 8; done ) > gpurun_out/dot_tl.txt 2>&1
