timeout 300 python tools/probe_zerocopy.py > gpurun_out/zerocopy.txt 2>&1
