timeout 300 python tools/probe_duplex.py > gpurun_out/duplex.txt 2>&1
