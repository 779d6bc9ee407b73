timeout 600 python -m pytest tests -m gpu -q -x -k "concurrent or dot or capi or graph or stream_host" > gpurun_out/conc.log 2>&1; echo rc=$? >> gpurun_out/conc.log
