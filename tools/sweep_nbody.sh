mkdir -p gpurun_out
# (historical: some knobs below belonged to experimental kernel variants that were measured and
# removed — their patches / results are under profiles/; the script is kept as the record of the sweep)
export STEPS=10
bash tools/sweep.sh nbody "RISE_ALLPAIRS_PREFETCH=0" "RISE_ALLPAIRS_PREFETCH=1" "RISE_ALLPAIRS_PREFETCH=1 RISE_ALLPAIRS_FULLTILE=1" \
  "RISE_ALLPAIRS_PREFETCH=1 RISE_ALLPAIRS_UNROLL=16" "RISE_ALLPAIRS_PREFETCH=1 RISE_ALLPAIRS_JT=128" "RISE_ALLPAIRS_PREFETCH=1 RISE_ALLPAIRS_JT=32" \
  "RISE_ALLPAIRS_PREFETCH=1 RISE_ALLPAIRS_FULLTILE=1 RISE_ALLPAIRS_UNROLL=64" "RISE_ALLPAIRS_PREFETCH=1 RISE_ALLPAIRS_SPLIT=8" \
  "RISE_ALLPAIRS_PREFETCH=0" > gpurun_out/sweep_nbody.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -k "nbody or allpairs" > gpurun_out/pytest_nbody.log 2>&1
