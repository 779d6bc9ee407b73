#!/bin/bash
# A/B against the committed tree.  Here (needs git):  tools/ab_scratch.sh prepare
# copies HEAD's package + bench.py into scratch_old/ (git-ignored, travels with
# gpurun).  On the box:  WORKLOAD=dot ROUNDS=3 tools/ab_scratch.sh run  alternates
# bench.py of the working tree and of scratch_old/ and writes gpurun_out/ab_<workload>.txt
set -e
cd "$(dirname "$0")/.."
if [ "$1" = prepare ]; then
  rm -rf scratch_old; mkdir -p scratch_old/baseline
  git archive HEAD paper_2201_03611_b200 bench.py oracle tools | tar -x -C scratch_old
  cp -r paper_2201_03611_b200/_lib scratch_old/paper_2201_03611_b200/
  cp -r oracle/_build oracle/_ref scratch_old/oracle/ 2>/dev/null || true
  cp MEASURED_PEAKS.json scratch_old/ 2>/dev/null || true
  ln -sfn ../../baseline/_ref scratch_old/baseline/_ref
  exit 0
fi
mkdir -p gpurun_out
w=${WORKLOAD:-dot}
for i in $(seq ${ROUNDS:-3}); do
  for d in . scratch_old; do
    echo "== $d $EXTRA"
    (cd $d && env $EXTRA timeout 300 python bench.py --workload $w --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline 2>&1) | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['unit'], d['ms_per_step'], d.get('roofline',{}).get('frac'), d.get('clocks',{}).get('sm_mhz'))
    elif 'Error' in l: print(l[:300])
"
  done
done > gpurun_out/ab_$w.txt 2>&1
