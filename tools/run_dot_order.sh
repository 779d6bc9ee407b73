( for i in 1 2; do
  echo "== --workload dot"; timeout 300 python bench.py --workload dot --steps 20 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  echo "== --configs dot (gemv headline first)"; timeout 300 python bench.py --configs dot --steps 20 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); v=d['per_config']['dot']; print(v['value'], v['roofline']['frac'], 'headline', d['value'])"
  echo "== --configs dot,dot"; timeout 300 python bench.py --workload dot --configs dot --steps 20 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); v=d['per_config']['dot']; print(v['value'], v['roofline']['frac'], 'headline', d['value'])"
done ) > gpurun_out/dot_order.txt 2>&1
