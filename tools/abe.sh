timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for rep in 1 2; do
for lib in "$@"; do
  for c in 2 5; do
    NLG_LIBRARY=$PWD/$lib timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$lib', $c, round(d['ms_per_step'],2), 'e2e ms', round(d['e2e']['ms_per_step'],2), 'e2e %.3g' % d['e2e']['value'])"
  done
done
done
