timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for lib in "$@"; do
  for a in "--config 4 --emulate-shard 0/8 --steps 1 --warmup 3" "--config 5 --steps 2 --warmup 3"; do
    NLG_LIBRARY=$PWD/$lib timeout 900 python bench.py $a --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; ph=r['phase_ms']
print('$lib', '$a'.split()[1], round(d['ms_per_step'],1), d['config']['epi'], r['batches'], {k[3:]: round(v,1) for k,v in ph.items() if k in ('ms_candidates','ms_partial','ms_merge')})"
  done
done
