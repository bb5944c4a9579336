for f in 0.55 0.65 0.45; do
  NLG_PLAN_FRAC=$f timeout 900 python bench.py --config 4 --emulate-shard 0/8 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/pf.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pf.json')); r=d['roofline']; ph=r['phase_ms']
print('$f', round(d['ms_per_step'],1), r['batches'], {k[3:]: round(v,1) for k,v in ph.items() if k in ('ms_candidates','ms_partial','ms_merge')})"
done
