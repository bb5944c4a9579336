for lib in "$@"; do
  NLG_LIBRARY=$PWD/$lib timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); ph=d['roofline']['phase_ms']
print('$lib', round(d['ms_per_step'],3), {k[3:]: round(v,2) for k,v in ph.items() if k in ('ms_full','ms_partial','ms_merge')})"
done
