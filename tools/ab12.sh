for lib in "$@"; do
  for a in "--config 1 --steps 10 --warmup 3" "--config 2 --steps 5 --warmup 3"; do
    NLG_LIBRARY=$PWD/$lib timeout 600 python bench.py $a --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); ph=d['roofline']['phase_ms']
print('$lib', '$a'.split()[1], round(d['ms_per_step'],3), {k[3:]: round(v,3) for k,v in ph.items() if k in ('ms_merge',)})"
  done
done
