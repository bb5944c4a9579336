for lib in "$@"; do
  for a in "--config 5 --steps 2 --warmup 3" "--config 4 --emulate-shard 0/32 --steps 1 --warmup 3"; do
    NLG_LIBRARY=$PWD/$lib timeout 600 python bench.py $a --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); ph=d['roofline']['phase_ms']
print('$lib', '$a'.split()[1], round(d['ms_per_step'],3), {k[3:]: round(v,2) for k,v in ph.items() if k in ('ms_partial',)})"
  done
done
