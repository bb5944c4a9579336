for lib in "$@"; do
  for c in 2 3; do
    NLG_LIBRARY=$PWD/$lib timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); ph=d['roofline']['phase_ms']
print('$lib cfg$c', round(d['ms_per_step'],2), 'merge', round(ph['ms_merge'],2))"
  done
done
