timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -x -q -m gpu 2>&1 | tail -1
for lib in "$@"; do
  for a in "--config 2 --steps 5 --warmup 3" "--config 3 --steps 2 --warmup 3" "--config 5 --steps 2 --warmup 3"; do
    NLG_LIBRARY=$PWD/$lib timeout 600 python bench.py $a --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); ph=d['roofline']['phase_ms']
print('$lib', '$a'.split()[1], round(d['ms_per_step'],3), {k[3:]: round(v,2) for k,v in ph.items() if k in ('ms_partial',)})"
  done
done
