for w in 1 2 4 8; do
  timeout 600 python bench.py --config 2 --emulate-shard 0/$w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/s.json')); ph=d['roofline']['phase_ms']
print('0/$w', round(d['ms_per_step'],3), 'epi', d['config']['epi'], {k[3:]: round(v,2) for k,v in ph.items()})"
done
for w in 2 4 8; do
  r=$((w-1))
  timeout 600 python bench.py --config 2 --emulate-shard $r/$w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/s.json'));
print('$r/$w', round(d['ms_per_step'],3), 'epi', d['config']['epi'])"
done
