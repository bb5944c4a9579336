# round evidence (T = tag): default bench line (config 5, e2e, cpu_baseline), the reference arm, configs 1-3, config 4 by emulated shards
T=${1:-r02d}
timeout 900 python bench.py > gpurun_out/${T}_bench_cfg5.json 2> gpurun_out/${T}_bench_cfg5.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_reference_cfg5.json 2>/dev/null; echo "ref rc=$?"
for C in 1 2 3; do timeout 600 python bench.py --config $C --steps 5 --warmup 3 > gpurun_out/${T}_bench_cfg$C.json 2>/dev/null; echo "cfg$C rc=$?"; done
timeout 1500 python bench.py --config 4 --emulate-shards 8 --steps 1 --warmup 2 --no-cpu --no-e2e > gpurun_out/${T}_bench_cfg4_shards8.json 2> gpurun_out/${T}_bench_cfg4.err; echo "cfg4 rc=$?"
python - $T <<'PY'
import json,sys,glob
for f in sorted(glob.glob(f'gpurun_out/{sys.argv[1]}_*.json')):
    for line in open(f):
        if line.startswith('{'):
            d=json.loads(line)
            print(f, round(d.get('ms_per_step',0),1), 'value %.3e'%d['value'], 'e2e', (d.get('e2e') or {}).get('ms_per_step'), 'frac', (d.get('roofline') or {}).get('frac'))
PY
