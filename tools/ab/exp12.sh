ph() { python - "$1" <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); p=d['roofline']['phase_ms']
        print(sys.argv[1], 'ms', round(d['ms_per_step'],2), 'partial', round(p['ms_partial'],2), 'merge', round(p['ms_merge'],2), 'cand', round(p['ms_candidates'],2), d['step_ms'])
PY
}
for C in 3 5 3; do timeout 600 python bench.py --config $C --steps 4 --warmup 2 --no-cpu --no-e2e > gpurun_out/exp12_cfg$C.json 2>/dev/null; ph gpurun_out/exp12_cfg$C.json; done
