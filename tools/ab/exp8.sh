ph() { python - "$1" <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); p=d['roofline']['phase_ms']
        print(sys.argv[1], 'ms', round(d['ms_per_step'],2), 'partial', round(p['ms_partial'],2), 'merge', round(p['ms_merge'],2), 'cand', round(p['ms_candidates'],2))
PY
}
for C in 5 3 2; do timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/exp8_cfg$C.json 2>/dev/null; ph gpurun_out/exp8_cfg$C.json; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp8_gputest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp8_gputest.log
