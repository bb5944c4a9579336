ph() { python - "$1" <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); p=d['roofline']['phase_ms']
        print(sys.argv[1], 'ms', round(d['ms_per_step'],1), 'partial', round(p['ms_partial'],1), 'merge', round(p['ms_merge'],1), 'cand', round(p['ms_candidates'],1))
PY
}
for V in 3 5 2 1; do NLG_CLIP_WL=$V timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/exp7_wl$V.json 2>/dev/null; ph gpurun_out/exp7_wl$V.json; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp7_gputest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp7_gputest.log
