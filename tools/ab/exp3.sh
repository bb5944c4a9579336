timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp3_gputest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp3_gputest.log
timeout 900 python bench.py --no-cpu > gpurun_out/exp3_bench.json 2> gpurun_out/exp3_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
for line in open('gpurun_out/exp3_bench.json'):
    if line.startswith('{'):
        d=json.loads(line); print(d['ms_per_step'], d['e2e'], d['roofline']['phase_ms'])
PY
NLG_TRACE=1 timeout 600 python tools/e2ediag.py 5 2>&1 | grep -v "^\[nlg\] clip" | tail -34 > gpurun_out/exp3_trace.log
