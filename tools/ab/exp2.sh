# A/B on the GPU box: element-centric rim phase (tests + timing), grid pitch, staging on/off traces
ph() { python - "$1" <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); p=d['roofline']['phase_ms']
        print(sys.argv[1], 'ms', round(d['ms_per_step'],1), {k:round(v,1) for k,v in p.items()})
PY
}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp2_gputest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp2_gputest.log
for D in 2 6 2 4; do
  NLG_GRID_DIV=$D timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/exp2_div$D.json 2>/dev/null; ph gpurun_out/exp2_div$D.json
done
NLG_GRID_DIV=6 timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp2_gputest_div6.log 2>&1; echo "tests div6 rc=$?"; tail -3 gpurun_out/exp2_gputest_div6.log
NLG_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e 2>&1 | grep "^\[nlg" | tail -30 > gpurun_out/exp2_trace_dev.log
NLG_NO_STAGE=1 NLG_TRACE=1 timeout 600 python tools/e2ediag.py 5 2>&1 | grep -v "^\[nlg\] clip" | tail -32 > gpurun_out/exp2_trace_nostage.log
