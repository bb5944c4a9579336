# A/B on the GPU box: grid pitch, merge phase split (NLG_DEBUG bits 4 / 8 / 16), e2e trace
ph() { python - "$1" <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); p=d['roofline']['phase_ms']
        print(sys.argv[1], 'ms', round(d['ms_per_step'],1), {k:round(v,1) for k,v in p.items()})
PY
}
for D in 2 3 4 6 8 12; do
  NLG_GRID_DIV=$D timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/exp1_div$D.json 2>/dev/null; ph gpurun_out/exp1_div$D.json
done
for B in 4 8 16 12 28; do
  NLG_DEBUG=$B timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/exp1_dbg$B.json 2>/dev/null; ph gpurun_out/exp1_dbg$B.json
done
NLG_TRACE=1 timeout 600 python tools/e2ediag.py 5 > gpurun_out/exp1_e2e.log 2>&1; tail -60 gpurun_out/exp1_e2e.log
