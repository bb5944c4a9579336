# A/B timing of library variants: bash tools/ab.sh libA.so libB.so ... (alternating runs)
for rep in 1 2; do
  for lib in "$@"; do
    NLG_LIBRARY=$PWD/$lib timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
    python - "$lib" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
ph = d["roofline"]["phase_ms"]
print(f"{sys.argv[1]:24s} step {d['ms_per_step']:7.2f}  " + "  ".join(f"{k[3:]} {v:6.2f}" for k, v in ph.items()))
PY
  done
done
