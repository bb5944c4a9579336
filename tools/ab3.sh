# A/B on config 3 (peridynamic, 6x6 blocks)
for rep in 1 2; do
  for lib in "$@"; do
    NLG_LIBRARY=$PWD/$lib timeout 600 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab3.json 2>/dev/null
    python - "$lib" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab3.json"))
ph = d["roofline"]["phase_ms"]
print(f"{sys.argv[1]:24s} step {d['ms_per_step']:8.2f}  " + "  ".join(f"{k[3:]} {v:7.2f}" for k, v in ph.items()))
PY
  done
done
