for D in 0 4 8 12 16 28; do
  echo "dbg=$D"; NLG_DEBUG=$D timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(d['roofline']['phase_ms']['ms_merge'], d['roofline']['phase_ms']['ms_candidates'], d['roofline']['phase_ms']['ms_partial'])"
done
