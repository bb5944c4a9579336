# k_clipped variants on config 5 (NLG_CLIP_WL: 0 block queue, 1-4 k_clipped_cf shapes)
for V in 0 1 2 3 4; do
  echo -n "WL=$V "; NLG_CLIP_WL=$V timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']; print(round(d['ms_per_step'],1), 'clipped', round(p['ms_partial'],1))"
done
