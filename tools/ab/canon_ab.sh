for E in "NLG_CLIP_WL=3" "NLG_CLIP_WL=3 NLG_DEBUG=32" "NLG_CLIP_WL=0" "NLG_CLIP_WL=0 NLG_DEBUG=32" "NLG_CLIP_WL=3"; do
  echo -n "$E: "; env $E timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); p=d['roofline']['phase_ms']; print(round(d['ms_per_step'],1), 'clipped', round(p['ms_partial'],1), 'merge', round(p['ms_merge'],1), 'cand', round(p['ms_candidates'],1))"
done
