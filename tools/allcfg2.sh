# all configs, bench lines with cpu baseline (cfg4: rank 0 of 8 projection)
for c in 1 2 3 5; do
  W=3; S=5; if [ $c = 5 ]; then S=3; fi
  timeout 1200 python bench.py --config $c --steps $S --warmup $W --ref-seconds 8 > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.err; echo "cfg$c rc=$?"
  python tools/show.py gpurun_out/cfg$c.json 2>/dev/null | head -2
done
timeout 1500 python bench.py --config 4 --emulate-shard 0/8 --steps 2 --warmup 3 --ref-seconds 8 --no-e2e > gpurun_out/cfg4.json 2> gpurun_out/cfg4.err; echo "cfg4 rc=$?"
python tools/show.py gpurun_out/cfg4.json 2>/dev/null | head -2
