for c in 1 2 3 5; do
  W=3; S=5; if [ $c = 5 ]; then S=3; fi
  timeout 1200 python bench.py --config $c --steps $S --warmup $W --ref-seconds 8 > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.err; echo "cfg$c rc=$?"
  python tools/show.py gpurun_out/cfg$c.json | head -3
done
