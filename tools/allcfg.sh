for c in 1 2 3 5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 --ref-seconds 8 > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.err; echo "cfg$c rc=$?"
done
