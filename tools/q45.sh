timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for a in "--config 4 --emulate-shard 0/32 --steps 1 --warmup 1" "--config 5 --steps 2 --warmup 1" "--config 1 --steps 5 --warmup 3"; do
  timeout 900 python bench.py $a --no-cpu --no-e2e > gpurun_out/q.json 2> gpurun_out/q.err; echo "[$a] rc=$?"; python tools/show.py gpurun_out/q.json 2>/dev/null | head -3
done
