timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for a in "--config 3 --steps 3 --warmup 3" "--config 2 --steps 3 --warmup 3"; do
  timeout 900 python bench.py $a --no-cpu --no-e2e > gpurun_out/q.json 2> gpurun_out/q.err; echo "[$a] rc=$?"; python tools/show.py gpurun_out/q.json 2>/dev/null | head -3
done
