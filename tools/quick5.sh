timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for i in 1 2 3; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/quick_$i.json 2>/dev/null; python tools/show.py gpurun_out/quick_$i.json | head -2; done
