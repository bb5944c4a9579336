set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?"
tail -3 gpurun_out/bench3.err
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu3.log 2>&1; echo "ncu rc=$?"
