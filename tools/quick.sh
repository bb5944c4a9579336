# quick GPU check: parity tests + one bench line (phase times)
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e "$@" > gpurun_out/quick.json 2> gpurun_out/quick.err; echo "bench rc=$?"; tail -2 gpurun_out/quick.err
