# e2e check: parity tests + e2e breakdown + full bench line
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/e2ediag.py > gpurun_out/e2ediag.log 2>&1; echo "diag rc=$?"; tail -12 gpurun_out/e2ediag.log
timeout 600 python bench.py > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench rc=$?"; cat gpurun_out/bench_e2e.json; tail -2 gpurun_out/bench_e2e.err
