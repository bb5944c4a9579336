# GPU check: full gpu test suite (analytic on, then off for the kid 2/3 fixtures), cfg2 + cfg4-shard bench lines
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests.log
NLG_NO_ANALYTIC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/gputests_noan.log 2>&1; echo "tests(no analytic) rc=$?"; tail -2 gpurun_out/gputests_noan.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/q2.json 2> gpurun_out/q2.err; echo "cfg2 rc=$?"; python tools/show.py gpurun_out/q2.json | head -3
timeout 900 python bench.py --config 4 --emulate-shard 0/32 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/q4.json 2> gpurun_out/q4.err; echo "cfg4/32 rc=$?"; python tools/show.py gpurun_out/q4.json | head -3
