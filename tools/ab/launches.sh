# launch list of one bench step (ncu timing only), summarised
T=${1:-x}; shift
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e "$@" > gpurun_out/plain_$T.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e "$@" > gpurun_out/ncul_$T.log 2>&1; echo "launch rc=$?"
python tools/launch_summary.py gpurun_out/launches_$T.csv | head -32
