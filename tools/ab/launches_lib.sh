# per-kernel launch summary for a library variant: bash tools/launches_lib.sh lib.so tag
L=$1; T=$2
NLG_LIBRARY=$PWD/$L timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "launch rc=$?"
python tools/launch_summary.py gpurun_out/launches_$T.csv | head -40
