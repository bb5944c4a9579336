# Evidence for one config (run on the GPU box from the repo root):
#   bash tools/prof_cfg.sh TAG CONFIG [kernel regex ...]
# 1. the plain bench step (must exit 0 before any ncu run);
# 2. the ncu launch list of one step (cold, serialised) -> profiles-ready summary;
# 3. one `ncu --set full` capture per named kernel (first launch), summarised.
T=$1; C=$2; shift 2
timeout 900 python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${T}_plain.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${T}_ncul.log 2>&1; echo "launch rc=$?"
python tools/launch_summary.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches.txt 2>&1
for KS in "$@"; do
  # KERNEL or KERNEL:SKIP (skip the first SKIP launches of that kernel)
  K=${KS%%:*}; SKIP=0; [ "$KS" != "$K" ] && SKIP=${KS##*:}
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip $SKIP -c 1 -o gpurun_out/${T}_$K \
    python bench.py --config $C --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/${T}_ncu_$K.log 2>&1; echo "ncu $K rc=$?"
  python tools/ncu_summary.py gpurun_out/${T}_$K.ncu-rep > gpurun_out/${T}_${K}_ncu_summary.txt 2>&1
  ncu -i gpurun_out/${T}_$K.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${T}_$K.csv 2>/dev/null
  python tools/srcprof.py /tmp/${T}_$K.csv 40 > gpurun_out/${T}_${K}_source.txt 2>&1
  rm -f gpurun_out/${T}_$K.ncu-rep
done
