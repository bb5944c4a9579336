# round evidence: launch list + ncu --set full of the given kernels (each capture after a plain run)
T=$1; shift
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain_$T.log 2>&1; echo "plain rc=$?"
if [ "$LAUNCH" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "launch rc=$?"
fi
for K in "$@"; do
  timeout 1200 ncu --set full --clock-control none $SRC -k regex:$K -c 1 -o gpurun_out/${T}_$K python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_${T}_$K.log 2>&1; echo "$K rc=$?"
done
ls -la gpurun_out/
