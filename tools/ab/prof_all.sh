# current-version evidence: launch list of one bench step + ncu --set full of k_clipped (source page)
T=${1:-v7}
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain_$T.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncul_$T.log 2>&1; echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_clipped -c 1 -o gpurun_out/clip_$T python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncuf_$T.log 2>&1; echo "full rc=$?"
