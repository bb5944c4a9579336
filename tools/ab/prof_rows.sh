bash tools/launches.sh rows2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_row_asm -c 1 -o gpurun_out/rows2 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_rows2.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_row_asm -s 3 -c 1 -o gpurun_out/rows4 python bench.py --config 4 --emulate-shard 0/64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_rows4.log 2>&1; echo "ncu4 rc=$?"
