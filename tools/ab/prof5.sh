T=r01i_cfg5
timeout 600 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_clipped -c 1 -o gpurun_out/${T}_k_clipped python bench.py --config 5 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_${T}.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/${T}_k_clipped.ncu-rep > gpurun_out/${T}_k_clipped_ncu_summary.txt 2>&1
ncu -i gpurun_out/${T}_k_clipped.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${T}.csv 2>/dev/null
python tools/srcprof.py /tmp/${T}.csv 40 > gpurun_out/${T}_k_clipped_source.txt 2>&1
rm -f gpurun_out/${T}_k_clipped.ncu-rep
