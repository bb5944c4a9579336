# per-phase stall mix of k_clipped_cf (config 5): one ncu --set full capture, binned by source line ranges
T=${1:-r02e}
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${T}_plain.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_clipped_cf -c 1 -o gpurun_out/${T}_cf python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/${T}_cf.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${T}_cf.csv 2>/dev/null
python tools/srcprof.py /tmp/${T}_cf.csv 25 "setup=nlg.cu:1968-2006" "classify=nlg.cu:2007-2080" "clipq=nlg.cu:2081-2091" "geom=nlg_geom.cuh:1-400" "moments=nlg.cu:2092-2137+nlg.cu:1420-1480" "fold=nlg.cu:2138-2170+nlg.cu:1300-1419" "store=nlg.cu:2171-2215" > gpurun_out/${T}_cf_bins.txt 2>&1
python tools/ncu_summary.py gpurun_out/${T}_cf.ncu-rep > gpurun_out/${T}_cf_ncu_summary.txt 2>&1
gzip -c /tmp/${T}_cf.csv > gpurun_out/${T}_cf_source.csv.gz; rm -f gpurun_out/${T}_cf.ncu-rep
