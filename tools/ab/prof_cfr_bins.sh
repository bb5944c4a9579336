# per-phase stall mix of k_clipped_cfr (config 5): one ncu --set full capture, binned by source line ranges
# (the ranges follow nlg.cu: check them against the kernel's phase comments before a run)
T=${1:-r02l}
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${T}_plain.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_clipped_cfr -c 1 -o gpurun_out/${T}_cfr python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/${T}_cfr.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${T}_cfr.csv 2>/dev/null
python tools/srcprof.py /tmp/${T}_cfr.csv 40 "setup=nlg.cu:2259-2313" "classify=nlg.cu:2314-2394" "clipq=nlg.cu:2395-2416" "geom=nlg_geom.cuh:1-400" "moments=nlg.cu:2417-2466+nlg.cu:1420-1483" "fold=nlg.cu:2467-2504+nlg.cu:1300-1419" "store=nlg.cu:2505-2560" > gpurun_out/${T}_cfg5_k_clipped_cfr_phase_bins.txt 2>&1
python tools/srcprof.py /tmp/${T}_cfr.csv 40 > gpurun_out/${T}_cfg5_k_clipped_cfr_source.txt 2>&1
python tools/ncu_summary.py gpurun_out/${T}_cfr.ncu-rep > gpurun_out/${T}_cfg5_k_clipped_cfr_ncu_summary.txt 2>&1
rm -f gpurun_out/${T}_cfr.ncu-rep
