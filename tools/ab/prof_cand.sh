summ() {
  python tools/ncu_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1_ncu_summary.txt 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source cuda,sass > /tmp/$1_src.csv 2>/dev/null
  python tools/srcprof.py /tmp/$1_src.csv 50 > gpurun_out/$1_source.txt 2>&1
  rm -f gpurun_out/$1.ncu-rep
}
timeout 600 python bench.py --config 4 --emulate-shard 0/64 --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_candidates<\(bool\)1>' -c 1 -o gpurun_out/cand4f python bench.py --config 4 --emulate-shard 0/64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_cand4f.log 2>&1; echo "ncu rc=$?"
summ cand4f
