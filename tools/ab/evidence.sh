# round evidence: cfg2 launch list + ncu --set full of the main kernels (summarised on the box; the
# .ncu-rep files are deleted there except the dominant kernel's); cfg4 candidates fill
T=${T:-r01e}
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain_$T.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "launch rc=$?"
python tools/launch_summary.py gpurun_out/launches_$T.csv > gpurun_out/launches_$T.txt
summ() {  # $1 report base name
  python tools/ncu_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1_ncu_summary.txt 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source cuda,sass > /tmp/$1_src.csv 2>/dev/null
  python tools/srcprof.py /tmp/$1_src.csv 40 > gpurun_out/$1_source.txt 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/$1_raw.csv 2>/dev/null
}
for K in k_clipped k_row_asm k_singular k_full k_candidates; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/${T}_$K python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_${T}_$K.log 2>&1; echo "$K rc=$?"
  summ ${T}_$K
  [ $K = k_clipped ] || rm -f gpurun_out/${T}_$K.ncu-rep
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_candidates -s 1 -c 1 -o gpurun_out/${T}_cand4fill python bench.py --config 4 --emulate-shard 0/64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_${T}_cand4.log 2>&1; echo "cand4 rc=$?"
summ ${T}_cand4fill; rm -f gpurun_out/${T}_cand4fill.ncu-rep
du -sh gpurun_out
