# final round evidence: tests, smoke, bench lines of all configs, reference arm, launch list, ncu of the dominant kernel
T=r01k
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/default.json 2> gpurun_out/default.err; echo "default rc=$?"; python tools/show.py gpurun_out/default.json 2>/dev/null | head -2
for c in 1 3 5; do
  W=3; S=5; if [ $c = 5 ]; then S=3; fi
  timeout 1200 python bench.py --config $c --steps $S --warmup $W --ref-seconds 8 > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.err; echo "cfg$c rc=$?"
  python tools/show.py gpurun_out/cfg$c.json 2>/dev/null | head -2
done
timeout 1500 python bench.py --config 4 --emulate-shard 0/8 --steps 2 --warmup 3 --ref-seconds 8 --no-e2e > gpurun_out/cfg4.json 2> gpurun_out/cfg4.err; echo "cfg4 rc=$?"
python tools/show.py gpurun_out/cfg4.json 2>/dev/null | head -2
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref2.json 2> gpurun_out/ref2.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "launch rc=$?"
python tools/launch_summary.py gpurun_out/launches_$T.csv > gpurun_out/launches_$T.txt
for K in k_clipped k_row_asm; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/${T}_$K python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_${T}_$K.log 2>&1; echo "$K rc=$?"
  python tools/ncu_summary.py gpurun_out/${T}_$K.ncu-rep > gpurun_out/${T}_${K}_ncu_summary.txt 2>&1
  ncu -i gpurun_out/${T}_$K.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${T}_$K.csv 2>/dev/null
  python tools/srcprof.py /tmp/${T}_$K.csv 40 > gpurun_out/${T}_${K}_source.txt 2>&1
  rm -f gpurun_out/${T}_$K.ncu-rep
done
du -sh gpurun_out
