timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 1 2 3 5; do
  W=3; S=5; if [ $c = 5 ]; then S=3; fi
  timeout 1200 python bench.py --config $c --steps $S --warmup $W --ref-seconds 8 > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.err; echo "cfg$c rc=$?"
  python tools/show.py gpurun_out/cfg$c.json 2>/dev/null | head -2
done
timeout 1500 python bench.py --config 4 --emulate-shard 0/8 --steps 2 --warmup 3 --ref-seconds 8 --no-e2e > gpurun_out/cfg4.json 2> gpurun_out/cfg4.err; echo "cfg4 rc=$?"
python tools/show.py gpurun_out/cfg4.json 2>/dev/null | head -2
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref2.json 2> gpurun_out/ref2.err; echo "ref rc=$?"; cat gpurun_out/ref2.json | head -c 600; echo
