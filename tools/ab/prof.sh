# usage: bash tools/prof.sh <kernel-regex> <outname> [bench args...]
K=$1; OUT=$2; shift 2
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e "$@" > gpurun_out/plain_$OUT.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/$OUT python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e "$@" > gpurun_out/ncu_$OUT.log 2>&1; echo "ncu rc=$?"
