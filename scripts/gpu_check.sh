#!/bin/bash
# usage: scripts/gpu_check.sh TAG [ncu-kernel-regex] -- GPU tests + bench (+ optional ncu full capture)
TAG=${1:-run}; KRE=${2:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
if [ -n "$KRE" ]; then
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_short.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 5 -c 1 \
     -o $OUT/prof python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.log 2>&1
fi
echo done
