#!/bin/bash
# usage: scripts/gpu_quick.sh TAG -- GPU tests (per-test timeout, durations) + short benches
TAG=${1:-quick}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout ${PYT:-1200} python -m pytest tests -m gpu -q -rf --timeout 400 --durations=30 ${PYARGS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for w in ${WORKLOADS:-evd_c64 evd_r64 step_r64 step_c64 batched_c64}; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo "rc=$?" >> $OUT/bench_$w.err
done
echo done
