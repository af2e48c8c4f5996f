#!/bin/bash
# usage: scripts/gpu_batched_iter.sh TAG -- batched-SVD iteration: its GPU
# parity tests, two bench lines, one ncu capture of the configs[3] kernel
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_svd.py -m gpu -x -q -k "batched or config4" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for i in 0 1; do
  timeout 600 python bench.py --workload batched_c64 --no-cpu-baseline > $OUT/bench_$i.json 2> $OUT/bench_$i.err
done
[ -n "$NCU" ] && timeout 900 ncu --set full --clock-control none --import-source on -k regex:batched_fast -s 3 -c 1 \
  -o $OUT/prof_batched_c64 python bench.py --workload batched_c64 --no-cpu-baseline --steps 4 --warmup 3 > $OUT/ncu.log 2>&1
echo done
