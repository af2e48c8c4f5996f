#!/bin/bash
# A/B of the step kernel geometry (JSVD_STEP_SMEM) on configs[2]
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_svd.py -q -rf --timeout 600 -k "sweep_step or gesvj_bitwise or config3" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 1 0; do
  for w in step_r64 gesvj_r64; do
    JSVD_STEP_SMEM=$v timeout 600 python bench.py --workload $w --no-cpu-baseline > $OUT/bench_${w}_$v.json 2> $OUT/bench_${w}_$v.err
  done
done
echo done
