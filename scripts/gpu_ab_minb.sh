#!/bin/bash
OUT=gpurun_out/${1:-abm}; mkdir -p $OUT
for v in 4 5; do for w in evd_r64 evd_c64; do
  JSVD_EVD_MINB=$v timeout 300 python bench.py --workload $w --steps 100 --warmup 3 --no-cpu-baseline > $OUT/bench_${w}_m$v.json 2>&1
done; done
JSVD_EVD_MINB=5 timeout 600 python -m pytest tests/test_gpu_evd.py -q -x > $OUT/pytest_m5.log 2>&1
echo done
