#!/bin/bash
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
for v in 0 1; do for w in evd_r64 evd_c64; do
  JSVD_EVD_PERSIST=$v timeout 300 python bench.py --workload $w --steps 40 --warmup 3 --no-cpu-baseline > $OUT/bench_${w}_p$v.json 2>&1
done; done
echo done
