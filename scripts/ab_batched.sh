#!/bin/bash
# A/B of the configs[3] kernels in one call: batched_fast.cu (default), batched.cu's
# kernel in its fast mode (JSVD_BATCHED_KERNEL=0) and in exact mode (JSVD_BATCHED_FAST=0)
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in "X=1" "JSVD_BATCHED_KERNEL=0" "JSVD_BATCHED_FAST=0"; do
  env $v timeout 600 python bench.py --workload batched_c64 --no-cpu-baseline > $OUT/bench_$v.json 2> $OUT/bench_$v.err
done
echo done
