#!/bin/bash
# usage: scripts/ab_lib.sh TAG ALT_LIB "WORKLOADS" -- bench each workload with the
# default library and with ALT_LIB (JSVD_LIB), in one call
TAG=$1; ALT=$2; W=$3; OUT=gpurun_out/$TAG; mkdir -p $OUT
for w in $W; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $OUT/bench_${w}_default.json 2> $OUT/bench_${w}_default.err
  JSVD_LIB=$ALT timeout 600 python bench.py --workload $w --no-cpu-baseline > $OUT/bench_${w}_alt.json 2> $OUT/bench_${w}_alt.err
done
echo done
