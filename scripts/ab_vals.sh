#!/bin/bash
# usage: scripts/ab_vals.sh TAG VAR "VALUES" "BENCH ARGS" -- one bench line per value of VAR
TAG=$1; VAR=$2; VALS=$3; ARGS=$4; OUT=gpurun_out/$TAG; mkdir -p $OUT
for rep in 0 1; do for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --no-cpu-baseline $ARGS > $OUT/bench_${v}_$rep.json 2> $OUT/bench_${v}_$rep.err
done; done
echo done
