#!/bin/bash
# usage: scripts/ab_env.sh TAG VAR "WORKLOADS" [pytest -k expr] -- each workload with VAR=1 and VAR=0
TAG=$1; VAR=$2; W=$3; K=${4:-}; OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 900 -k "$K" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
fi
for w in $W; do for v in 1 0; do
  env $VAR=$v timeout 600 python bench.py --workload $w --no-cpu-baseline > $OUT/bench_${w}_$v.json 2> $OUT/bench_${w}_$v.err
done; done
echo done
