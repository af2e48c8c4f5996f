#!/bin/bash
# usage: scripts/gpu_ab.sh TAG VAR "VALS" WORKLOAD [pytest -k expr]
# bench one workload under each value of an env switch (A/B of kernel variants)
TAG=$1; VAR=$2; VALS=$3; W=$4; K=${5:-}; OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 -k "$K" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
fi
for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --workload $W --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline > $OUT/bench_${W}_$v.json 2> $OUT/bench_${W}_$v.err
done
echo done
