#!/bin/bash
# usage: scripts/gpu_evd_iter.sh TAG -- EVD iteration: primitive + EVD parity
# tests, the default bench line (200 and 20 launches), one ncu capture of the
# complex EVD kernel (instructions executed, stall samples per source line)
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_evd.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for i in 0 1; do
  timeout 300 python bench.py --no-cpu-baseline > $OUT/bench_200_$i.json 2> $OUT/bench_200_$i.err
  timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 3 > $OUT/bench_20_$i.json 2> $OUT/bench_20_$i.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:evd2_vec2 -s 5 -c 1 \
  -o $OUT/prof_evd_c64 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > $OUT/ncu.log 2>&1
echo done
