#!/bin/bash
OUT=gpurun_out/${1:-pr}; mkdir -p $OUT
B="python bench.py --no-cpu-baseline --warmup 3 --workload evd_r64"
$B --steps 20 > $OUT/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:evd2_vec2 -s 5 -c 1 \
  -o $OUT/prof_evd_r64 $B --steps 10 > $OUT/ncu.log 2>&1
echo done
