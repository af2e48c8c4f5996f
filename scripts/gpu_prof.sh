#!/bin/bash
# usage: scripts/gpu_prof.sh TAG -- launch list of the default bench + ncu --set full of the top kernels
TAG=${1:-prof}; OUT=gpurun_out/$TAG; mkdir -p $OUT
B="python bench.py --no-cpu-baseline --warmup 3"
$B --steps 20 > $OUT/plain_evd.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_evd_c64.csv \
  $B --steps 20 > $OUT/ncu_launch.log 2>&1
for w in ${KW:-evd_c64 evd_r64 step_c64 step_r64 batched_c64}; do
  case $w in evd_c32) K=evd2f_; S=5;; evd_*) K=evd2_; S=5;; step_*) K=step_kernel; S=5;; batched_c64) K=batched_svd; S=3;; esac
  $B --workload $w --steps 4 > $OUT/plain_$w.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
    -o $OUT/prof_$w $B --workload $w --steps 4 > $OUT/ncu_$w.log 2>&1
done
echo done
