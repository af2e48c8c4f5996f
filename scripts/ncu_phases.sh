#!/bin/bash
# usage: scripts/ncu_phases.sh TAG -- one ncu --set full capture per hot kernel
# (after its own plain run exited 0), for scripts/phase_breakdown.py
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
B="python bench.py --no-cpu-baseline --warmup 3"
for w in ${KW:-evd_c64 step_r64 step_c64 batched_c64}; do
  case $w in evd_c64) K=evd2_vec2;; evd_r64) K=evd2_scalar;; step_*) K=step_kernel;;
    batched_c64) K=batched_fast;; norm_c64) K=norm_ef;; gs_r64) K=dgsscl;; esac
  S=5; [ $w = batched_c64 ] && S=3
  $B --workload $w --steps 4 > $OUT/plain_$w.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
    -o $OUT/prof_$w $B --workload $w --steps 4 > $OUT/ncu_$w.log 2>&1
done
echo done
