#!/bin/bash
# usage: scripts/gpu_round_end.sh TAG -- the round-end evidence in one call:
# GPU tests, smoke, the default bench (+ oracle baseline), the reference arm,
# every workload's bench line, the default bench's ncu launch list, and one
# ncu --set full capture of each workload's kernel (each after its own
# command exited 0 without ncu)
TAG=${1:-final}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nproc > $OUT/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" > $OUT/lscpu.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 400 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "rc=$?" >> $OUT/bench_default.err
timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench_default_20.json 2> $OUT/bench_default_20.err; echo "rc=$?" >> $OUT/bench_default_20.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "rc=$?" >> $OUT/bench_reference.err
for w in ${WORKLOADS:-evd_r64 evd_c32 step_r64 step_c64 batched_c64 gesvj_r64 dist_c64 norm_c64 gs_r64}; do
  timeout 1200 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo "rc=$?" >> $OUT/bench_$w.err
done
B="python bench.py --no-cpu-baseline --warmup 3"
$B --steps 20 > $OUT/plain_launch.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_evd_c64.csv \
  $B --steps 20 > $OUT/ncu_launch.log 2>&1
for w in ${KW:-evd_c64 evd_r64 evd_c32 step_r64 step_c64 batched_c64 norm_c64 gs_r64}; do
  case $w in evd_c64) K=evd2_vec2;; evd_r64) K=evd2_scalar;; evd_c32) K=evd2f_;; step_*) K=step_kernel;;
    batched_c64) K=batched_fast;; norm_c64) K=norm_ef;; gs_r64) K=dgsscl;; esac
  S=5; [ $w = batched_c64 ] && S=3
  $B --workload $w --steps 4 > $OUT/plain_$w.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
    -o $OUT/prof_$w $B --workload $w --steps 4 > $OUT/ncu_$w.log 2>&1
done
echo done
