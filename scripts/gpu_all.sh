#!/bin/bash
# usage: scripts/gpu_all.sh TAG -- GPU tests, default bench, every workload's bench line, launch list
TAG=${1:-all}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/smi.txt 2>&1; nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
for w in ${WORKLOADS:-evd_r64 step_r64 step_c64 batched_c64 gesvj_r64}; do
  timeout 900 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo "rc=$?" >> $OUT/bench_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
echo done
