#!/bin/bash
# usage: scripts/gpu_full.sh TAG -- the round-end sequence: smoke, default bench (with the
# oracle baseline), the reference arm, and the remaining workloads' bench lines
TAG=${1:-full}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nproc > $OUT/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" > $OUT/lscpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "rc=$?" >> $OUT/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "rc=$?" >> $OUT/bench_reference.err
for w in ${WORKLOADS:-evd_r64 step_r64 step_c64 batched_c64 gesvj_r64 dist_c64}; do
  timeout 1200 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo "rc=$?" >> $OUT/bench_$w.err
done
echo done
