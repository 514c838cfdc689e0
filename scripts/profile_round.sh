#!/bin/bash
# profile_round.sh TAG MODE [WORKLOAD] -- GPU-box helper for the committed ncu evidence.
#   MODE=launches: bench.py (WORKLOAD, default c2) once without ncu, then the same command under
#                  ncu's launch list (gpu__time_duration.sum) -> gpurun_out/TAG_launches_WORKLOAD.csv
#   MODE=full:     scripts/prof_step.py --workload WORKLOAD once without ncu, then under
#                  ncu --set full -> gpurun_out/TAG_WORKLOAD_full.ncu-rep
# Only one ncu command per invocation (one capture per gpurun call).
set -e
tag=$1; mode=$2; w=${3:-c2}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
if [ "$mode" = launches ]; then
  cmd="python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
  $cmd > gpurun_out/${tag}_bench_$w.log 2>&1
  $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
       --log-file gpurun_out/${tag}_launches_$w.csv $cmd > gpurun_out/${tag}_ncu_$w.log 2>&1
else
  cmd="python scripts/prof_step.py --workload $w --steps 3"
  $cmd > gpurun_out/${tag}_prof_$w.log 2>&1
  $NCU --set full --import-source on --clock-control none -f -o gpurun_out/${tag}_${w}_full $cmd \
       > gpurun_out/${tag}_ncu_$w.log 2>&1
fi
echo done
