#!/usr/bin/env bash
# The profiling recipe behind profiles/ (B200_PROFILING.md), for one workload:
#   gpurun --timeout 1800 -- 'bash scripts/profile.sh c3 k_gs_chunked'
# 1. the bench line without ncu; 2. every launch of one bench step with its device
# time; 3. one --set full capture of the named kernel.  Outputs in gpurun_out/.
set -euo pipefail
WL=${1:-c3}
KERNEL=${2:-k_gs_chunked}
CMD="python bench.py --workload $WL --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-free"
$CMD > gpurun_out/prof_${WL}_plain.json 2> gpurun_out/prof_${WL}_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof_${WL}_launches.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:${KERNEL} -c 1 \
    -o gpurun_out/prof_${WL}_${KERNEL} $CMD > gpurun_out/prof_${WL}_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_${WL}_launches.csv > gpurun_out/prof_${WL}_launches_summary.txt
