#!/usr/bin/env bash
# Round-2 ncu captures of the new kernels (each command ran clean without ncu first).
set -u
C5="python bench.py --workload c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-free"
C3="python bench.py --workload c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-free"
R2="python scripts/probe_rounds.py 24 2"
$C5 > gpurun_out/p_c5.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_masks_all|k_detect_all" -c 2 \
      -o gpurun_out/r2_net_c5 $C5 > gpurun_out/p_c5_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5.csv $C5 \
    > /dev/null 2>&1
$C3 > gpurun_out/p_c3.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_count_d1 -c 1 \
      -o gpurun_out/r2_verify_c3 $C3 > gpurun_out/p_c3_ncu.log 2>&1
$R2 > gpurun_out/p_r2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_emit_short|k_changed_events" -c 4 \
      -o gpurun_out/r2_detect_c3p2 $R2 > gpurun_out/p_r2_ncu.log 2>&1
ls -la gpurun_out/*.ncu-rep
