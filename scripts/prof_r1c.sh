#!/bin/bash
# round-1 final profiling pass (1 GPU)
O=gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
python scripts/probe_c1.py > $O/c1_probe.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_final.csv $B > $O/ncu_l2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_final.csv $B --workload c3 > $O/ncu_l3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gs_cluster -s 3 -c 1 -o $O/gs_cluster_c2_final $B > $O/ncu_f2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_color_light|k_color_tiny|k_heavy_waves|k_losers" -s 12 -c 5 -o $O/free_c3_final $B --workload c3 > $O/ncu_f3.log 2>&1
ls $O
