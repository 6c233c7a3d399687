#!/bin/bash
# round-1 (session d) profiling pass, 1 GPU: launch lists + k_gs_cluster full capture (C2 runs)
O=gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_r1d.csv $B > $O/ncu_l2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gs_cluster -s 3 -c 1 -o $O/gs_cluster_c2_r1d $B > $O/ncu_f2.log 2>&1
ls $O
