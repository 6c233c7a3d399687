#!/bin/bash
# round-1 profiling pass: traces, launch lists and ncu full captures of the top kernels
O=gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
CHROMA_FREE_TRACE=1 python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/c3_trace.json 2> $O/c3_trace.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv $B > $O/ncu_l2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv $B --workload c3 > $O/ncu_l3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gs_d1 -s 3 -c 1 -o $O/gs_d1_c2 $B > $O/ncu_f2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_color_light|k_heavy_waves|k_losers_light" -s 6 -c 4 -o $O/free_c3 $B --workload c3 > $O/ncu_f3.log 2>&1
ls -la $O
