#!/bin/bash
# round-1 (session d) 1-GPU pass: full GPU suite, bench (C2, C3), launch list, k_gs_cluster full capture
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_final.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_final.log 2>&1; echo "smoke rc=$?" >> $O/smoke_final.log
timeout 600 python bench.py > $O/bench_final_c2.json 2> $O/bench_final_c2.err
timeout 600 python bench.py --workload c3 > $O/bench_final_c3.json 2> $O/bench_final_c3.err
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_r1d.csv $B > $O/ncu_l2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gs_cluster -s 3 -c 1 -o $O/gs_cluster_c2_r1d $B > $O/ncu_f2.log 2>&1
tail -2 $O/pytest_gpu_final.log; tail -2 $O/smoke_final.log
for f in $O/bench_final_c2.json $O/bench_final_c3.json; do python -c "import json; d=json.load(open('$f')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['value'], d['e2e']['value'] if d.get('e2e') else None)"; done
