#!/bin/bash
# 1 GPU, final code of round 1: GPU suite, smoke, bench C2/C3/reference, C2 launch list, k_run_step full capture
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/f_pytest.log 2>&1; echo "pytest rc=$?" >> $O/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/f_smoke.log 2>&1; echo "smoke rc=$?" >> $O/f_smoke.log
timeout 600 python bench.py > $O/f_bench_c2.json 2> $O/f_bench_c2.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > $O/f_bench_c3.json 2> $O/f_bench_c3.err
timeout 300 python bench.py --impl reference > $O/f_bench_ref.json 2> $O/f_bench_ref.err
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/f_launches_c2.csv $B > $O/f_ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_run_step -s 100 -c 1 -o $O/f_run_step_c2 $B > $O/f_ncu_f.log 2>&1
tail -2 $O/f_pytest.log; tail -2 $O/f_smoke.log
for f in $O/f_bench_c2.json $O/f_bench_c3.json; do python -c "import json; d=json.load(open('$f')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['value'], d['e2e']['value'] if d.get('e2e') else None, d['clocks'])"; done
cat $O/f_bench_ref.json; tail -3 $O/f_ncu_f.log
