#!/bin/bash
# 1 GPU: GPU suite, smoke, bench C2 (default) and C3, reference arm, C2 launch list
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/e1_pytest.log 2>&1; echo "pytest rc=$?" >> $O/e1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/e1_smoke.log 2>&1; echo "smoke rc=$?" >> $O/e1_smoke.log
timeout 600 python bench.py > $O/e1_bench_c2_n1.json 2> $O/e1_bench_c2_n1.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > $O/e1_bench_c3_n1.json 2> $O/e1_bench_c3_n1.err
timeout 300 python bench.py --impl reference > $O/e1_bench_ref.json 2> $O/e1_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/e1_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/e1_ncu.log 2>&1
tail -3 $O/e1_pytest.log; tail -2 $O/e1_smoke.log
cat $O/e1_bench_c2_n1.json $O/e1_bench_c3_n1.json $O/e1_bench_ref.json
