#!/bin/bash
# 1 GPU, end of round: GPU suite, smoke, bench C2 (default), reference arm
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/g1_pytest.log 2>&1; echo "pytest rc=$?" >> $O/g1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/g1_smoke.log 2>&1; echo "smoke rc=$?" >> $O/g1_smoke.log
timeout 600 python bench.py > $O/g1_bench_c2_n1.json 2> $O/g1_bench_c2_n1.err
timeout 300 python bench.py --impl reference > $O/g1_bench_ref.json 2> $O/g1_bench_ref.err
tail -3 $O/g1_pytest.log; tail -2 $O/g1_smoke.log
cat $O/g1_bench_c2_n1.json $O/g1_bench_ref.json
