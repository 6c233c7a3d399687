#!/bin/bash
# round-1 re-entry check: full GPU suite, smoke, default bench, C3 bench (1 GPU)
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --workload c3 > $O/bench_c3.json 2> $O/bench_c3.err
tail -3 $O/pytest_gpu.log; cat $O/bench_c2.json $O/bench_c3.json
