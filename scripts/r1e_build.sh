#!/bin/bash
# 1 GPU: world build k_rowlen / k_fill fast paths — full GPU suite, build phase split, C2 bench
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/b_pytest.log 2>&1; echo "pytest rc=$?" >> $O/b_pytest.log
CHROMA_BUILD_TIMING=1 timeout 300 python scripts/probe_e2e.py 2>&1 | tail -8 > $O/b_e2e.log
timeout 300 python scripts/probe_pin.py > $O/b_pin.log 2>&1
timeout 300 python bench.py > $O/b_bench_c2.json 2> $O/b_bench_c2.err
tail -2 $O/b_pytest.log; cat $O/b_e2e.log $O/b_pin.log
python -c "import json; d=json.load(open('$O/b_bench_c2.json')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['value'], d['e2e'], d['cpu_baseline'])"
