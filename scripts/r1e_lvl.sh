#!/bin/bash
# 1 GPU: run level build (head membership, warp-wide expansion, lazily grown host size copy)
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/l_pytest.log 2>&1; echo "pytest rc=$?" >> $O/l_pytest.log
CHROMA_LEVEL_TRACE=1 timeout 300 python scripts/probe_e2e.py 2>&1 | grep -E "levels|h2d|level" | tail -3 > $O/l_e2e.log 2>&1
CHROMA_LEVEL_TRACE=1 timeout 300 python tests/c1_probe.py 2>&1 | grep -E "levels\]|^run|^8b" > $O/l_c1.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > $O/l_bench_c2.json 2> $O/l_bench_c2.err
tail -2 $O/l_pytest.log; cat $O/l_e2e.log $O/l_c1.log
python -c "import json; d=json.load(open('$O/l_bench_c2.json')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['value'], d['e2e'])"
