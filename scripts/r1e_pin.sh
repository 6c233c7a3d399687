#!/bin/bash
# 1 GPU: run_distributed colours returned in pinned host memory
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_free_gpu.py -m gpu -x -q > $O/n_pytest.log 2>&1; echo "pytest rc=$?" >> $O/n_pytest.log
timeout 300 python scripts/probe_e2e.py > $O/n_e2e.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > $O/n_bench_c2.json 2> $O/n_bench_c2.err
tail -2 $O/n_pytest.log; tail -3 $O/n_e2e.log
python -c "import json; d=json.load(open('$O/n_bench_c2.json')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['value'], d['e2e'])"
