#!/bin/bash
# 1 GPU: parity subset touching round-0 schedules + C2 bench (P=1 and 4 virtual ranks via trace)
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_free_gpu.py -m gpu -x -q > $O/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $O/pytest_quick.log
CHROMA_LEVEL_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c2_trace.json 2> $O/bench_c2_trace.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c2_quick.json 2> $O/bench_c2_quick.err
tail -2 $O/pytest_quick.log; grep -E "levels|cluster" $O/bench_c2_trace.err | head -3
python -c "import json; d=json.load(open('$O/bench_c2_quick.json')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['value'])"
